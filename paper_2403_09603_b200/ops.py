"""Device-level north-star operators on CUDA tensors.

``round_and_log`` -- trainer side: FP64 tensor -> FP32 (or FP64) rounded
tensor + sparse log of every element whose rounding direction must be
recorded, i.e. whose distance to the rounding midpoint is within the
adaptive band (reference semantics: ``direction_array(x, b_r, tau) != 1``,
pkg/src/vtrain/fpround.py:164-177).  One fused kernel, one HBM pass.

``replay`` -- auditor side: FP64 tensor + sparse log -> rounded tensor with
the logged direction forced on every logged element (``rev_array``,
fpround.py:227-247), plus the correction count of
``protocol._AuditorChannel.process`` (protocol.py:212-216).

Sparse log layout (pinned here): one uint64 word per
logged element, ``(global_index << 1) | up`` with ``up = (code == UP)``,
strictly ascending.  It is the lossless recoding of the reference's dense
ternary stream: absent index -> code 1, bit 1 -> code 2, bit 0 -> code 0.
Words are stored in an int64 tensor (same bits).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import _device as D
from . import _lib
from .fpround import _check_b


class LogOverflow(RuntimeError):
    """The sparse log did not fit the provided capacity."""


class SparseLogError(ValueError):
    """A sparse log is not strictly ascending, or does not cover the tensor."""


@dataclass
class SparseLog:
    words: torch.Tensor  # int64 [count]: (global_index << 1) | up
    count: int

    def indices(self) -> torch.Tensor:
        return torch.bitwise_right_shift(self.words, 1)

    def up(self) -> torch.Tensor:
        return torch.bitwise_and(self.words, 1).to(torch.bool)


@dataclass
class PendingRound:
    """Result of an unchecked call (``check=False``): buffers + device flags."""

    y: torch.Tensor
    words: torch.Tensor
    flags: D.Flags

    def finish(self) -> tuple[torch.Tensor, SparseLog]:
        err, cnt = self.flags.read()
        D.raise_fpround(err)
        if cnt[0] > self.words.numel():
            raise LogOverflow(f"sparse log needs {cnt[0]} words, capacity {self.words.numel()}")
        return self.y, SparseLog(self.words[: cnt[0]], cnt[0])


def round_and_log(x: torch.Tensor, b_r: int, tau: float, *, out_dtype=torch.float32,
                  global_base: int = 0, out: torch.Tensor | None = None,
                  log_out: torch.Tensor | None = None, codes_out: torch.Tensor | None = None,
                  check: bool = True):
    """Fused rnd + direction + stream compaction (one kernel launch)."""
    _check_b(b_r)
    D.require_cuda()
    shape = tuple(x.shape) if x.dim() else (1,)
    t = D.aligned_f64(x.reshape(-1))
    n = t.numel()
    kind = _lib.OUT_F32 if out_dtype == torch.float32 else _lib.OUT_F64
    y = out if out is not None else torch.empty(n, dtype=out_dtype, device=t.device)
    words = log_out if log_out is not None else torch.empty(max(n, 1), dtype=torch.int64, device=t.device)
    ws = D.workspace(int(_lib.lib().vt_round_log_workspace(n)), "round_log")
    f = D.Flags()
    if n:
        _lib.call("vt_round_log", D.ptr(t), n, b_r, float(tau), kind, D.ptr(y),
                  D.ptr(words), words.numel(), int(global_base), None, None, D.ptr(codes_out),
                  None, 0, None, f.cnt_ptr, f.err_ptr, D.ptr(ws), ws.numel(), D.stream_ptr())
    pending = PendingRound(y.reshape(shape) if out is None else y, words, f)
    return pending.finish() if check else pending


def replay(x: torch.Tensor, b_r: int, log: SparseLog | torch.Tensor, *, out_dtype=torch.float32,
           global_base: int = 0, out: torch.Tensor | None = None, strict: bool = True,
           check: bool = True):
    """Fused rev with a sparse log; returns (y, corrections)."""
    _check_b(b_r)
    D.require_cuda()
    words = log.words if isinstance(log, SparseLog) else log
    words = words.contiguous()
    shape = tuple(x.shape) if x.dim() else (1,)
    t = D.aligned_f64(x.reshape(-1))
    n = t.numel()
    kind = _lib.OUT_F32 if out_dtype == torch.float32 else _lib.OUT_F64
    y = out if out is not None else torch.empty(n, dtype=out_dtype, device=t.device)
    ws = D.workspace(int(_lib.lib().vt_replay_workspace(n)), "replay")
    f = D.Flags()
    if n:
        _lib.call("vt_replay", D.ptr(t), n, b_r, _lib.LOG_SPARSE, D.ptr(words), words.numel(),
                  int(global_base), kind, D.ptr(y), f.cnt_ptr, f.err_ptr, D.ptr(ws), ws.numel(),
                  D.stream_ptr())
    if not check:
        return y, f
    err, cnt = f.read()
    if err & _lib.ERR_BAD_SPARSE:
        raise SparseLogError("sparse log is not strictly ascending")
    D.raise_fpround(err)
    if strict and n and (cnt[1] != 0 or cnt[2] != words.numel()):
        raise SparseLogError(
            f"sparse log covers words [{cnt[1]}, {cnt[2]}) of {words.numel()} for this tensor")
    return (y.reshape(shape) if out is None else y), cnt[0]


def normalized_distance(x: torch.Tensor, b_r: int) -> torch.Tensor:
    """p = |x - rnd(x)| / max(scale(x), 2^-126) per element (fpround.py:171-173)."""
    _check_b(b_r)
    t = D.aligned_f64(x.reshape(-1))
    out = torch.empty_like(t)
    f = D.Flags()
    if t.numel():
        _lib.call("vt_norm_distance", D.ptr(t), t.numel(), b_r, D.ptr(out), f.err_ptr, D.stream_ptr())
        D.raise_fpround(f.read()[0])
    return out.reshape(x.shape)
