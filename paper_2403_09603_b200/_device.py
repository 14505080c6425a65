"""Device plumbing: tensors in and out of the C ABI, workspaces, error bits.

PyTorch is used only for device memory, streams and copies; all compute is
in ``libvtrain_b200.so``.  Host (NumPy / list) inputs are the drop-in
parity mode of the reference API (copied to HBM, results copied back); CUDA
tensors are zero-copy when contiguous and 32-byte aligned.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

_WS: dict[tuple, torch.Tensor] = {}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2403_09603_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    _lib.lib()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(device=None) -> int:
    return int(torch.cuda.current_stream(device).cuda_stream)


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else int(t.data_ptr())


def aligned_f64(t: torch.Tensor) -> torch.Tensor:
    """Contiguous FP64 CUDA tensor whose data pointer is 32-byte aligned."""
    if t.dtype != torch.float64:
        t = t.to(torch.float64)
    t = t.contiguous()
    if t.data_ptr() % 32:
        t = t.clone()
    return t


def to_device_f64(x) -> tuple[torch.Tensor, bool, tuple]:
    """(flat FP64 CUDA tensor, came_from_host, result shape).

    Result shape follows the reference: the input's shape, except 0-d -> (1,)
    (fpround.py:135 ``out.reshape(np.shape(x)) if np.shape(x) else out``).
    """
    dev = require_cuda()
    if isinstance(x, torch.Tensor) and x.is_cuda:
        shape = tuple(x.shape) if x.dim() else (1,)
        return aligned_f64(x.reshape(-1)), False, shape
    a = np.asarray(x.cpu().numpy() if isinstance(x, torch.Tensor) else x, dtype=np.float64)
    shape = a.shape if a.shape else (1,)
    t = torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).to(dev, non_blocking=False)
    return aligned_f64(t), True, shape


def back(t: torch.Tensor, host: bool, shape: tuple):
    t = t.reshape(shape)
    return t.cpu().numpy() if host else t


def workspace(nbytes: int, tag: str) -> torch.Tensor:
    """Per (device, tag) scratch buffer, grown on demand.  Operators that may
    run concurrently on different streams use different tags.  Zero-filled
    once at allocation (vt_round_log keeps an epoch header and epoch-tagged
    status words in it that must start out zero)."""
    key = (torch.cuda.current_device(), tag)
    ws = _WS.get(key)
    if ws is None or ws.numel() < nbytes:
        ws = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device="cuda")
        _WS[key] = ws
    return ws


class Flags:
    """Device int32 error word + int64 counters for one call."""

    def __init__(self, n_counters: int = 4, buf: torch.Tensor | None = None):
        # buf: a caller-owned, zeroed int64 slot of 2 + n_counters words (e.g. a
        # row of a per-step arena, so a step allocates nothing)
        self.buf = buf if buf is not None else torch.zeros(2 + n_counters, dtype=torch.int64, device="cuda")
        self.err_ptr = self.buf.data_ptr()
        self.cnt_ptr = self.buf.data_ptr() + 16

    def read(self) -> tuple[int, list[int]]:
        v = self.buf.tolist()
        return int(v[0]) & 0xFFFFFFFF, [int(c) for c in v[2:]]


def raise_fpround(err: int, neighbor_semantics: bool = False) -> None:
    """Reference check order: finite first, then range (fpround.py:131-134, 189-191)."""
    if err & _lib.ERR_NONFINITE:
        raise ValueError("non-finite value")
    if err & (_lib.ERR_RANGE | _lib.ERR_RANGE_NEIGHBOR):
        raise ValueError("out of representable range")
