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

    def finish(self, err: int | None = None, cnt: list | None = None) -> tuple[torch.Tensor, SparseLog]:
        if err is None:
            err, cnt = self.flags.read()
        D.raise_fpround(err)
        if cnt[0] > self.words.numel():
            raise LogOverflow(f"sparse log needs {cnt[0]} words, capacity {self.words.numel()}")
        return self.y, SparseLog(self.words[: cnt[0]], cnt[0])


def default_log_capacity(n: int) -> int:
    """Default sparse-log capacity (words) when the caller passes no log_out:
    1/8 of the elements (configs 0/1 log ~10%), at least 64 Ki words, at most
    n.  With check=True a call whose log needs more is re-run once with the
    exact size; with check=False finish() raises LogOverflow -- pass log_out
    (up to n words) for inputs that may log more than 1/8."""
    return max(1, min(n, max(n // 8, 1 << 16)))


def _out_kind(out_dtype) -> int:
    if out_dtype == torch.float32:
        return _lib.OUT_F32
    if out_dtype == torch.float64:
        return _lib.OUT_F64
    raise ValueError(f"out_dtype must be torch.float32 or torch.float64, got {out_dtype}")


def round_and_log(x: torch.Tensor, b_r: int, tau: float, *, out_dtype=torch.float32,
                  global_base: int = 0, out: torch.Tensor | None = None,
                  log_out: torch.Tensor | None = None, codes_out: torch.Tensor | None = None,
                  check: bool = True, workspace: torch.Tensor | None = None,
                  flags_out: torch.Tensor | None = None):
    """Fused rnd + direction + stream compaction (one kernel launch).

    Reentrant across streams and host threads: the call's scratch state lives
    in a workspace keyed by the current stream (or the caller's
    ``workspace``, a zero-initialised uint8 CUDA tensor of at least
    ``vt_round_log_workspace(n)`` bytes used by one stream at a time).
    ``flags_out`` (a zeroed int64[6] CUDA tensor: error bits, -, entry count,
    ...) replaces the per-call flag allocation, e.g. a row of a per-step
    arena, as ``round_and_log_adaptive``'s."""
    _check_b(b_r)
    D.require_cuda()
    shape = tuple(x.shape) if x.dim() else (1,)
    t = D.aligned_f64(x.reshape(-1))
    n = t.numel()
    kind = _out_kind(out_dtype)
    D.check_out(out, n, out_dtype, t.device, "out")
    D.check_out(log_out, 0, torch.int64, t.device, "log_out")
    D.check_out(codes_out, n, torch.uint8, t.device, "codes_out")
    y = out if out is not None else torch.empty(n, dtype=out_dtype, device=t.device)
    words = log_out if log_out is not None else torch.empty(default_log_capacity(n), dtype=torch.int64,
                                                            device=t.device)
    need = int(_lib.lib().vt_round_log_workspace(n))
    ws = workspace if workspace is not None else D.workspace(need, "round_log")
    D.check_out(ws, need, torch.uint8, t.device, "workspace")
    D.check_out(flags_out, 6, torch.int64, t.device, "flags_out")
    f = D.Flags(buf=flags_out)
    if n:
        _lib.call("vt_round_log", D.ptr(t), n, b_r, float(tau), kind, D.ptr(y),
                  D.ptr(words), words.numel(), int(global_base), None, None, D.ptr(codes_out),
                  None, 0, None, f.cnt_ptr, f.err_ptr, D.ptr(ws), ws.numel(), D.stream_ptr())
    pending = PendingRound(y.reshape(shape) if out is None else y, words, f)
    if not check:
        return pending
    err, cnt = f.read()
    if log_out is None and err == 0 and cnt[0] > words.numel():
        # more entries than the default capacity: once more with the exact size
        words = torch.empty(cnt[0], dtype=torch.int64, device=t.device)
        if flags_out is not None:
            flags_out.zero_()
        return round_and_log(x, b_r, tau, out_dtype=out_dtype, global_base=global_base, out=out,
                             log_out=words, codes_out=codes_out, check=True, workspace=workspace,
                             flags_out=flags_out)
    return pending.finish(err, cnt)


def replay(x: torch.Tensor, b_r: int, log: SparseLog | torch.Tensor, *, out_dtype=torch.float32,
           global_base: int = 0, out: torch.Tensor | None = None, strict: bool = True,
           check: bool = True, workspace: torch.Tensor | None = None, flags_out: torch.Tensor | None = None):
    """Fused rev with a sparse log; returns (y, corrections).  Reentrant
    across streams (workspace keyed by the current stream, or the caller's
    zeroed ``workspace`` of ``vt_replay_workspace(n)`` bytes); ``flags_out``
    as for ``round_and_log``."""
    _check_b(b_r)
    D.require_cuda()
    words = log.words if isinstance(log, SparseLog) else log
    words = words.contiguous()
    shape = tuple(x.shape) if x.dim() else (1,)
    t = D.aligned_f64(x.reshape(-1))
    n = t.numel()
    kind = _out_kind(out_dtype)
    D.check_out(out, n, out_dtype, t.device, "out")
    if words.dtype != torch.int64 or words.device != t.device:
        raise ValueError("log words must be an int64 tensor on the input's device")
    y = out if out is not None else torch.empty(n, dtype=out_dtype, device=t.device)
    need = int(_lib.lib().vt_replay_workspace(n))
    ws = workspace if workspace is not None else D.workspace(need, "replay")
    D.check_out(ws, need, torch.uint8, t.device, "workspace")
    D.check_out(flags_out, 6, torch.int64, t.device, "flags_out")
    f = D.Flags(buf=flags_out)
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


@dataclass
class PendingAdaptive:
    """Result of round_and_log_adaptive(check=False): buffers + device tau."""

    y: torch.Tensor
    words: torch.Tensor
    tau: torch.Tensor  # float64[1] on the device
    flags: D.Flags

    def finish(self) -> tuple[torch.Tensor, SparseLog, float]:
        err, cnt = self.flags.read()
        D.raise_fpround(err)
        if cnt[0] > self.words.numel():
            raise LogOverflow(f"sparse log needs {cnt[0]} words, capacity {self.words.numel()}")
        return self.y, SparseLog(self.words[: cnt[0]], cnt[0]), float(self.tau.item())


def round_and_log_adaptive(x: torch.Tensor, b_r: int, budget: int, *, iters: int = 30,
                           out_dtype=torch.float32, global_base: int = 0, out: torch.Tensor | None = None,
                           log_out: torch.Tensor | None = None, check: bool = True, tag: str = "adaptive",
                           tau_out: torch.Tensor | None = None, flags_out: torch.Tensor | None = None,
                           workspace: torch.Tensor | None = None):
    """Per-tensor adaptive threshold + round-and-log, all on the device.

    tau = protocol.search_tau_budget(x, b_r, budget, iters) (bit-identical:
    same selection, same FP64 bisection run by one device thread), then the
    sparse round-and-log at tau.  No host synchronisation unless check=True,
    so a whole model's worth of tensors can be queued or graph-captured.
    tau_out (float64[1]) and flags_out (zeroed int64[6]) let a caller supply
    the per-call result slots, so repeated calls allocate nothing."""
    _check_b(b_r)
    D.require_cuda()
    shape = tuple(x.shape) if x.dim() else (1,)
    t = D.aligned_f64(x.reshape(-1))
    n = t.numel()
    kind = _out_kind(out_dtype)
    D.check_out(out, n, out_dtype, t.device, "out")
    D.check_out(log_out, 0, torch.int64, t.device, "log_out")
    D.check_out(tau_out, 1, torch.float64, t.device, "tau_out")
    D.check_out(flags_out, 6, torch.int64, t.device, "flags_out")
    y = out if out is not None else torch.empty(n, dtype=out_dtype, device=t.device)
    words = log_out if log_out is not None else torch.empty(max(budget + 1, 1), dtype=torch.int64, device=t.device)
    tau = tau_out if tau_out is not None else torch.empty(1, dtype=torch.float64, device=t.device)
    need = int(_lib.lib().vt_round_log_adaptive_workspace(n))
    ws = workspace if workspace is not None else D.workspace(need, tag)
    D.check_out(ws, need, torch.uint8, t.device, "workspace")
    f = D.Flags(buf=flags_out)
    if n:
        _lib.call("vt_round_log_adaptive", D.ptr(t), n, b_r, int(budget), int(iters), kind, D.ptr(y), D.ptr(words),
                  words.numel(), int(global_base), None, None, D.ptr(tau), f.cnt_ptr, f.err_ptr, D.ptr(ws),
                  ws.numel(), D.stream_ptr())
    pending = PendingAdaptive(y.reshape(shape) if out is None else y, words, tau, f)
    return pending.finish() if check else pending


@dataclass
class PendingAdaptiveBatch:
    """Result of round_and_log_adaptive_batch(check=False)."""

    ys: list
    words: list
    taus: torch.Tensor   # float64 [m] on the device
    flags: torch.Tensor  # int64 [m, 4]: error bits, -, log entries, -

    def finish(self) -> list[tuple[torch.Tensor, SparseLog, float]]:
        f = self.flags.cpu().tolist()
        taus = self.taus.cpu().tolist()
        out = []
        for y, w, fl, tau in zip(self.ys, self.words, f, taus):
            D.raise_fpround(int(fl[0]) & 0xFFFFFFFF)
            if fl[2] > w.numel():
                raise LogOverflow(f"sparse log needs {fl[2]} words, capacity {w.numel()}")
            out.append((y, SparseLog(w[: fl[2]], int(fl[2])), float(tau)))
        return out


_BATCH_SIG: dict = {}


def round_and_log_adaptive_batch(xs, b_r: int, budgets, *, iters: int = 30, out_dtype=torch.float32,
                                 global_bases=None, outs=None, log_outs=None, check: bool = True,
                                 tag: str = "adaptive_batch"):
    """``round_and_log_adaptive`` over many independent tensors at once.

    Per tensor the result is identical to ``round_and_log_adaptive(xs[i],
    b_r, budgets[i])`` (same tau bits, log words and rounded output); the
    device work is one fused rounding pass over all tensors plus a fixed
    number of selection / filter launches (``vt_round_log_adaptive_batch``),
    instead of ~12 launches per tensor.  Outputs must not alias the inputs
    (the in-place form stays per tensor).  Returns a list of (y, SparseLog,
    tau), or a PendingAdaptiveBatch with ``check=False``."""
    import ctypes as C

    _check_b(b_r)
    dev = D.require_cuda()
    xs = list(xs)
    m = len(xs)
    budgets = [int(b) for b in budgets]
    if len(budgets) != m:
        raise ValueError("one budget per tensor")
    for name, seq in (("global_bases", global_bases), ("outs", outs), ("log_outs", log_outs)):
        if seq is not None and len(seq) != m:
            raise ValueError(f"{name}: one entry per tensor")
    kind = _out_kind(out_dtype)
    flat = [D.aligned_f64(x.reshape(-1)) for x in xs]
    for i in range(m):
        if outs is not None:
            D.check_out(outs[i], flat[i].numel(), out_dtype, dev, f"outs[{i}]")
        if log_outs is not None:
            D.check_out(log_outs[i], 0, torch.int64, dev, f"log_outs[{i}]")
    ys = list(outs) if outs is not None else [torch.empty(t.numel(), dtype=out_dtype, device=dev) for t in flat]
    words = list(log_outs) if log_outs is not None else [
        torch.empty(max(b + 1, 1), dtype=torch.int64, device=dev) for b in budgets]
    bases = [int(b) for b in global_bases] if global_bases is not None else [0] * m
    taus = torch.empty(max(m, 1), dtype=torch.float64, device=dev)
    flags = torch.zeros((max(m, 1), 4), dtype=torch.int64, device=dev)
    live = [i for i in range(m) if flat[i].numel()]
    if live:
        segs = (_lib.AdaptiveSegment * len(live))()
        for k, i in enumerate(live):
            segs[k] = _lib.AdaptiveSegment(D.ptr(flat[i]), flat[i].numel(), budgets[i], D.ptr(ys[i]),
                                           D.ptr(words[i]), words[i].numel(), bases[i],
                                           taus.data_ptr() + 8 * i, flags.data_ptr() + 32 * i)
        ns = (C.c_int64 * len(live))(*[flat[i].numel() for i in live])
        nbytes = int(_lib.lib().vt_round_log_adaptive_batch_workspace(ns, len(live)))
        ws = D.workspace(nbytes, tag)
        # per-tensor state sits at offsets set by the batch's sizes: a new
        # size signature starts from a zeroed workspace
        sig = (ws.data_ptr(), tuple(ns))
        key = (torch.cuda.current_device(), D.stream_ptr(), tag)
        if _BATCH_SIG.get(key) != sig:
            ws.zero_()
            _BATCH_SIG[key] = sig
        _lib.call("vt_round_log_adaptive_batch", C.cast(segs, C.c_void_p), len(live), b_r, int(iters), kind,
                  D.ptr(ws), ws.numel(), D.stream_ptr())
    for i in range(m):
        if not flat[i].numel():  # empty tensor: nothing to select, tau as the host search
            from .protocol import search_tau_budget
            taus[i].fill_(search_tau_budget(flat[i], b_r, budgets[i], iters))
    pending = PendingAdaptiveBatch(
        [y.reshape(tuple(x.shape) if x.dim() else (1,)) if outs is None else y for x, y in zip(xs, ys)],
        words, taus[:m], flags[:m])
    return pending.finish() if check else pending


class _HostPipe:
    """Double-buffered device staging for host-resident tensors: H2D copies,
    kernels and D2H copies run on three streams so PCIe traffic in both
    directions overlaps the HBM-bound kernels chunk by chunk."""

    def __init__(self, chunk: int, device):
        self.chunk = chunk
        self.dev = device
        self.s_in = torch.cuda.Stream(device)
        self.s_run = torch.cuda.Stream(device)
        self.s_out = torch.cuda.Stream(device)
        self.xbuf = [torch.empty(chunk, dtype=torch.float64, device=device) for _ in range(2)]
        self.ybuf = [torch.empty(chunk, dtype=torch.float32, device=device) for _ in range(2)]
        self.ev_loaded = [torch.cuda.Event() for _ in range(2)]
        self.ev_xfree = [torch.cuda.Event() for _ in range(2)]
        self.ev_done = [torch.cuda.Event() for _ in range(2)]
        self.ev_yfree = [torch.cuda.Event() for _ in range(2)]
        for e in self.ev_xfree + self.ev_yfree:
            e.record(torch.cuda.current_stream(device))

    def _load(self, x_h: torch.Tensor, i: int) -> None:
        n = x_h.numel()
        lo = i * self.chunk
        hi = min(n, lo + self.chunk)
        k = i & 1
        with torch.cuda.stream(self.s_in):
            self.s_in.wait_event(self.ev_xfree[k])
            self.xbuf[k][: hi - lo].copy_(x_h[lo:hi], non_blocking=True)
            self.ev_loaded[k].record(self.s_in)

    def preload(self, x_h: torch.Tensor) -> int:
        """Start the H2D copies of the first two chunks now (both staging
        buffers), e.g. while the host waits on earlier work; run() then skips
        them.  Returns the number of chunks preloaded."""
        k = min(2, (x_h.numel() + self.chunk - 1) // self.chunk)
        for i in range(k):
            self._load(x_h, i)
        return k

    def run(self, x_h: torch.Tensor, y_h: torch.Tensor, kernel, preloaded: int = 0) -> None:
        n = x_h.numel()
        for i, lo in enumerate(range(0, n, self.chunk)):
            hi = min(n, lo + self.chunk)
            k = i & 1
            xb = self.xbuf[k][: hi - lo]
            yb = self.ybuf[k][: hi - lo]
            if i >= preloaded:
                self._load(x_h, i)
            with torch.cuda.stream(self.s_run):
                self.s_run.wait_event(self.ev_loaded[k])
                self.s_run.wait_event(self.ev_yfree[k])
                kernel(xb, yb, lo)
                self.ev_xfree[k].record(self.s_run)
                self.ev_done[k].record(self.s_run)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(self.ev_done[k])
                y_h[lo:hi].copy_(yb, non_blocking=True)
                self.ev_yfree[k].record(self.s_out)
        torch.cuda.current_stream(self.dev).wait_stream(self.s_out)
        torch.cuda.current_stream(self.dev).wait_stream(self.s_run)


_PIPES: dict = {}


def round_and_log_replay_host(xt_h: torch.Tensor, xa_h: torch.Tensor, b_r: int, tau: float,
                              yt_h: torch.Tensor, ya_h: torch.Tensor, log_h: torch.Tensor,
                              global_base: int = 0, chunk: int = 1 << 22) -> tuple[int, int, int]:
    """End-to-end trainer + auditor step from pinned host memory.

    Trainer: chunked H2D of the FP64 tensor, fused round-and-log (log chunks
    appended on the device through cursor chaining, global indices), D2H of
    the FP32 output, then D2H of the sparse log.  Auditor: chunked H2D of its
    FP64 tensor, fused replay against the device log, D2H of the FP32 output.
    Returns (log entries, corrections, log bytes copied to the host).
    """
    _check_b(b_r)
    dev = D.require_cuda()
    n = xt_h.numel()
    # one pipeline per side: the auditor's first H2D chunks stream into their
    # own staging buffers while the host waits for the trainer's log length
    pipes = []
    for side in ("trainer", "auditor"):
        key = (dev.index, D.stream_ptr(), chunk, side)  # per calling stream: reentrant like the operators
        if key not in _PIPES:
            _PIPES[key] = _HostPipe(chunk, dev)
        pipes.append(_PIPES[key])
    pipe, pipe_a = pipes
    # the device log holds as many words as the caller's host log can take
    words = D.workspace(8 * max(min(int(log_h.numel()), n), 1024), "host_log").view(torch.int64)
    n_chunks = (n + chunk - 1) // chunk
    cursors = torch.zeros(n_chunks + 1, dtype=torch.int64, device=dev)
    ws_rl = [D.workspace(int(_lib.lib().vt_round_log_workspace(chunk)), f"hp_rl{k}") for k in range(2)]
    fl = D.Flags()
    fl_a = D.Flags()
    cap = words.numel()

    def rl(xb, yb, lo):
        i = lo // chunk
        ws = ws_rl[i & 1]
        _lib.call("vt_round_log", D.ptr(xb), xb.numel(), b_r, float(tau), _lib.OUT_F32, D.ptr(yb),
                  D.ptr(words), cap, int(global_base + lo), cursors.data_ptr() + 8 * i,
                  cursors.data_ptr() + 8 * (i + 1), None, None, 0, None, fl.cnt_ptr, fl.err_ptr,
                  D.ptr(ws), ws.numel(), D.stream_ptr())

    torch.cuda.current_stream(dev).synchronize()
    pipe.run(xt_h, yt_h, rl)
    pre = pipe_a.preload(xa_h)  # PCIe stays busy across the host wait below
    err, cnt = fl.read()  # syncs the trainer's streams only: the auditor needs the log length
    D.raise_fpround(err)
    count = cnt[0]
    if count > cap or count > log_h.numel():
        raise LogOverflow(f"sparse log needs {count} words")
    log_h[:count].copy_(words[:count], non_blocking=True)
    ws_rp = [D.workspace(int(_lib.lib().vt_replay_workspace(chunk)), f"hp_rp{k}") for k in range(2)]

    def rp(xb, yb, lo):
        i = lo // chunk
        ws = ws_rp[i & 1]
        _lib.call("vt_replay", D.ptr(xb), xb.numel(), b_r, _lib.LOG_SPARSE, D.ptr(words), count,
                  int(global_base + lo), _lib.OUT_F32, D.ptr(yb), fl_a.cnt_ptr, fl_a.err_ptr,
                  D.ptr(ws), ws.numel(), D.stream_ptr())

    pipe_a.run(xa_h, ya_h, rp, preloaded=pre)
    err_a, cnt_a = fl_a.read()
    if err_a & _lib.ERR_BAD_SPARSE:
        raise SparseLogError("sparse log is not strictly ascending")
    D.raise_fpround(err_a)
    return count, cnt_a[0], 8 * count


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
