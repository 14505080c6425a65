"""Device plumbing: tensors in and out of the C ABI, workspaces, error bits.

PyTorch is used only for device memory, streams and copies; all compute is
in ``libvtrain_b200.so``.  Host (NumPy / list) inputs are the drop-in
parity mode of the reference API (copied to HBM, results copied back); CUDA
tensors are zero-copy when contiguous and 32-byte aligned.
"""

from __future__ import annotations

import threading
import warnings

import numpy as np
import torch

from . import _lib

_WS: dict[tuple, torch.Tensor] = {}
_RETIRED: list[torch.Tensor] = []
_WS_LOCK = threading.Lock()
_WARNED: set = set()


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2403_09603_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    _lib.lib()
    return torch.device("cuda", torch.cuda.current_device())


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_ptr(device=None) -> int:
    """The current CUDA stream of ``device`` (default: the current device) as
    a raw cudaStream_t.  The direct C accessor skips torch.cuda.current_stream's
    Python device-index handling (~7 us per call, which the reference-API
    channels on small tensors pay on every call)."""
    if _RAW_STREAM is not None and device is None:
        return int(_RAW_STREAM(torch.cuda.current_device()))
    return int(torch.cuda.current_stream(device).cuda_stream)


def sync_stream(stream: int | None = None) -> None:
    """Wait for the current (or the given raw) stream on the host."""
    _lib.call("vt_stream_synchronize", stream_ptr() if stream is None else stream)


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
    """Scratch buffer per (device, current stream, tag), grown on demand.

    Keyed by stream so the public operators are reentrant across streams and
    host threads: the ticketed kernels keep a ticket counter,
    an epoch and epoch-tagged look-back words in their workspace, and two
    grids drawing from one counter at once would corrupt each other.  Calls
    on ONE stream may share a workspace because the stream serialises them.
    Zero-filled once at allocation (the epoch scheme needs a zero start).
    A grown-out-of buffer is retired, not freed: a CUDA graph captured with
    the old pointer (or queued work) may still use it.  Growth is by at
    least 1.5x, so a run of ever larger calls retires O(log) buffers whose
    total stays below twice the live one."""
    key = (torch.cuda.current_device(), stream_ptr(), tag)
    with _WS_LOCK:
        ws = _WS.get(key)
        if ws is None or ws.numel() < nbytes:
            if ws is not None:
                _RETIRED.append(ws)
            if torch.cuda.is_current_stream_capturing() and key not in _WARNED:
                _WARNED.add(key)
                warnings.warn(f"paper_2403_09603_b200: workspace '{tag}' first allocated inside a CUDA graph capture; "
                              "its zero-fill becomes part of the graph.  Warm up on the capture stream "
                              "(torch.cuda.graph(g, stream=s)) or pass workspace=.", stacklevel=3)
            grow = ws.numel() * 3 // 2 if ws is not None else 0
            ws = torch.zeros(max(nbytes, 1 << 20, grow), dtype=torch.uint8, device="cuda")
            _WS[key] = ws
        return ws


def check_out(t: torch.Tensor | None, n: int, dtype: torch.dtype, device: torch.device, name: str = "out") -> None:
    """Caller-supplied output buffers go to the C ABI as raw pointers: require
    the element count, dtype, contiguity and device before the call."""
    if t is None:
        return
    if not isinstance(t, torch.Tensor):
        raise ValueError(f"{name} must be a torch.Tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} has dtype {t.dtype}, expected {dtype}")
    if t.numel() < n:
        raise ValueError(f"{name} holds {t.numel()} elements, needs {n}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")


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


class HostStage:
    """Pinned host <-> device staging for host-array calls of one channel
    (protocol._run hands the channels NumPy arrays of a few thousand
    elements): the call's input and zeroed flag words go over in ONE H2D copy,
    every output (flags, side outputs, the FP64 result) comes back in ONE D2H
    copy, and the host waits once -- instead of a pageable copy, a flag read
    and a result read, each synchronising.

    Layout (host and device alike, 256-byte aligned regions):
        [ x: in_bytes | flags: 256 | out regions ... ]
    H2D covers [0, flags_end); D2H covers [flags_off, end).  One stage per
    channel object; calls on it are sequential (the channel is).

    Zero-copy form for small calls (``ZERO_COPY_MAX`` elements and below):
    the kernel reads x from and writes its outputs to the pinned host buffer
    directly (pinned memory is device-addressable under UVA, ``hptr``); only
    the flag words, which the kernel accumulates with atomics, live on the
    device -- zeroed before the call and read back with one 64-byte copy."""

    ZERO_COPY_MAX = (1 << 18) - 1  # below the TMA-pipelined kernels' size threshold

    def __init__(self):
        self.cap = 0
        self.host = self.dev = None

    @staticmethod
    def _al(v: int) -> int:
        return (v + 255) & ~255

    def layout(self, in_bytes: int, out_sizes: list[int]) -> tuple[int, list[int], int]:
        flags_off = self._al(in_bytes)
        offs, o = [], flags_off + 256
        for sz in out_sizes:
            offs.append(o)
            o = self._al(o + sz)
        return flags_off, offs, o

    def ensure(self, nbytes: int) -> None:
        if nbytes > self.cap:
            cap = max(nbytes, 2 * self.cap, 1 << 16)
            self.host = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
            self.dev = torch.empty(cap, dtype=torch.uint8, device=require_cuda())
            self.host_np = self.host.numpy()
            self.cap = cap

    def h2d(self, end: int) -> None:
        self.dev[:end].copy_(self.host[:end], non_blocking=True)

    def hptr(self, off: int) -> int:
        """Device-usable address of the pinned host buffer at ``off`` (UVA)."""
        return self.host.data_ptr() + off

    def zero_dev(self, off: int, nbytes: int) -> None:
        self.dev[off:off + nbytes].zero_()

    def d2h_wait(self, lo: int, hi: int) -> None:
        self.host[lo:hi].copy_(self.dev[lo:hi], non_blocking=True)
        sync_stream()

    def hview(self, off: int, n: int, dtype) -> np.ndarray:
        return self.host_np[off:off + n * np.dtype(dtype).itemsize].view(dtype)

    def dptr(self, off: int) -> int:
        return self.dev.data_ptr() + off
