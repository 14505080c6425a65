"""Reduced-precision grid arithmetic on the B200 -- drop-in for ``vtrain.fpround``.

Same names, signatures, argument meaning and exception text as the
reference (pkg/src/vtrain/fpround.py); every array operator runs in
``libvtrain_b200.so``:

=====================  ===========================  =========================
function               reference                    kernel
=====================  ===========================  =========================
rnd_array / rnd        fpround.py:127-140           round_log_kernel (no log)
direction_array        fpround.py:164-177           round_log_kernel (codes)
rev_array / rev        fpround.py:227-252           replay_kernel (codes)
grid_neighbors_array   fpround.py:185-224           neighbors_kernel
exponent_scale_array   fpround.py:149-161           exponent_scale_kernel
is_on_grid             fpround.py:255-264           on_grid_kernel
=====================  ===========================  =========================

NumPy / list inputs return NumPy arrays (the reference's contract: FP64,
input shape, 0-d -> (1,)); CUDA tensors return CUDA tensors on the current
stream.  Scalar helpers (``tau_bounds``, ``grid_max``, ``epsilon``,
``RoundingParams``) are host arithmetic, as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _lib

DOWN = 0
IGNORE = 1
UP = 2
MIN_B = 10
MAX_B = 32
SCALE_FLOOR = 2.0 ** -126


def _check_b(b_r) -> None:
    if not isinstance(b_r, (int, np.integer)) or not MIN_B <= b_r <= MAX_B:
        raise ValueError(f"b_r must be an integer in [{MIN_B}, {MAX_B}], got {b_r!r}")


def tau_bounds(b_r: int) -> tuple[float, float]:
    """Valid [lower, upper] relative threshold (fpround.py:49-52)."""
    _check_b(b_r)
    return 2.0 ** -25, 2.0 ** (8 - b_r)


def grid_max(b_r: int) -> float:
    """Largest grid magnitude (fpround.py:55-59)."""
    _check_b(b_r)
    return (2.0 - 2.0 ** (9 - b_r)) * 2.0 ** 127


def epsilon(b_r: int, exponent_scale: float) -> float:
    """Grid spacing at an exponent scale (fpround.py:143-146)."""
    _check_b(b_r)
    return exponent_scale * 2.0 ** (9 - b_r)


@dataclass(frozen=True)
class RoundingParams:
    """Rounding amount, threshold and working precision (fpround.py:62-84)."""

    b_r: int
    tau: float
    b_tr: int = 64

    def __post_init__(self) -> None:
        _check_b(self.b_r)
        if self.b_tr != 64:
            raise ValueError("training precision must be 64")
        if self.tau != 0.0:
            lo, hi = tau_bounds(self.b_r)
            if not lo <= self.tau <= hi:
                raise ValueError(f"tau {self.tau!r} outside [{lo!r}, {hi!r}] for b_r={self.b_r}")


def _round_call(t: torch.Tensor, b_r: int, tau: float, out_kind: int, out: torch.Tensor | None,
                codes: torch.Tensor | None) -> D.Flags:
    f = D.Flags()
    _lib.call("vt_round_log", D.ptr(t), t.numel(), b_r, float(tau), out_kind, D.ptr(out),
              None, 0, 0, None, None, D.ptr(codes), None, 0, None,
              f.cnt_ptr, f.err_ptr, None, 0, D.stream_ptr())
    return f


def rnd_array(x, b_r: int):
    """Round each element onto the b_r grid, nearest, ties to even."""
    _check_b(b_r)
    t, host, shape = D.to_device_f64(x)
    out = torch.empty_like(t)
    if t.numel():
        err, _ = _round_call(t, b_r, 0.0, _lib.OUT_F64, out, None).read()
        D.raise_fpround(err)
    return D.back(out, host, shape)


def rnd(x: float, b_r: int) -> float:
    return float(rnd_array(x, b_r)[0])


def exponent_scale_array(x):
    """2^E per element with 1 <= |x|/2^E < 2; zero maps to 2^-126."""
    t, host, shape = D.to_device_f64(x)
    out = torch.empty_like(t)
    if t.numel():
        f = D.Flags()
        _lib.call("vt_exponent_scale", D.ptr(t), t.numel(), D.ptr(out), f.err_ptr, D.stream_ptr())
        D.raise_fpround(f.read()[0])
    return D.back(out, host, shape)


def exponent_scale(x: float) -> float:
    return float(exponent_scale_array(x)[0])


def direction_array(x, b_r: int, tau: float):
    """Ternary code per element: 2 up, 0 down, 1 within tau of the grid."""
    _check_b(b_r)
    t, host, shape = D.to_device_f64(x)
    codes = torch.empty(t.numel(), dtype=torch.uint8, device=t.device)
    if t.numel():
        err, _ = _round_call(t, b_r, float(tau), _lib.OUT_NONE, None, codes).read()
        D.raise_fpround(err)
    return D.back(codes, host, shape)


def direction(x: float, p: RoundingParams) -> int:
    return int(direction_array(x, p.b_r, p.tau)[0])


def grid_neighbors_array(x, b_r: int):
    """Largest grid value <= x and smallest grid value >= x."""
    _check_b(b_r)
    t, host, shape = D.to_device_f64(x)
    lo = torch.empty_like(t)
    hi = torch.empty_like(t)
    if t.numel():
        f = D.Flags()
        _lib.call("vt_grid_neighbors", D.ptr(t), t.numel(), b_r, D.ptr(lo), D.ptr(hi), f.err_ptr,
                  D.stream_ptr())
        D.raise_fpround(f.read()[0])
    return D.back(lo, host, shape), D.back(hi, host, shape)


def grid_neighbors(x: float, b_r: int) -> tuple[float, float]:
    lo, hi = grid_neighbors_array(x, b_r)
    return float(lo[0]), float(hi[0])


def _codes_u8(codes, n_shape: tuple, dev) -> torch.Tensor:
    """Validated uint8 device codes (fpround.py:235-239 order: shape, then range)."""
    if isinstance(codes, torch.Tensor) and codes.is_cuda:
        c = codes if codes.dim() else codes.reshape(1)
        if tuple(c.shape) != n_shape:
            raise ValueError(f"codes shape {tuple(c.shape)} does not match values shape {n_shape}")
        if c.dtype != torch.uint8:
            if c.numel() and bool(((c < DOWN) | (c > UP)).any()):
                raise ValueError("invalid direction code")
            c = c.to(torch.uint8)
        return c.contiguous().reshape(-1)
    a = np.atleast_1d(np.asarray(codes.cpu().numpy() if isinstance(codes, torch.Tensor) else codes))
    if a.shape != n_shape:
        raise ValueError(f"codes shape {a.shape} does not match values shape {n_shape}")
    t = torch.from_numpy(np.ascontiguousarray(a).reshape(-1)).to(dev)
    if t.dtype != torch.uint8:
        if t.numel() and bool(((t < DOWN) | (t > UP)).any()):
            raise ValueError("invalid direction code")
        t = t.to(torch.uint8)
    return t


def rev_array(x, b_r: int, codes):
    """Replay rounding with recorded codes."""
    t, host, shape = D.to_device_f64(x)
    c = _codes_u8(codes, shape, t.device)
    if not (isinstance(b_r, (int, np.integer)) and MIN_B <= b_r <= MAX_B):
        if c.numel() and bool((c > UP).any()):
            raise ValueError("invalid direction code")
        _check_b(b_r)
    out = torch.empty_like(t)
    if t.numel():
        f = D.Flags()
        _lib.call("vt_replay", D.ptr(t), t.numel(), b_r, _lib.LOG_CODES, D.ptr(c), c.numel(), 0,
                  _lib.OUT_F64, D.ptr(out), f.cnt_ptr, f.err_ptr, None, 0, D.stream_ptr())
        err, _ = f.read()
        if err & _lib.ERR_BAD_CODE:
            raise ValueError("invalid direction code")
        D.raise_fpround(err)
    return D.back(out, host, shape)


def rev(x: float, b_r: int, c: int) -> float:
    return float(rev_array(x, b_r, np.asarray([c]))[0])


def is_on_grid(x, b_r: int):
    """Finite, exactly FP32-representable, low 32-b_r bits clear."""
    _check_b(b_r)
    t, host, shape = D.to_device_f64(x)
    out = torch.empty(t.numel(), dtype=torch.uint8, device=t.device)
    if t.numel():
        _lib.call("vt_is_on_grid", D.ptr(t), t.numel(), b_r, D.ptr(out), D.stream_ptr())
    res = D.back(out.to(torch.bool), host, shape)
    return res
