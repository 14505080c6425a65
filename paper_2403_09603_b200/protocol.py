"""Trainer / auditor channels and threshold search on the B200.

Drop-in for the hot-path parts of ``vtrain.protocol``
(pkg/src/vtrain/protocol.py):

* ``GpuTrainerChannel`` / ``GpuAuditorChannel`` / ``GpuPlainChannel``
  satisfy the channel duck type ``process(values, tau) -> (ndarray,
  directed, corrections)`` consumed by ``protocol._run`` (protocol.py:268,
  278, 283), replacing ``_TrainerChannel`` / ``_AuditorChannel`` /
  ``_PlainChannel`` (protocol.py:191-226) with single fused kernels.
* ``search_tau`` keeps ``protocol.search_tau`` (protocol.py:494-506)
  bit for bit: the all(p >= tau) predicate is a device min-reduction,
  the FP64 bisection runs on the host on that one scalar.
* ``search_tau_budget`` is the north-star per-tensor budget search
  (SURVEY.md Appendix A.4): largest band (= smallest reference-form tau in
  ``tau_bounds``) whose log stays within ``budget`` entries, via the device
  radix select of the (budget+1)-th largest normalized distance.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from . import _lib
from .fpround import _check_b, rnd_array, tau_bounds
from .roundlog import LogExhaustedError, LogReader, LogWriter


class AuditFailure(RuntimeError):
    """The audit could not be completed against the provided artifacts."""


def _host_like(values, y: torch.Tensor):
    return y.cpu().numpy() if not (isinstance(values, torch.Tensor) and values.is_cuda) else y


class GpuTrainerChannel:
    """Classify, record, round -- one fused kernel per tensor."""

    def __init__(self, writer, b_r: int):
        self.writer = writer
        self.b_r = b_r

    def process(self, values, tau: float):
        if isinstance(self.writer, LogWriter):
            if not isinstance(values, torch.Tensor):  # the reference loop's NumPy arrays: staged path
                y, directed = self.writer.write_values_host(values, tau)
                return y, int(directed), 0
            y, directed = self.writer.write_values(values, tau)
            return _host_like(values, y), int(directed), 0
        # foreign writer with the reference interface: hand it the codes
        t, _, shape = D.to_device_f64(values)
        y = torch.empty_like(t)
        codes = torch.empty(t.numel(), dtype=torch.uint8, device=t.device)
        f = D.Flags()
        if t.numel():
            _lib.call("vt_round_log", D.ptr(t), t.numel(), self.b_r, float(tau), _lib.OUT_F64, D.ptr(y),
                      None, 0, 0, None, None, D.ptr(codes), None, 0, None, f.cnt_ptr, f.err_ptr, None, 0,
                      D.stream_ptr())
        err, cnt = f.read()
        D.raise_fpround(err)
        self.writer.write_array(codes.cpu().numpy())
        return _host_like(values, y.reshape(shape)), int(cnt[0]), 0


class GpuAuditorChannel:
    """Read, replay -- one fused kernel per tensor."""

    def __init__(self, reader, b_r: int):
        self.reader = reader
        self.b_r = b_r
        self._stage = None

    def _process_host(self, values, tau: float):
        """NumPy input with a device-resident .vtrl payload: one H2D copy of
        [x | zeroed flags], the fused packed replay, one D2H copy of
        [flags | y], one host wait; small arrays zero-copy (the kernel reads
        x from and writes y to the pinned buffer, only the flags come back)."""
        a = np.asarray(values, dtype=np.float64)
        shape = a.shape if a.shape else (1,)
        n = a.size
        payload, pos = self.reader.take_device(n)
        if n == 0:
            return np.zeros(shape, dtype=np.float64), 0, 0
        st = self._stage
        if st is None:
            st = self._stage = D.HostStage()
        fo, (oy,), end = st.layout(8 * n, [8 * n])
        st.ensure(end)
        np.copyto(st.hview(0, n, np.float64), a.reshape(-1))
        ws = D.workspace(int(_lib.lib().vt_replay_workspace(n)), "replay_packed")
        if n <= st.ZERO_COPY_MAX:  # zero-copy: x and y in the pinned buffer, flags on the device
            st.zero_dev(fo, 64)
            _lib.call("vt_replay", st.hptr(0), n, self.b_r, _lib.LOG_PACKED, D.ptr(payload),
                      self.reader.payload_nbytes, pos, _lib.OUT_F64, st.hptr(oy), st.dptr(fo + 16), st.dptr(fo),
                      D.ptr(ws), ws.numel(), D.stream_ptr())
            st.d2h_wait(fo, fo + 64)
        else:
            st.hview(fo, 32, np.int64)[:] = 0
            st.h2d(fo + 256)
            _lib.call("vt_replay", st.dptr(0), n, self.b_r, _lib.LOG_PACKED, D.ptr(payload),
                      self.reader.payload_nbytes, pos, _lib.OUT_F64, st.dptr(oy), st.dptr(fo + 16), st.dptr(fo),
                      D.ptr(ws), ws.numel(), D.stream_ptr())
            st.d2h_wait(fo, oy + 8 * n)
        fl = st.hview(fo, 6, np.int64)
        err = int(fl[0]) & 0xFFFFFFFF
        if err & _lib.ERR_BAD_LOG_BYTE:
            from .roundlog import LogFormatError
            raise LogFormatError("corrupt log byte")
        D.raise_fpround(err)
        return st.hview(oy, n, np.float64).copy().reshape(shape), 0, int(fl[2])

    def process(self, values, tau: float):
        if isinstance(self.reader, LogReader) and not isinstance(values, torch.Tensor):
            return self._process_host(values, tau)
        t, _, shape = D.to_device_f64(values)
        n = t.numel()
        y = torch.empty_like(t)
        f = D.Flags()
        if isinstance(self.reader, LogReader):
            payload, pos = self.reader.take_device(n)
            if n:
                ws = D.workspace(int(_lib.lib().vt_replay_workspace(n)), "replay_packed")
                _lib.call("vt_replay", D.ptr(t), n, self.b_r, _lib.LOG_PACKED, D.ptr(payload),
                          self.reader.payload_nbytes, pos, _lib.OUT_F64, D.ptr(y), f.cnt_ptr, f.err_ptr,
                          D.ptr(ws), ws.numel(), D.stream_ptr())
        else:
            codes = np.ascontiguousarray(self.reader.read_array(n), dtype=np.uint8)
            c = torch.from_numpy(codes).to(t.device)
            if n:
                _lib.call("vt_replay", D.ptr(t), n, self.b_r, _lib.LOG_CODES, D.ptr(c), n, 0,
                          _lib.OUT_F64, D.ptr(y), f.cnt_ptr, f.err_ptr, None, 0, D.stream_ptr())
        err, cnt = f.read()
        if err & _lib.ERR_BAD_LOG_BYTE:
            from .roundlog import LogFormatError
            raise LogFormatError("corrupt log byte")
        if err & _lib.ERR_BAD_CODE:
            raise ValueError("invalid direction code")
        D.raise_fpround(err)
        return _host_like(values, y.reshape(shape)), 0, int(cnt[0])


class GpuPlainChannel:
    """Round only; the negative control (protocol.py:219-226)."""

    def __init__(self, b_r: int):
        self.b_r = b_r

    def process(self, values, tau: float):
        return rnd_array(values, self.b_r), 0, 0


def _device_min(samples) -> tuple[float, bool]:
    if isinstance(samples, torch.Tensor) and samples.is_cuda:
        s = samples.reshape(-1).to(torch.float64).contiguous()
    else:
        s = torch.as_tensor(np.asarray(samples, dtype=np.float64).reshape(-1)).to(D.require_cuda())
    out = torch.empty(1, dtype=torch.float64, device=s.device)
    f = D.Flags()
    _lib.call("vt_min_f64", D.ptr(s), s.numel(), D.ptr(out), f.err_ptr, D.stream_ptr())
    nan = bool(f.read()[0] & 1)
    return float(out.item()), nan


def search_tau(samples, b_r: int, iters: int) -> float:
    """Largest threshold no recorded straddle undercuts (protocol.py:494-506)."""
    lower, upper = tau_bounds(b_r)
    if len(samples) == 0:
        return upper
    m, has_nan = _device_min(samples)
    tau = lower
    for _ in range(iters):
        tau = (lower + upper) / 2.0
        if (not has_nan) and m >= tau:
            lower = tau
        else:
            upper = tau
    return tau


def straddle_min(y1, y2, b_r: int) -> tuple[float, int, bool]:
    """(min sample, sample count, any NaN) of the straddle samples that
    collect_divergence_samples (protocol.py:483-490) draws from two profiles'
    outputs of the same layer on the same inputs."""
    _check_b(b_r)
    t1, _, s1 = D.to_device_f64(y1)
    t2, _, s2 = D.to_device_f64(y2)
    if s1 != s2:
        raise ValueError(f"output shapes differ: {s1} vs {s2}")
    out = torch.empty(2, dtype=torch.float64, device=t1.device)
    f = D.Flags()
    _lib.call("vt_straddle_min", D.ptr(t1), D.ptr(t2), t1.numel(), b_r, D.ptr(out), out.data_ptr() + 8,
              f.cnt_ptr, f.err_ptr, D.stream_ptr())
    err, cnt = f.read()
    D.raise_fpround(err)
    m, c = out.tolist()
    return m, int(np.array([c], dtype=np.float64).view(np.int64)[0]), bool(cnt[0] & 1)


def threshold_from_outputs(y1, y2, b_r: int, iters: int) -> float:
    """protocol.threshold_search (protocol.py:509-516) once the layer has been
    run under both profiles: search_tau over the straddle samples, with the
    all(p >= tau) predicate evaluated as min(samples) >= tau on the device."""
    if iters < 1:
        raise ValueError("n_samples and iters must be >= 1")
    lower, upper = tau_bounds(b_r)
    m, count, has_nan = straddle_min(y1, y2, b_r)
    if count == 0:
        return upper
    tau = lower
    for _ in range(iters):
        tau = (lower + upper) / 2.0
        if (not has_nan) and m >= tau:
            lower = tau
        else:
            upper = tau
    return tau


def kth_largest_distance(x, b_r: int, rank: int) -> float:
    """(rank+1)-th largest p = |x - rnd(x)| / max(scale, 2^-126), exactly."""
    _check_b(b_r)
    t, _, _ = D.to_device_f64(x)
    n = t.numel()
    if rank >= n:
        return 0.0
    ws = D.workspace(int(_lib.lib().vt_tau_workspace(n)), "tau")
    key = torch.zeros(1, dtype=torch.int64, device=t.device)
    f = D.Flags()
    _lib.call("vt_tau_kth_key", D.ptr(t), n, b_r, int(rank), D.ptr(key), f.err_ptr, D.ptr(ws), ws.numel(),
              D.stream_ptr())
    err = f.read()[0]
    D.raise_fpround(err)
    return float(np.array([key.item()], dtype=np.int64).view(np.float64)[0])


def _budget_select(x, b_r: int, budget: int, iters: int) -> tuple[float, float]:
    """(tau, v'): ``vt_tau_budget`` -- one streaming read of x for the
    candidates above a threshold below the expected tau, then the exact
    selection of the (budget+1)-th largest p among them and the FP64
    bisection on the device (exact multi-pass fallback in the same launch)."""
    _check_b(b_r)
    lower, upper = tau_bounds(b_r)
    t, _, _ = D.to_device_f64(x)
    n = t.numel()
    if n == 0 or budget >= n:  # every tau is feasible: v' = tau_lo
        return _bisect(lower, lower, upper, iters), lower
    ws = D.workspace(int(_lib.lib().vt_tau_budget_workspace(n)), "tau_budget")
    out = torch.empty(2, dtype=torch.float64, device=t.device)  # [tau, key bits]
    f = D.Flags()
    _lib.call("vt_tau_budget", D.ptr(t), n, b_r, int(budget), int(iters), D.ptr(out), out.data_ptr() + 8,
              f.err_ptr, D.ptr(ws), ws.numel(), D.stream_ptr())
    tau, key = out.tolist()
    D.raise_fpround(f.read()[0])
    return tau, key


def _bisect(v: float, lower: float, upper: float, iters: int) -> float:
    for _ in range(iters):
        tau = (lower + upper) / 2.0
        if v <= tau:
            upper = tau
        else:
            lower = tau
    return upper


def budget_key(x, b_r: int, budget: int) -> float:
    """v' = the (budget+1)-th largest p, clamped for a bisection strictly inside
    tau_bounds(b_r): tau_lo if v <= tau_lo, +inf if v > tau_hi, else v."""
    return _budget_select(x, b_r, int(budget), 30)[1]


def search_tau_budget(x, b_r: int, budget: int, iters: int = 30) -> float:
    """Per-tensor adaptive threshold: the search_tau skeleton with predicate
    count(p > tau) <= budget, feasible -> upper = tau, returns ``upper``
    (bisection on the device, bit-identical to the host FP64 loop)."""
    return _budget_select(x, b_r, int(budget), int(iters))[0]


__all__ = ["AuditFailure", "GpuAuditorChannel", "GpuPlainChannel", "GpuTrainerChannel",
           "LogExhaustedError", "budget_key", "kth_largest_distance", "search_tau", "search_tau_budget"]
