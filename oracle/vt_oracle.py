"""CPU oracle for the vtrain hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker the GPU path is compared against.  Only
``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import it.  The product
package (``paper_2403_09603_b200``) never imports, links or executes
anything under ``oracle/``.

It is a NumPy restatement of the reference algorithms (reference =
``vtrain`` 0.1.0 under ``/root/reference/pkg/src/vtrain``); every function
names the reference lines it follows.  It is *pinned* against outputs of
the reference itself: ``tests/golden/make_golden.py`` imports the real
reference in the build container and freezes its outputs as fixtures, and
``tests/test_oracle_golden.py`` checks this module against them bit for bit
(bit patterns, so the sign of zero is pinned too).

SHA-256 comes from ``hashlib`` (OpenSSL 3.0.x), which is exactly the
third-party dependency the reference calls (``merkle.py:24-25``); FIPS
180-4 known-answer vectors pin it in the tests.

North-star forms with no reference symbol (sparse log, budget tau search,
4 KiB-chunk Merkle) are restated *only* in terms of the functions above
(SURVEY.md Appendix A.2/A.4/A.5), so their parity is pinned by
construction.
"""

from __future__ import annotations

import hashlib
import zlib

import numpy as np

DOWN, IGNORE, UP = 0, 1, 2
MIN_B, MAX_B = 10, 32
SCALE_FLOOR = 2.0 ** -126
_SIGN = np.uint64(1 << 63)
_MAG = np.uint64((1 << 63) - 1)
_NORMAL_MIN_BITS = np.uint64(0x3810000000000000)  # bits of 2^-126


# --------------------------------------------------------------------------
# grid arithmetic  (reference: pkg/src/vtrain/fpround.py)
# --------------------------------------------------------------------------

def check_b(b_r) -> None:
    """fpround.py:44-46 -- same predicate and message."""
    if not isinstance(b_r, (int, np.integer)) or not MIN_B <= b_r <= MAX_B:
        raise ValueError(f"b_r must be an integer in [{MIN_B}, {MAX_B}], got {b_r!r}")


def tau_bounds(b_r: int) -> tuple[float, float]:
    """fpround.py:49-52."""
    check_b(b_r)
    return 2.0 ** -25, 2.0 ** (8 - b_r)


def grid_max(b_r: int) -> float:
    """fpround.py:55-59: (2 - 2^-(b_r-9)) * 2^127."""
    check_b(b_r)
    return (2.0 - 2.0 ** (9 - b_r)) * 2.0 ** 127


def epsilon(b_r: int, scale: float) -> float:
    """fpround.py:143-146."""
    check_b(b_r)
    return scale * 2.0 ** (9 - b_r)


def _as_f64(x) -> np.ndarray:
    return np.atleast_1d(np.asarray(x, dtype=np.float64))


def _finite_or_raise(a: np.ndarray) -> None:
    """fpround.py:87-89."""
    if not np.isfinite(a).all():
        raise ValueError("non-finite value")


def _shape_back(res: np.ndarray, x) -> np.ndarray:
    shp = np.shape(x)
    return res.reshape(shp) if shp else res


def _split(a: np.ndarray, b_r: int):
    """Bit fields shared by rnd / neighbours (fpround.py:92-124, 185-204)."""
    bits = a.view(np.uint64)
    mag = bits & _MAG
    sign = bits & _SIGN
    drop = np.uint64(52 - (b_r - 9))
    base = mag >> drop
    low = mag & ((np.uint64(1) << drop) - np.uint64(1))
    return bits, mag, sign, drop, base, low


def _tiny_scale(b_r: int) -> tuple[float, float]:
    """Absolute grid step below 2^-126: 2^q with q = (32-b_r)-149 (fpround.py:119-122)."""
    q = (32 - b_r) - 149
    return 2.0 ** -q, 2.0 ** q


def _rnd_core(a: np.ndarray, b_r: int) -> np.ndarray:
    """RNE onto the b_r grid without checks (fpround.py:99-124)."""
    _, mag, sign, drop, base, low = _split(a, b_r)
    half = np.uint64(1) << (drop - np.uint64(1))
    inc = (low > half) | ((low == half) & ((base & np.uint64(1)) != 0))
    normal = (sign | ((base + inc.astype(np.uint64)) << drop)).view(np.float64)
    up_s, dn_s = _tiny_scale(b_r)
    small = np.where(mag >= _NORMAL_MIN_BITS, 0.0, a)
    tiny = np.rint(small * up_s) * dn_s
    return np.where(mag >= _NORMAL_MIN_BITS, normal, tiny)


def rnd_array(x, b_r: int) -> np.ndarray:
    """fpround.py:127-135: check b, finite, round, range-check the result."""
    check_b(b_r)
    a = _as_f64(x).copy()
    _finite_or_raise(a)
    r = _rnd_core(a, b_r)
    if (np.abs(r) > grid_max(b_r)).any():
        raise ValueError("out of representable range")
    return _shape_back(r, x)


def exponent_scale_array(x) -> np.ndarray:
    """fpround.py:149-156: 2^E with 1 <= |x|/2^E < 2; zero -> 2^-126."""
    a = _as_f64(x)
    _finite_or_raise(a)
    _, e = np.frexp(a)
    s = np.ldexp(1.0, e - 1)
    return _shape_back(np.where(a == 0.0, SCALE_FLOOR, s), x)


def direction_array(x, b_r: int, tau: float) -> np.ndarray:
    """fpround.py:164-177: strict |x - rnd(x)| > max(scale, 2^-126)*tau."""
    a = _as_f64(x)
    r = rnd_array(a, b_r)
    scale = np.maximum(exponent_scale_array(a), SCALE_FLOOR)
    logged = np.abs(a - r) > scale * np.float64(tau)
    codes = np.ones(a.shape, dtype=np.uint8)
    codes[logged & (a > r)] = DOWN
    codes[logged & (a < r)] = UP
    return _shape_back(codes, x)


def grid_neighbors_array(x, b_r: int) -> tuple[np.ndarray, np.ndarray]:
    """fpround.py:185-218: truncate-and-step in magnitude space; floor/ceil below 2^-126."""
    check_b(b_r)
    a = _as_f64(x).copy()
    _finite_or_raise(a)
    if (np.abs(a) > grid_max(b_r)).any():
        raise ValueError("out of representable range")
    _, mag, sign, drop, base, low = _split(a, b_r)
    trunc = base << drop
    away = trunc + np.where(low == 0, np.uint64(0), np.uint64(1) << drop)
    t_val = (sign | trunc).view(np.float64)
    a_val = (sign | away).view(np.float64)
    nonneg = a >= 0.0
    lo_n = np.where(nonneg, t_val, a_val)
    hi_n = np.where(nonneg, a_val, t_val)
    up_s, dn_s = _tiny_scale(b_r)
    scaled = np.where(mag >= _NORMAL_MIN_BITS, 0.0, a) * up_s
    lo = np.where(mag >= _NORMAL_MIN_BITS, lo_n, np.floor(scaled) * dn_s)
    hi = np.where(mag >= _NORMAL_MIN_BITS, hi_n, np.ceil(scaled) * dn_s)
    return _shape_back(lo, x), _shape_back(hi, x)


def rev_array(x, b_r: int, codes) -> np.ndarray:
    """fpround.py:227-247: take the neighbour on the coded side when rnd disagrees."""
    a = _as_f64(x)
    c = np.atleast_1d(np.asarray(codes))
    if c.shape != a.shape:
        raise ValueError(f"codes shape {c.shape} does not match values shape {a.shape}")
    if c.size and (c.min() < DOWN or c.max() > UP):
        raise ValueError("invalid direction code")
    r = rnd_array(a, b_r)
    lo, hi = grid_neighbors_array(a, b_r)
    out = r.copy()
    to_lo = (c == DOWN) & (a < r)
    to_hi = (c == UP) & (a > r)
    out[to_lo] = lo[to_lo]
    out[to_hi] = hi[to_hi]
    return _shape_back(out, x)


def is_on_grid(x, b_r: int) -> np.ndarray:
    """fpround.py:255-264."""
    check_b(b_r)
    a = _as_f64(x)
    f = a.astype(np.float32)
    exact = np.isfinite(f) & (f.astype(np.float64) == a)
    mask = np.uint32((1 << (32 - b_r)) - 1)
    return _shape_back(exact & ((f.view(np.uint32) & mask) == 0), x)


def normalized_distance(x, b_r: int) -> np.ndarray:
    """p = |x - rnd(x)| / max(scale(x), 2^-126): the quantity direction_array
    thresholds (fpround.py:171-173).  Exact in FP64."""
    a = _as_f64(x)
    r = rnd_array(a, b_r)
    scale = np.maximum(exponent_scale_array(a), SCALE_FLOOR)
    return np.abs(a - r) / scale


# --------------------------------------------------------------------------
# sparse log (north-star form)
# --------------------------------------------------------------------------

def sparse_from_codes(codes, base: int = 0) -> np.ndarray:
    """Lossless recoding of dense ternary codes: one uint64 word per code != 1,
    word = (global_index << 1) | (code == UP), ascending index."""
    c = np.asarray(codes, dtype=np.uint8).reshape(-1)
    idx = np.flatnonzero(c != IGNORE).astype(np.uint64)
    return ((idx + np.uint64(base)) << np.uint64(1)) | (c[idx.astype(np.int64)] == UP).astype(np.uint64)


def codes_from_sparse(words, n: int, base: int = 0) -> np.ndarray:
    w = np.asarray(words, dtype=np.uint64)
    out = np.ones(n, dtype=np.uint8)
    idx = (w >> np.uint64(1)).astype(np.int64) - base
    out[idx] = np.where((w & np.uint64(1)) != 0, UP, DOWN).astype(np.uint8)
    return out


# --------------------------------------------------------------------------
# .vtrl codec  (reference: pkg/src/vtrain/roundlog.py)
# --------------------------------------------------------------------------

HEADER_LEN = 15
_POW3 = np.array([1, 3, 9, 27, 81], dtype=np.uint16)


def pack_groups(digits) -> bytes:
    """roundlog.py:67-70: little-endian base 3, five digits per byte."""
    d = np.asarray(digits, dtype=np.uint16).reshape(-1, 5)
    return (d * _POW3).sum(axis=1).astype(np.uint8).tobytes()


def unpack_groups(raw: bytes) -> np.ndarray:
    """roundlog.py:73-82 (raises on a byte > 242)."""
    v = np.frombuffer(raw, dtype=np.uint8).astype(np.uint16)
    if v.size and int(v.max()) > 242:
        raise ValueError("corrupt log byte")
    cols = [(v // p) % 3 for p in _POW3]
    return np.stack(cols, axis=1).astype(np.uint8).reshape(-1)


def vtrl_bytes(chunks, b_r: int, compress: bool = False) -> bytes:
    """The exact file LogWriter produces for a sequence of write_array calls
    (roundlog.py:85-152): header with patched count, 5-digit groups, the
    final partial group padded with IGNORE, optional DEFLATE payload."""
    parts = [np.asarray(c, dtype=np.uint8).reshape(-1) for c in chunks]
    allc = np.concatenate(parts) if parts else np.zeros(0, np.uint8)
    if allc.size and int(allc.max()) > 2:
        raise ValueError("direction out of range")
    n = int(allc.size)
    pad = (-n) % 5
    payload = pack_groups(np.concatenate([allc, np.ones(pad, np.uint8)]))
    flags = 1 if compress else 0
    if compress:
        payload = zlib.compress(payload)
    header = b"VTRL" + bytes([1, b_r, flags]) + n.to_bytes(8, "little")
    return header + payload


# --------------------------------------------------------------------------
# threshold search  (reference: pkg/src/vtrain/protocol.py:494-506)
# --------------------------------------------------------------------------

def search_tau(samples, b_r: int, iters: int) -> float:
    """protocol.py:494-506: bisection with predicate all(p >= tau), returns the
    last midpoint; empty -> upper bound."""
    lo, hi = tau_bounds(b_r)
    s = list(samples)
    if not s:
        return hi
    t = lo
    for _ in range(iters):
        t = (lo + hi) / 2.0
        if all(p >= t for p in s):
            lo = t
        else:
            hi = t
    return t


def straddle_samples(y1, y2, b_r: int) -> list[float]:
    """protocol.py:483-490: where two profiles' outputs round to different
    grid points from opposite sides, both normalized distances."""
    a, b = _as_f64(y1).reshape(-1), _as_f64(y2).reshape(-1)
    r1, r2 = rnd_array(a, b_r), rnd_array(b, b_r)
    st = (r1 != r2) & (((a > r1) & (b < r2)) | ((a < r1) & (b > r2)))
    out: list[float] = []
    if st.any():
        for y, r in ((a, r1), (b, r2)):
            scale = np.maximum(exponent_scale_array(y[st]), SCALE_FLOOR)
            out.extend((np.abs(y[st] - r[st]) / scale).tolist())
    return out


def search_tau_budget(x, b_r: int, budget: int, iters: int = 30) -> float:
    """North-star budget search: the search_tau skeleton
    (same bounds, same midpoint) with predicate count(p > tau) <= budget;
    feasible -> upper = tau, else lower = tau; returns ``upper`` (always
    feasible)."""
    p = normalized_distance(x, b_r).reshape(-1)
    lo, hi = tau_bounds(b_r)
    for _ in range(iters):
        t = (lo + hi) / 2.0
        if int(np.count_nonzero(p > t)) <= budget:
            hi = t
        else:
            lo = t
    return hi


def kth_largest(p, k: int) -> float:
    """The (k+1)-th largest value of p (k 0-based from the top), by
    np.partition: the order statistic the budget predicate reduces to,
    count(p > tau) <= k  <=>  kth_largest(p, k) <= tau."""
    a = np.asarray(p, dtype=np.float64).reshape(-1)
    return float(np.partition(a, a.size - 1 - k)[a.size - 1 - k])


def bisect_budget(v, b_r: int, iters: int = 30) -> float:
    """The search_tau skeleton (protocol.py:494-506 bounds and midpoint) on the
    order-statistic predicate v <= tau; v None = no element can exceed the
    budget (n <= budget): every tau is feasible.  Returns ``upper``."""
    lo, hi = tau_bounds(b_r)
    for _ in range(iters):
        t = (lo + hi) / 2.0
        if v is None or v <= t:
            hi = t
        else:
            lo = t
    return hi


def search_tau_budget_kth(x, b_r: int, budget: int, iters: int = 30) -> float:
    """search_tau_budget through the order statistic (one np.partition instead
    of ``iters`` counting passes); equal to it bit for bit
    (tests/test_oracle_golden.py checks the two against each other)."""
    p = normalized_distance(x, b_r).reshape(-1)
    return bisect_budget(kth_largest(p, budget) if p.size > budget else None, b_r, iters)


# --------------------------------------------------------------------------
# Merkle  (reference: pkg/src/vtrain/merkle.py)
# --------------------------------------------------------------------------

def sha256(data: bytes) -> bytes:
    return hashlib.sha256(data).digest()


def merkle_levels(leaves: list[bytes]) -> list[list[bytes]]:
    """merkle.py:55-72: node = SHA-256(left || right); an unpaired last node is
    promoted unchanged; every level kept."""
    if not leaves:
        raise ValueError("cannot build a Merkle tree with no leaves")
    levels = [list(leaves)]
    while len(levels[-1]) > 1:
        cur = levels[-1]
        nxt = [sha256(cur[i] + cur[i + 1]) for i in range(0, len(cur) - 1, 2)]
        if len(cur) % 2:
            nxt.append(cur[-1])
        levels.append(nxt)
    return levels


def chunk_leaves(data: bytes, leaf_bytes: int = 4096) -> list[bytes]:
    """North-star chunked leaves: SHA-256 of each
    ``leaf_bytes`` slice; the last slice may be short."""
    return [sha256(data[i:i + leaf_bytes]) for i in range(0, len(data), leaf_bytes)]


def hash_weights(tensors) -> bytes:
    """merkle.py:155-166: one SHA-256 over the FP32 little-endian bytes."""
    h = hashlib.sha256()
    for i, t in enumerate(tensors):
        a = np.ascontiguousarray(t, dtype=np.float64)
        if not np.isfinite(a).all():
            bad = int(np.flatnonzero(~np.isfinite(a))[0])
            raise ValueError(f"non-finite weight in tensor {i} at flat index {bad}")
        h.update(a.astype("<f4").tobytes())
    return h.digest()
