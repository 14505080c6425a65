"""Parallel driver for the CPU oracle at BASELINE sizes -- TEST INFRASTRUCTURE ONLY.

The oracle (``vt_oracle``) is element-wise NumPy: every function of the
reference path except the order statistic of the budget search is exact on
any contiguous chunk.  This module runs it over all host cores so the GPU
results at the full BASELINE sizes (2^26 pairs, the 161 ResNet-50 tensors,
full-size GPT-2 activations, the 1.5e9-parameter Merkle tree) can be checked
against it in seconds:

* the parent process holds the inputs AND the GPU's outputs as NumPy arrays
  in ``_SHARED`` and forks a pool; the children see them copy-on-write (no
  pickling of large arrays), recompute the oracle on their chunk and compare
  there, returning only mismatch counts and the first bad position;
* the (budget+1)-th largest normalized distance is exact: each chunk returns
  its own top budget+1 values, the parent selects among their union.

Only ``tests/`` and ``bench.py``'s CPU legs may import it (like the oracle).
Children never touch CUDA.
"""

from __future__ import annotations

import hashlib
import multiprocessing as mp
import os

import numpy as np

import vt_oracle as O

_SHARED: dict = {}


def cores() -> int:
    return len(os.sched_getaffinity(0))


def _pool(procs: int | None = None):
    return mp.get_context("fork").Pool(procs or cores())


def chunks(n: int, chunk: int) -> list[tuple[int, int]]:
    return [(lo, min(n, lo + chunk)) for lo in range(0, n, chunk)]


def _first_bad(a: np.ndarray, b: np.ndarray) -> tuple[int, int]:
    if a.shape != b.shape:
        return max(a.size, b.size), 0
    bad = np.flatnonzero(a != b)
    return int(bad.size), int(bad[0]) if bad.size else -1


def _words_in(words: np.ndarray, lo: int, hi: int, base: int) -> np.ndarray:
    idx = words >> np.uint64(1)
    a = int(np.searchsorted(idx, np.uint64(lo + base)))
    b = int(np.searchsorted(idx, np.uint64(hi + base)))
    return words[a:b]


# ---------------------------------------------------------------------------
# round-and-log / replay
# ---------------------------------------------------------------------------

def _uint(a: np.ndarray):
    return {8: np.uint64, 4: np.uint32, 2: np.uint16, 1: np.uint8}[a.dtype.itemsize]


def _check_chunk(job):
    t, lo, hi = job
    S = _SHARED["items"][t]
    b_r, tau, base = S["b_r"], S["tau"], S["base"]
    xt = S["xt"][lo:hi]
    codes = O.direction_array(xt, b_r, tau)
    out = {"t": t, "lo": lo, "n_log": int(np.count_nonzero(codes != O.IGNORE))}
    want_w = O.sparse_from_codes(codes, base=lo + base)
    got_w = _words_in(S["words"], lo, hi, base)
    out["log"] = _first_bad(got_w, want_w)
    if S.get("yt") is not None:
        want = O.rnd_array(xt, b_r).astype(S["yt"].dtype)
        out["yt"] = _first_bad(S["yt"][lo:hi].view(_uint(want)), want.view(_uint(want)))
    if S.get("xa") is not None:
        want = O.rev_array(S["xa"][lo:hi], b_r, codes).astype(S["ya"].dtype)
        out["ya"] = _first_bad(S["ya"][lo:hi].view(_uint(want)), want.view(_uint(want)))
        # _AuditorChannel.process: corrections = count(out != rnd(x')) (protocol.py:212-216)
        r = O.rnd_array(S["xa"][lo:hi], b_r).astype(S["ya"].dtype)
        out["corr"] = int(np.count_nonzero(want.view(_uint(want)) != r.view(_uint(r))))
    return out


def check_many(items: list[dict], chunk: int = 1 << 22, procs: int | None = None) -> list[dict]:
    """``check_round_and_log`` for many tensors in one pool.  Each item: xt,
    b_r, tau, words (GPU sparse log), optional yt (GPU rounded output, FP32 or
    FP64), optional xa / ya (auditor input and GPU replay output), base."""
    _SHARED.clear()
    _SHARED["items"] = [{"base": 0, **it} for it in items]
    for it in _SHARED["items"]:
        it["words"] = np.asarray(it["words"]).view(np.uint64)
    jobs = [(t, lo, hi) for t, it in enumerate(_SHARED["items"]) for lo, hi in chunks(it["xt"].size, chunk)]
    try:
        with _pool(procs) as pool:
            res = pool.map(_check_chunk, jobs)
    finally:
        _SHARED.clear()
    out = []
    for t, it in enumerate(items):
        rs = [r for r in res if r["t"] == t]
        tot = {"n_log": sum(r["n_log"] for r in rs), "words": int(np.asarray(it["words"]).size)}
        for k in ("log", "yt", "ya"):
            if rs and k in rs[0]:
                bad = [(r["lo"] + r[k][1], r[k][0]) for r in rs if r[k][0]]
                tot[k + "_mismatches"] = sum(b for _, b in bad)
                tot[k + "_first_bad"] = bad[0][0] if bad else -1
        if rs and "corr" in rs[0]:
            tot["corrections"] = sum(r["corr"] for r in rs)
        out.append(tot)
    return out


def check_round_and_log(xt: np.ndarray, b_r: int, tau: float, words: np.ndarray, yt: np.ndarray | None = None,
                        xa: np.ndarray | None = None, ya: np.ndarray | None = None, base: int = 0,
                        chunk: int = 1 << 22, procs: int | None = None) -> dict:
    """Compare a GPU round-and-log (sparse log ``words``, rounded ``yt``) and
    optionally a GPU replay of ``xa`` (``ya``) with the oracle, chunk by chunk
    over all cores.  Returns totals: entries the oracle logs, mismatches per
    output (0 = bit-exact) and the oracle's correction count."""
    return check_many([dict(xt=xt, b_r=b_r, tau=tau, words=words, yt=yt, xa=xa, ya=ya, base=base)],
                      chunk, procs)[0]


def assert_clean(r: dict, what: str = "") -> None:
    """Every output bit-exact and the GPU log as long as the oracle's."""
    for k, v in r.items():
        if k.endswith("_mismatches"):
            assert v == 0, (what, r)
    assert r["n_log"] == r["words"], (what, r)


# ---------------------------------------------------------------------------
# budget search: exact (budget+1)-th largest p over chunks
# ---------------------------------------------------------------------------

def _top_chunk(job):
    key, lo, hi, k = job
    p = O.normalized_distance(_SHARED[key][lo:hi], _SHARED["b_r"]).reshape(-1)
    if p.size > k:
        p = np.partition(p, p.size - k)[p.size - k:]
    return p


def _tau_from_top(tops: list[np.ndarray], n: int, b_r: int, budget: int, iters: int) -> float:
    allp = np.concatenate(tops) if tops else np.zeros(0)
    v = O.kth_largest(allp, budget) if n > budget else None
    return O.bisect_budget(v, b_r, iters)


def search_tau_budget_many(tensors: list[np.ndarray], b_r: int, budgets: list[int], iters: int = 30,
                           chunk: int = 1 << 22, procs: int | None = None) -> list[float]:
    """oracle.search_tau_budget_kth for many tensors at once, over all cores."""
    _SHARED.clear()
    _SHARED["b_r"] = b_r
    jobs, owner = [], []
    for t, (x, B) in enumerate(zip(tensors, budgets)):
        _SHARED[t] = np.asarray(x).reshape(-1)
        # each chunk returns its top budget+1 values: large tensors in fewer,
        # larger chunks (about two per core) to keep that traffic small
        step = max(chunk, -(-_SHARED[t].size // (2 * cores())))
        for lo, hi in chunks(_SHARED[t].size, step):
            jobs.append((t, lo, hi, int(B) + 1))
            owner.append(t)
    try:
        with _pool(procs) as pool:
            res = pool.map(_top_chunk, jobs)
    finally:
        _SHARED.clear()
    out = []
    for t, (x, B) in enumerate(zip(tensors, budgets)):
        tops = [r for r, o in zip(res, owner) if o == t]
        out.append(_tau_from_top(tops, int(np.asarray(x).size), b_r, int(B), iters))
    return out


# ---------------------------------------------------------------------------
# Merkle: 4 KiB leaves and every level
# ---------------------------------------------------------------------------

def _leaf_chunk(job):
    lo, hi = job
    raw = _SHARED["data"]
    lb = _SHARED["leaf"]
    return b"".join(hashlib.sha256(raw[i * lb:(i + 1) * lb]).digest() for i in range(lo, hi))


def _level_chunk(job):
    lo, hi = job
    cur = _SHARED["level"]
    return b"".join(hashlib.sha256(cur[64 * i: 64 * i + 64]).digest() for i in range(lo, hi))


def merkle_levels_bytes(data: memoryview | bytes, leaf_bytes: int = 4096, procs: int | None = None) -> list[bytes]:
    """merkle.build over the chunked leaves, every level as the
    concatenation of its 32-byte nodes; leaves and pair hashes over all cores
    (hashlib = the reference's own SHA-256)."""
    nbytes = memoryview(data).nbytes
    n_leaves = (nbytes + leaf_bytes - 1) // leaf_bytes
    if n_leaves == 0:
        raise ValueError("cannot build a Merkle tree with no leaves")
    per = max(1, n_leaves // (4 * cores()))
    _SHARED.clear()
    _SHARED.update(data=memoryview(data).cast("B"), leaf=leaf_bytes)
    try:
        with _pool(procs) as pool:
            levels = [b"".join(pool.map(_leaf_chunk, chunks(n_leaves, per)))]
        while len(levels[-1]) > 32:
            cur = levels[-1]
            m = len(cur) // 32
            pairs = m // 2
            _SHARED["level"] = cur
            if pairs > 4096:
                with _pool(procs) as pool:
                    nxt = b"".join(pool.map(_level_chunk, chunks(pairs, max(1, pairs // (4 * cores())))))
            else:
                nxt = _level_chunk((0, pairs))
            if m % 2:
                nxt += cur[-32:]  # unpaired last node promoted unchanged (merkle.py:63-71)
            levels.append(nxt)
    finally:
        _SHARED.clear()
    return levels
