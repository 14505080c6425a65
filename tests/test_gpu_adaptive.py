"""GPU parity of the one-pass adaptive round-and-log (ops.round_and_log_adaptive:
candidates at a threshold below tau during the rounding pass, exact selection
among them, FP64 bisection, ordered filter; exact multi-pass fallback) against
the oracle's budget search (the protocol.search_tau skeleton of
pkg/src/vtrain/protocol.py:494-506 in budget form) and the
oracle direction codes at that tau (fpround.py:164-177)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu


def _check(oracle, x, b_r, B, base=0, out_dtype=None):
    import torch
    from paper_2403_09603_b200 import ops
    kw = {} if out_dtype is None else {"out_dtype": out_dtype}
    y, log, tau = ops.round_and_log_adaptive(torch.from_numpy(x).cuda(), b_r, B, global_base=base, **kw)
    t_or = oracle.search_tau_budget(x, b_r, B)
    assert tau == t_or, (tau.hex(), t_or.hex())
    codes = oracle.direction_array(x, b_r, t_or)
    want = oracle.sparse_from_codes(codes, base=base)
    assert log.count == want.size
    assert np.array_equal(log.words.cpu().numpy().view(np.uint64), want)
    r = oracle.rnd_array(x, b_r)
    got = y.cpu().numpy()
    assert np.array_equal(bits(got), bits(r if got.dtype == np.float64 else r.astype(np.float32)))
    return log.count


@pytest.mark.parametrize("n", [1, 7, 1000, 5_000, 200_003, 4_000_037])
def test_fast_path_sizes(oracle, n):
    x = np.random.default_rng(n).normal(0.0, 0.7, size=n)
    B = int(0.005 * n)
    cnt = _check(oracle, x, 32, B, base=3 * n)
    assert cnt <= B


@pytest.mark.parametrize("B", [0, 1, 17, 2_500])
def test_budgets(oracle, B):
    x = np.random.default_rng(100 + B).normal(0.0, 5.0, size=500_000)
    _check(oracle, x, 32, B)


def test_fallbacks(oracle):
    """Inputs the candidate threshold cannot decide: too few candidates
    (mostly on-grid data), too many (exact midpoints, a 40% budget)."""
    rng = np.random.default_rng(7)
    n = 300_000
    sparse = np.where(rng.random(n) < 0.9, np.round(rng.normal(0, 100, n)), rng.normal(0, 1, n))
    _check(oracle, sparse, 32, int(0.005 * n))
    from paper_2403_09603_b200 import workloads
    _check(oracle, workloads.config0_x(n, 8), 32, int(0.005 * n))
    _check(oracle, rng.normal(0, 1, n), 32, int(0.4 * n))


def test_general_grid_and_fp64_out(oracle):
    import torch
    x = np.random.default_rng(9).normal(0.0, 2.0, size=123_457)
    _check(oracle, x, 26, 600, out_dtype=torch.float64)
    _check(oracle, x, 10, 600)


def test_tiny_magnitudes(oracle):
    """Values below 2^-126 (absolute grid, FP64 distance) mixed with normal ones."""
    rng = np.random.default_rng(10)
    x = rng.normal(0, 1, 100_000) * np.exp2(rng.integers(-160, 4, 100_000))
    _check(oracle, x, 32, 500)


def test_repeated_calls_share_workspace(oracle):
    """The filter's epoch / ticket state and the candidate histograms are
    reset by the kernels themselves: many calls of mixed sizes on one
    workspace, including fallbacks in between."""
    from paper_2403_09603_b200 import workloads
    rng = np.random.default_rng(11)
    xs = [rng.normal(0, 1, 250_000), workloads.config0_x(60_000, 12), rng.normal(0, 1e-3, 31_000),
          rng.normal(0, 1, 250_000)]
    for rep in range(3):
        for x in xs:
            _check(oracle, x, 32, int(0.005 * x.size))


def test_in_place_fp64(oracle):
    """y written over x (the hooks' use): the selection runs on x before the
    rounding pass overwrites it."""
    import torch
    from paper_2403_09603_b200 import ops
    x = np.random.default_rng(13).normal(0.0, 0.3, size=333_333)
    xt = torch.from_numpy(x.copy()).cuda()
    B = int(0.005 * x.size)
    y, log, tau = ops.round_and_log_adaptive(xt, 32, B, out_dtype=torch.float64, out=xt)
    t_or = oracle.search_tau_budget(x, 32, B)
    assert tau == t_or
    assert np.array_equal(log.words.cpu().numpy().view(np.uint64),
                          oracle.sparse_from_codes(oracle.direction_array(x, 32, t_or)))
    assert np.array_equal(bits(xt.cpu().numpy()), bits(oracle.rnd_array(x, 32)))


@pytest.mark.parametrize("b_r,kind", [(32, "zeros"), (32, "tiny"), (32, "ragged"), (26, "normal"), (10, "tiny")])
def test_in_place_key_pass(oracle, b_r, kind):
    """The in-place key pass (adapt_keys32_kernel for b_r = 32, the general
    kernel otherwise): exact zeros (never candidates on the fast test),
    values below 2^-126 and beyond FP32 (the FP64 key path), and sizes that
    end inside a CTA iteration."""
    import torch
    from paper_2403_09603_b200 import ops
    rng = np.random.default_rng(17 + b_r)
    n = {"ragged": 4096 * 37 + 1234}.get(kind, 250_001)
    x = rng.normal(0.0, 1.0, n)
    if kind == "zeros":
        x[rng.random(n) < 0.4] = 0.0
        x[rng.random(n) < 0.01] = -0.0
    elif kind == "tiny":
        x = x * np.exp2(rng.integers(-160, 20, n))
    xt = torch.from_numpy(x.copy()).cuda()
    B = int(0.005 * n)
    y, log, tau = ops.round_and_log_adaptive(xt, b_r, B, out_dtype=torch.float64, out=xt)
    t_or = oracle.search_tau_budget(x, b_r, B)
    assert tau == t_or, (tau.hex(), t_or.hex())
    assert np.array_equal(log.words.cpu().numpy().view(np.uint64),
                          oracle.sparse_from_codes(oracle.direction_array(x, b_r, t_or)))
    assert np.array_equal(bits(xt.cpu().numpy()), bits(oracle.rnd_array(x, b_r)))


@pytest.mark.parametrize("case", ["on_grid", "midpoints", "huge_budget", "low"])
def test_in_place_tail_decisions(oracle, case):
    """Every decision of the cooperative tail, in place: too few candidates
    (mostly on-grid data -> exact fallback), too many (exact midpoints, a 40%
    budget), and v <= tau_lo settled from the key pass's count alone."""
    import torch
    from paper_2403_09603_b200 import ops, workloads
    rng = np.random.default_rng(23)
    n = 300_000
    B = int(0.005 * n)
    if case == "on_grid":
        x = np.where(rng.random(n) < 0.9, np.round(rng.normal(0, 100, n)), rng.normal(0, 1, n))
    elif case == "midpoints":
        x = workloads.config0_x(n, 8)
    elif case == "huge_budget":
        x = rng.normal(0, 1, n)
        B = int(0.4 * n)
    else:  # nearly everything on the grid, the rest far from the midpoint: p <= tau_lo for all
        x = np.round(rng.normal(0, 100, n))
        k = rng.random(n) < 0.002
        x[k] += 0.25
    xt = torch.from_numpy(x.copy()).cuda()
    y, log, tau = ops.round_and_log_adaptive(xt, 32, B, out_dtype=torch.float64, out=xt)
    t_or = oracle.search_tau_budget(x, 32, B)
    assert tau == t_or, (tau.hex(), t_or.hex())
    assert np.array_equal(log.words.cpu().numpy().view(np.uint64),
                          oracle.sparse_from_codes(oracle.direction_array(x, 32, t_or)))
    assert np.array_equal(bits(xt.cpu().numpy()), bits(oracle.rnd_array(x, 32)))
    # the workspace is clean afterwards: a plain call on fresh data still matches
    z = rng.normal(0, 1, 50_000)
    zt = torch.from_numpy(z.copy()).cuda()
    _, log2, tau2 = ops.round_and_log_adaptive(zt, 32, 250, out_dtype=torch.float64, out=zt)
    assert tau2 == oracle.search_tau_budget(z, 32, 250)


@pytest.mark.parametrize("in_place", [False, True])
def test_hot_digit_tail(oracle, in_place):
    """More than 2048 keys in the selected digit, all tied: the tail's
    multi-level exact selection (not the direct count) with the (B+1)-th
    largest key inside a run of equal keys."""
    import torch
    from paper_2403_09603_b200 import ops
    rng = np.random.default_rng(29)
    n = 1_000_000
    x = rng.normal(0.0, 1.0, n)
    hot = rng.random(n) < 0.03
    b = x.view(np.uint64).copy()
    b[hot] = (b[hot] & ~np.uint64(0x1FFFFFFF)) | np.uint64((1 << 28) - 5)  # same low 29 bits: equal p
    x = b.view(np.float64)
    B = int(0.005 * n)
    xt = torch.from_numpy(x.copy()).cuda()
    kw = dict(out_dtype=torch.float64, out=xt) if in_place else {}
    y, log, tau = ops.round_and_log_adaptive(xt, 32, B, **kw)
    t_or = oracle.search_tau_budget(x, 32, B)
    assert tau == t_or, (tau.hex(), t_or.hex())
    assert np.array_equal(log.words.cpu().numpy().view(np.uint64),
                          oracle.sparse_from_codes(oracle.direction_array(x, 32, t_or)))
    r = oracle.rnd_array(x, 32)
    got = (xt if in_place else y).cpu().numpy()
    assert np.array_equal(bits(got), bits(r if got.dtype == np.float64 else r.astype(np.float32)))


@pytest.mark.parametrize("frac", [0.02, 0.1])
def test_out_of_place_dense_candidates(oracle, frac):
    """Out of place, the rounding pass stages each candidate's x for the
    tail; rows with more candidates than it stages (budgets of 2 % / 10 %)
    are gathered from x.  tau, log and y equal the oracle's."""
    import torch
    from paper_2403_09603_b200 import ops
    rng = np.random.default_rng(int(1000 * frac) + 7)
    for x in (rng.normal(0.0, 1.0, 300_001),
              rng.normal(0.0, 1.0, 100_000) * np.exp2(rng.integers(-140, -120, 100_000))):
        B = int(frac * x.size)
        y, log, tau = ops.round_and_log_adaptive(torch.from_numpy(x).cuda(), 32, B)
        t_or = oracle.search_tau_budget(x, 32, B)
        assert tau == t_or
        want = oracle.sparse_from_codes(oracle.direction_array(x, 32, t_or))
        assert np.array_equal(log.words.cpu().numpy().view(np.uint64), want)
        assert np.array_equal(y.cpu().numpy().view(np.uint32), oracle.rnd_array(x, 32).astype(np.float32).view(np.uint32))
