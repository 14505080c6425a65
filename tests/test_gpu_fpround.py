"""GPU parity: grid operators and the fused round-and-log / replay kernels
against the reference goldens and the oracle, bit for bit."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu

B_VALUES = (10, 26, 29, 32)


@pytest.fixture(scope="module")
def fp():
    from paper_2403_09603_b200 import fpround
    return fpround


@pytest.mark.parametrize("b_r", B_VALUES)
def test_fpround_golden(golden, fp, b_r):
    g = golden.fpround
    x = g[f"x_{b_r}"]
    assert np.array_equal(bits(fp.rnd_array(x, b_r)), bits(g[f"rnd_{b_r}"]))
    lo, hi = fp.grid_neighbors_array(x, b_r)
    assert np.array_equal(bits(lo), bits(g[f"below_{b_r}"]))
    assert np.array_equal(bits(hi), bits(g[f"above_{b_r}"]))
    assert np.array_equal(bits(fp.exponent_scale_array(x)), bits(g[f"scale_{b_r}"]))
    assert np.array_equal(fp.is_on_grid(x, b_r), g[f"ongrid_{b_r}"])
    assert np.array_equal(bits(fp.rev_array(x, b_r, g[f"codes_{b_r}"])), bits(g[f"rev_{b_r}"]))
    for i, t in enumerate(g[f"taus_{b_r}"]):
        d = fp.direction_array(x, b_r, float(t))
        assert np.array_equal(d, g[f"dir_{b_r}_{i}"]), (b_r, t)
        assert np.array_equal(bits(fp.rev_array(x, b_r, d)), bits(g[f"revdir_{b_r}_{i}"]))


def _call(fp, case):
    x = np.array([float.fromhex(v) for v in case["x"]])
    fn, b_r = case["fn"], case["b_r"]
    if fn == "rnd_array":
        return fp.rnd_array(x, b_r)
    if fn == "grid_neighbors_array":
        return fp.grid_neighbors_array(x, b_r)
    if fn == "rev_array":
        return fp.rev_array(x, b_r, np.ones(x.shape, np.uint8))
    if fn == "direction_array":
        return fp.direction_array(x, b_r, 2.0 ** -25)
    if fn == "exponent_scale_array":
        return fp.exponent_scale_array(x)
    if fn.startswith("rev_array_badcode"):
        return fp.rev_array(x, b_r, np.full(x.shape, 3, np.uint8))
    if fn == "rev_array_shape":
        return fp.rev_array(x, b_r, np.ones(3, np.uint8))
    raise AssertionError(fn)


def test_error_semantics_golden(golden, fp):
    for case in golden.errors:
        if case["error"] is None:
            _call(fp, case)
        else:
            with pytest.raises(ValueError) as ei:
                _call(fp, case)
            assert str(ei.value) == case["error"], case


def test_known_answers(fp):
    # reference tests: test_fpround.py:55-123, 147-174, 214-248
    assert fp.rnd(1.0 + 2.0 ** -24, 32) == 1.0
    for b in B_VALUES:
        assert fp.rnd(0.0, b) == 0.0
    p = fp.RoundingParams(b_r=32, tau=0.25 * 2.0 ** -23)
    assert fp.direction(1.0 + 0.75 * 2.0 ** -23, p) == fp.IGNORE
    assert fp.direction(1.0 + 0.6 * 2.0 ** -23, p) == fp.UP
    assert fp.direction(1.0 + 0.4 * 2.0 ** -23, p) == fp.DOWN
    assert fp.rev(1.0 + 0.4 * 2.0 ** -23, 32, fp.UP) == 1.0 + 2.0 ** -23
    assert fp.rev(1.0 + 0.6 * 2.0 ** -23, 32, fp.UP) == 1.0 + 2.0 ** -23
    assert fp.rev(1.0 + 0.6 * 2.0 ** -23, 32, fp.DOWN) == 1.0
    g = fp.rnd(3.7, 28)
    for c in (0, 1, 2):
        assert fp.rev(g, 28, c) == g
    assert fp.grid_neighbors(1.0 + 0.5 * 2.0 ** -23, 32) == (1.0, 1.0 + 2.0 ** -23)
    assert bits(fp.rnd_array(-(2.0 ** -151), 32))[0] == bits(np.array([-0.0]))[0]
    assert fp.rnd_array(np.float64(2.5), 32).shape == (1,)
    with pytest.raises(ValueError):
        fp.RoundingParams(b_r=32, tau=0.6 * 2.0 ** -23)


@pytest.mark.parametrize("b_r", (26, 29, 32))
def test_random_wide_vs_oracle(oracle, fp, b_r):
    rng = np.random.default_rng(1000 + b_r)
    n = 300_001
    x = rng.normal(size=n) * np.exp2(rng.integers(-140, 120, size=n))
    x = x[np.abs(x) <= oracle.grid_max(b_r)]
    tau = 0.25 * 2.0 ** -23
    assert np.array_equal(bits(fp.rnd_array(x, b_r)), bits(oracle.rnd_array(x, b_r)))
    assert np.array_equal(fp.direction_array(x, b_r, tau), oracle.direction_array(x, b_r, tau))
    codes = rng.integers(0, 3, size=x.size).astype(np.uint8)
    assert np.array_equal(bits(fp.rev_array(x, b_r, codes)), bits(oracle.rev_array(x, b_r, codes)))


def test_sync_property(fp, oracle):
    # reference test_fpround.py:251-274 on the GPU operators
    for b_r in (26, 29, 32):
        rng = np.random.default_rng(b_r)
        n = 200_000
        tau = 0.25 * 2.0 ** -23
        x = rng.normal(size=n) * np.exp2(rng.integers(-30, 30, size=n))
        scale = np.maximum(oracle.exponent_scale_array(x), oracle.SCALE_FLOOR)
        bound = np.minimum(0.25 * oracle.epsilon(b_r, 1.0) * scale, tau * scale)
        xp = x + rng.uniform(-1.0, 1.0, size=n) * bound
        keep = (np.abs(xp - x) < bound) & (oracle.exponent_scale_array(xp) == oracle.exponent_scale_array(x))
        x, xp = x[keep], xp[keep]
        codes = fp.direction_array(x, b_r, tau)
        assert np.array_equal(bits(fp.rev_array(xp, b_r, codes)), bits(fp.rev_array(x, b_r, codes)))


def test_torch_in_torch_out(fp, oracle):
    import torch
    x = torch.randn(4099, dtype=torch.float64, device="cuda") * 3
    y = fp.rnd_array(x, 32)
    assert y.is_cuda and y.dtype == torch.float64 and y.shape == x.shape
    assert np.array_equal(bits(y.cpu().numpy()), bits(oracle.rnd_array(x.cpu().numpy(), 32)))
    # non-contiguous / misaligned views are handled by an aligned copy
    xv = x[1:]
    assert np.array_equal(bits(fp.rnd_array(xv, 32).cpu().numpy()), bits(oracle.rnd_array(xv.cpu().numpy(), 32)))
    x2 = x.reshape(-1, 1)[::2, 0]
    assert np.array_equal(bits(fp.rnd_array(x2, 32).cpu().numpy()), bits(oracle.rnd_array(x2.cpu().numpy(), 32)))


# ---------------------------------------------------------------------------
# fused north-star operators
# ---------------------------------------------------------------------------

def _sparse_np(log):
    return log.words.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 127, 128, 640, 5119, 5120, 5121, 10240 + 77, 200_003])
def test_round_and_log_ragged(oracle, n):
    import torch
    from paper_2403_09603_b200 import ops, workloads
    x = workloads.config0_x(n, seed=n) if n else np.zeros(0)
    tau = workloads.TAU_CONFIG0
    xt = torch.from_numpy(x).cuda()
    y, log = ops.round_and_log(xt, 32, tau, global_base=12345)
    codes = oracle.direction_array(x, 32, tau) if n else np.zeros(0, np.uint8)
    want = oracle.sparse_from_codes(codes, base=12345)
    assert log.count == want.size
    assert np.array_equal(_sparse_np(log), want)
    if n:
        assert np.array_equal(bits(y.cpu().numpy()), bits(oracle.rnd_array(x, 32).astype(np.float32)))
    y64, log64 = ops.round_and_log(xt, 32, tau, out_dtype=torch.float64)
    if n:
        assert np.array_equal(bits(y64.cpu().numpy()), bits(oracle.rnd_array(x, 32)))
    assert np.array_equal(_sparse_np(log64), oracle.sparse_from_codes(codes))
    # replay with the trainer's own input reproduces the trainer output
    ya, corr = ops.replay(xt, 32, log, global_base=12345)
    assert corr == 0
    assert np.array_equal(bits(ya.cpu().numpy()), bits(y.cpu().numpy()))


def test_config0_golden(golden):
    import torch
    from paper_2403_09603_b200 import ops, workloads
    c0 = golden.configs["config0"]
    x = workloads.config0_x(c0["n"], c0["seed"])
    assert hashlib.sha256(x.tobytes()).hexdigest() == c0["x_sha"]
    y, log = ops.round_and_log(torch.from_numpy(x).cuda(), 32, float.fromhex(c0["tau"]))
    assert hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest() == c0["rnd_f32_sha"]
    assert log.count == c0["logged"]
    assert hashlib.sha256(_sparse_np(log).tobytes()).hexdigest() == c0["sparse_sha"]
    assert int(log.up().sum()) == c0["n_up"]


def test_config1_golden(golden):
    import torch
    from paper_2403_09603_b200 import ops, workloads
    c1 = golden.configs["config1"]
    xt, xa = workloads.config1_pair(c1["n"], c1["seed"])
    tau = float.fromhex(c1["tau"])
    yt, log = ops.round_and_log(torch.from_numpy(xt).cuda(), 32, tau)
    ya, corr = ops.replay(torch.from_numpy(xa).cuda(), 32, log)
    assert hashlib.sha256(yt.cpu().numpy().tobytes()).hexdigest() == c1["trainer_f32_sha"]
    assert hashlib.sha256(ya.cpu().numpy().tobytes()).hexdigest() == c1["auditor_f32_sha"]
    assert corr == c1["corrections"]
    assert log.count == c1["logged"]


def test_config1_pair_4m_vs_oracle(oracle):
    import torch
    from paper_2403_09603_b200 import ops, workloads
    n = 1 << 22
    xt, xa = workloads.config1_pair(n, 7)
    tau = workloads.TAU_CONFIG0
    yt, log = ops.round_and_log(torch.from_numpy(xt).cuda(), 32, tau)
    ya, corr = ops.replay(torch.from_numpy(xa).cuda(), 32, log)
    codes = oracle.direction_array(xt, 32, tau)
    want = oracle.rev_array(xa, 32, codes)
    assert np.array_equal(bits(ya.cpu().numpy()), bits(want.astype(np.float32)))
    assert np.array_equal(bits(yt.cpu().numpy()), bits(ya.cpu().numpy()))
    assert corr == int(np.count_nonzero(want != oracle.rnd_array(xa, 32)))


def test_replay_forces_logged_direction(oracle):
    """Corrections happen: auditor values on the other side of the midpoint."""
    import torch
    from paper_2403_09603_b200 import ops
    rng = np.random.default_rng(3)
    n = 100_000
    base = (rng.integers(1 << 23, 1 << 24, size=n) + 0.5) * 2.0 ** -23  # FP32 midpoints in [1, 2)
    delta = rng.uniform(0.01, 0.2, size=n) * 2.0 ** -23
    xt = base + delta * np.where(rng.random(n) < 0.5, 1, -1)
    xa = xt.copy()
    flip = rng.random(n) < 0.3
    xa[flip] = base[flip] - (xt[flip] - base[flip])  # mirror across the midpoint
    tau = 2.0 ** -25
    _, log = ops.round_and_log(torch.from_numpy(xt).cuda(), 32, tau)
    ya, corr = ops.replay(torch.from_numpy(xa).cuda(), 32, log)
    want = oracle.rev_array(xa, 32, oracle.direction_array(xt, 32, tau))
    assert np.array_equal(bits(ya.cpu().numpy()), bits(want.astype(np.float32)))
    assert corr == int(np.count_nonzero(want != oracle.rnd_array(xa, 32))) > 0


def test_sparse_log_errors():
    import torch
    from paper_2403_09603_b200 import ops
    x = torch.randn(20000, dtype=torch.float64, device="cuda")
    _, log = ops.round_and_log(x, 32, 2.0 ** -25)
    assert log.count > 10
    bad = log.words.clone()
    bad[[3, 4]] = bad[[4, 3]]
    with pytest.raises(ops.SparseLogError):
        ops.replay(x, 32, bad)
    with pytest.raises(ops.SparseLogError):
        ops.replay(x[:1000], 32, log)  # entries beyond the tensor are not consumed


def test_round_and_log_errors():
    import torch
    from paper_2403_09603_b200 import ops
    x = torch.ones(10000, dtype=torch.float64, device="cuda")
    x[7777] = float("nan")
    x[5] = 1e39
    with pytest.raises(ValueError, match="non-finite value"):
        ops.round_and_log(x, 32, 2.0 ** -25)
    x[7777] = 1.0
    with pytest.raises(ValueError, match="out of representable range"):
        ops.round_and_log(x, 32, 2.0 ** -25)


def test_log_overflow_detected():
    import torch
    from paper_2403_09603_b200 import ops
    x = torch.randn(50000, dtype=torch.float64, device="cuda")
    with pytest.raises(ops.LogOverflow):
        ops.round_and_log(x, 32, 0.0, log_out=torch.empty(100, dtype=torch.int64, device="cuda"))


@pytest.mark.parametrize("b_r", (10, 26, 32))
def test_special_values_fused(oracle, b_r):
    import torch
    from paper_2403_09603_b200 import ops
    gm = oracle.grid_max(b_r)
    q = 2.0 ** ((32 - b_r) - 149)
    vals = np.array([0.0, -0.0, 2.0 ** -126, -(2.0 ** -126), q, -q, 0.5 * q, -0.5 * q, 1.5 * q, 2.5 * q,
                     np.nextafter(2.0 ** -126, 0), gm, -gm, 1.0, 1.0 + 2.0 ** -24, 1e-300, -1e-300] * 700)
    for tau in (0.0, 2.0 ** -25, 2.0 ** (8 - b_r), -1.0, float("inf")):
        y, log = ops.round_and_log(torch.from_numpy(vals).cuda(), b_r, tau, out_dtype=torch.float64)
        assert np.array_equal(bits(y.cpu().numpy()), bits(oracle.rnd_array(vals, b_r)))
        want = oracle.sparse_from_codes(oracle.direction_array(vals, b_r, tau))
        assert np.array_equal(_sparse_np(log), want), tau


def test_host_pipeline_e2e(oracle):
    """The e2e path of bench.py (pinned host buffers, chunked H2D / kernels /
    D2H on three streams, log chunks chained through device cursors)."""
    import torch
    from paper_2403_09603_b200 import ops, workloads
    n = (1 << 21) + 12345
    xt, xa = workloads.config1_pair(n, 11)
    tau = workloads.TAU_CONFIG0
    xt_h = torch.from_numpy(xt).pin_memory()
    xa_h = torch.from_numpy(xa).pin_memory()
    yt_h = torch.empty(n, dtype=torch.float32).pin_memory()
    ya_h = torch.empty(n, dtype=torch.float32).pin_memory()
    log_h = torch.empty(n // 4, dtype=torch.int64).pin_memory()
    count, corr, _ = ops.round_and_log_replay_host(xt_h, xa_h, 32, tau, yt_h, ya_h, log_h, global_base=777,
                                                   chunk=1 << 19)
    torch.cuda.synchronize()
    codes = oracle.direction_array(xt, 32, tau)
    want = oracle.sparse_from_codes(codes, base=777)
    assert count == want.size
    assert np.array_equal(log_h[:count].numpy().view(np.uint64), want)
    assert np.array_equal(bits(yt_h.numpy()), bits(oracle.rnd_array(xt, 32).astype(np.float32)))
    ya_want = oracle.rev_array(xa, 32, codes)
    assert np.array_equal(bits(ya_h.numpy()), bits(ya_want.astype(np.float32)))
    assert corr == int(np.count_nonzero(ya_want != oracle.rnd_array(xa, 32)))


@pytest.mark.slow
def test_large_properties():
    """2^27 elements: sortedness, count consistency, replay idempotence."""
    import torch
    from paper_2403_09603_b200 import ops, workloads
    n = 1 << 27
    x = workloads.config0_x_torch(n, 5)
    y, log = ops.round_and_log(x, 32, workloads.TAU_CONFIG0)
    idx = log.indices()
    assert bool((idx[1:] > idx[:-1]).all())
    assert 0.09 * n < log.count < 0.11 * n
    y2, corr = ops.replay(x, 32, log)
    assert corr == 0 and torch.equal(y.view(torch.int32), y2.view(torch.int32))
    assert torch.equal(y.view(torch.int32), x.float().view(torch.int32))  # b_r=32 is RNE to FP32


@pytest.mark.parametrize("b_r", list(range(10, 33)))
def test_every_grid_random_bit_patterns(oracle, fp, b_r):
    """Every b_r in [10, 32] (fpround.py:44-46): random FP64 BIT PATTERNS over
    the whole finite range below grid_max (FP64 subnormals, FP32-subnormal
    results, ties of the dropped bits, values at tau from the grid), through
    rnd / direction at three taus / grid neighbours / rev and the fused sparse
    round-and-log + replay, against the oracle bit for bit."""
    import torch

    from paper_2403_09603_b200 import ops
    rng = np.random.default_rng(7000 + b_r)
    n = 40_000
    raw = rng.integers(0, 1 << 63, size=n, dtype=np.uint64) | (rng.integers(0, 2, size=n, dtype=np.uint64) << 63)
    x = raw.view(np.float64)
    x = x[np.isfinite(x) & (np.abs(x) <= oracle.grid_max(b_r))]
    # exact ties and near-ties of the dropped bits on the normal FP32 range
    drop = 52 - (b_r - 9)
    base = rng.normal(size=2000)
    tb = (base.view(np.uint64) & ~np.uint64((1 << drop) - 1)) | np.uint64(1 << (drop - 1))
    ties = np.concatenate([tb.view(np.float64), np.nextafter(tb.view(np.float64), np.inf),
                           np.nextafter(tb.view(np.float64), -np.inf)])
    x = np.concatenate([x, ties, -ties, np.ldexp(rng.normal(size=500), -140), [0.0, -0.0]])
    lo, hi = oracle.tau_bounds(b_r)
    for tau in (0.0, lo, 0.5 * (lo + hi), hi):
        assert np.array_equal(fp.direction_array(x, b_r, tau), oracle.direction_array(x, b_r, tau)), tau
    assert np.array_equal(bits(fp.rnd_array(x, b_r)), bits(oracle.rnd_array(x, b_r)))
    glo, ghi = fp.grid_neighbors_array(x, b_r)
    wlo, whi = oracle.grid_neighbors_array(x, b_r)
    assert np.array_equal(bits(glo), bits(wlo)) and np.array_equal(bits(ghi), bits(whi))
    codes = rng.integers(0, 3, size=x.size).astype(np.uint8)
    assert np.array_equal(bits(fp.rev_array(x, b_r, codes)), bits(oracle.rev_array(x, b_r, codes)))
    # the fused sparse path, FP64 out (every grid value is exact in FP32 too)
    tau = 0.5 * (lo + hi)
    xd = torch.from_numpy(x).cuda()
    y, log = ops.round_and_log(xd, b_r, tau, out_dtype=torch.float64, global_base=3)
    want = oracle.direction_array(x, b_r, tau)
    assert np.array_equal(log.words.cpu().numpy().view(np.uint64), oracle.sparse_from_codes(want, base=3))
    assert np.array_equal(bits(y.cpu().numpy()), bits(oracle.rnd_array(x, b_r)))
    ya, corr = ops.replay(xd, b_r, log, out_dtype=torch.float64, global_base=3)
    assert np.array_equal(bits(ya.cpu().numpy()), bits(oracle.rev_array(x, b_r, want))) and corr == 0
