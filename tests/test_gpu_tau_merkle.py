"""GPU parity: threshold search (reference + budget forms) and SHA-256 Merkle."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu


def test_search_tau_golden(golden):
    from paper_2403_09603_b200 import protocol
    for case in golden.tau["search_tau"]:
        s = [float.fromhex(v) for v in case["samples"]]
        assert protocol.search_tau(s, case["b_r"], case["iters"]).hex() == case["tau"]


def test_search_tau_nan_and_limits():
    from paper_2403_09603_b200 import protocol
    lo, hi = 0.25 * 2.0 ** -23, 0.5 * 2.0 ** -23
    assert protocol.search_tau([], 32, 30) == hi
    d = 0.4 * 2.0 ** -23
    assert abs(protocol.search_tau([d], 32, 40) - d) <= (hi - lo) * 2.0 ** -39
    assert abs(protocol.search_tau([1.0], 32, 40) - hi) <= (hi - lo) * 2.0 ** -39
    assert protocol.search_tau([float("nan"), 1.0], 32, 10) == \
        __import__("vt_oracle").search_tau([float("nan"), 1.0], 32, 10)


def test_budget_golden(golden):
    from paper_2403_09603_b200 import fpround, protocol
    for case in golden.tau["budget"]:
        x = np.random.default_rng(case["seed"]).normal(0.0, 10.0 ** case["sigma_exp"], size=case["n"])
        t = protocol.search_tau_budget(x, 32, case["budget"])
        assert t.hex() == case["tau"]
        assert int(np.count_nonzero(fpround.direction_array(x, 32, t) != 1)) == case["logged"]


@pytest.mark.parametrize("b_r", (26, 32))
def test_kth_largest_vs_sort(oracle, b_r):
    from paper_2403_09603_b200 import protocol
    rng = np.random.default_rng(b_r)
    x = np.concatenate([rng.normal(size=250_000) * np.exp2(rng.integers(-60, 60, size=250_000)),
                        rng.normal(size=3000) * 1e-40, np.zeros(50), rng.normal(size=2000).astype(np.float32)])
    p = np.sort(oracle.normalized_distance(x, b_r))[::-1]
    for rank in (0, 1, 7, 1250, 100_000, x.size - 1, x.size - 60, x.size + 5):
        want = p[rank] if rank < x.size else 0.0
        assert protocol.kth_largest_distance(x, b_r, rank) == want, rank


def test_budget_matches_oracle_random(oracle):
    from paper_2403_09603_b200 import protocol
    for seed in range(4):
        rng = np.random.default_rng(50 + seed)
        n = int(rng.integers(1000, 300_000))
        x = rng.normal(0.0, 10.0 ** rng.uniform(-3, 1), size=n)
        B = int(0.005 * n)
        assert protocol.search_tau_budget(x, 32, B) == oracle.search_tau_budget(x, 32, B)


def test_budget_key_clamps_and_fallback(oracle):
    """Both early exits (v above / below the bisection range) and the exact
    fallback when one digit holds more candidates than the buffer."""
    from paper_2403_09603_b200 import protocol
    lo, hi = oracle.tau_bounds(32)
    # all p identical (2^21 copies of one value): the selected digit overflows
    x = np.full(1 << 21, 1.0 + 0.4 * 2.0 ** -23)
    x[::3] = 1.0 + 0.45 * 2.0 ** -23
    for B in (0, 5000, 700_000, 699_050):
        assert protocol.search_tau_budget(x, 32, B) == oracle.search_tau_budget(x, 32, B), B
    # every p below tau_lo (values near the grid): v <= tau_lo
    y = 1.0 + np.random.default_rng(1).uniform(0, 0.2, size=100_000) * 2.0 ** -23
    assert protocol.search_tau_budget(y, 32, 10) == oracle.search_tau_budget(y, 32, 10)
    # many p at the top (near midpoints): v > tau_hi impossible (p <= 2^-24) but
    # exactly-tied midpoints sit at p == tau_hi
    z = (np.random.default_rng(2).integers(1 << 23, 1 << 24, size=100_000) + 0.5) * 2.0 ** -23
    for B in (0, 10, 99_999):
        assert protocol.search_tau_budget(z, 32, B) == oracle.search_tau_budget(z, 32, B), B
    assert protocol.budget_key(z, 32, 10) == hi


def test_round_and_log_adaptive_matches_host_search(oracle):
    """Device bisection + fused round-and-log == oracle budget search, then
    oracle direction codes at that tau (log <= budget)."""
    import torch
    from paper_2403_09603_b200 import ops, workloads
    cases = [np.random.default_rng(60).normal(0, 10.0 ** -2.5, size=200_003),
             np.random.default_rng(61).normal(0, 3.0, size=4096 * 3 + 5),
             workloads.config0_x(100_000, 62)]
    for x in cases:
        B = int(0.005 * x.size)
        y, log, tau = ops.round_and_log_adaptive(torch.from_numpy(x).cuda(), 32, B)
        t_or = oracle.search_tau_budget(x, 32, B)
        assert tau == t_or
        codes = oracle.direction_array(x, 32, t_or)
        assert np.array_equal(log.words.cpu().numpy().view(np.uint64), oracle.sparse_from_codes(codes))
        assert log.count <= B
        assert np.array_equal(bits(y.cpu().numpy()), bits(oracle.rnd_array(x, 32).astype(np.float32)))


@pytest.mark.parametrize("b_r", (26, 32))
def test_straddle_threshold_vs_oracle(oracle, b_r):
    """§8f3: threshold_search's sample reduction on the device."""
    from paper_2403_09603_b200 import protocol
    rng = np.random.default_rng(70 + b_r)
    n = 300_000
    y1 = rng.normal(size=n) * np.exp2(rng.integers(-12, 4, size=n))
    # a second "profile": reduction-order noise ~2^-7 of the grid spacing
    y2 = y1 + y1 * rng.uniform(-1.0, 1.0, size=n) * 2.0 ** (2 - b_r)
    s = oracle.straddle_samples(y1, y2, b_r)
    m, count, nan = protocol.straddle_min(y1, y2, b_r)
    assert count == len(s) > 0 and not nan
    assert m == min(s)
    for iters in (1, 10, 30):
        assert protocol.threshold_from_outputs(y1, y2, b_r, iters) == oracle.search_tau(s, b_r, iters)
    assert protocol.threshold_from_outputs(y1, y1, b_r, 10) == oracle.tau_bounds(b_r)[1]


def test_normalized_distance(oracle):
    import torch
    from paper_2403_09603_b200 import ops
    rng = np.random.default_rng(9)
    x = rng.normal(size=100_000) * np.exp2(rng.integers(-140, 40, size=100_000))
    got = ops.normalized_distance(torch.from_numpy(x).cuda(), 32).cpu().numpy()
    assert np.array_equal(got.view(np.uint64), oracle.normalized_distance(x, 32).view(np.uint64))


# ---------------------------------------------------------------------------
# Merkle
# ---------------------------------------------------------------------------

def test_build_golden(golden):
    from paper_2403_09603_b200 import merkle
    for case in golden.merkle["build"]:
        leaves = [hashlib.sha256(f"leaf-{i}".encode()).digest() for i in range(case["n"])]
        t = merkle.build(leaves)
        assert [[d.hex() for d in lvl] for lvl in t.levels] == case["levels"]
    with pytest.raises(ValueError):
        merkle.build([])
    with pytest.raises(ValueError):
        merkle.build([b"short"])


def test_chunked_golden(golden):
    from paper_2403_09603_b200 import merkle
    ch = golden.merkle["chunked"]
    w = np.random.default_rng(ch["seed"]).normal(0.0, 0.02, size=ch["n_params"]).astype(np.float32)
    t = merkle.merkle_chunked(w, ch["leaf_bytes"])
    assert [[d.hex() for d in lvl] for lvl in t.levels] == ch["levels"]


@pytest.mark.parametrize("leaf_bytes", [64, 100, 4096, 4097, 1 << 16])
def test_sha256_leaves_vs_hashlib(oracle, leaf_bytes):
    from paper_2403_09603_b200 import merkle
    rng = np.random.default_rng(leaf_bytes)
    for nbytes in (1, 55, 56, 63, 64, 65, 119, 120, 4095, 4096, 4097, 3 * leaf_bytes + 17, 300_001):
        data = rng.integers(0, 256, size=nbytes, dtype=np.uint8).tobytes()
        got = merkle.sha256_leaves(data, leaf_bytes).cpu().numpy()
        want = oracle.chunk_leaves(data, leaf_bytes)
        assert [bytes(r) for r in got] == want, (leaf_bytes, nbytes)


def test_sha256_known_answers():
    from paper_2403_09603_b200 import merkle
    assert bytes(merkle.sha256_leaves(b"abc", 64).cpu().numpy()[0]).hex() == \
        "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
    msg = b"abcdbcdecdefdefgefghfghighijhijkijkljklmklmnlmnomnopnopq"
    assert bytes(merkle.sha256_leaves(msg, 1024).cpu().numpy()[0]).hex() == \
        "248d6a61d20638b8e5c026930c3e6039a33ce45964ff2167f6ecedd419db06c1"


def test_chunked_tree_vs_oracle_random(oracle):
    from paper_2403_09603_b200 import merkle
    rng = np.random.default_rng(77)
    for n_params in (1, 1023, 1024, 1025, 5 * 1024 + 3, 777_777):
        w = rng.normal(0, 0.02, size=n_params).astype(np.float32)
        t = merkle.merkle_chunked(w)
        want = oracle.merkle_levels(oracle.chunk_leaves(w.tobytes(), 4096))
        assert t.levels == want, n_params
        assert t.root == want[-1][0]


def test_sharded_budget_search_virtual_ranks(oracle):
    """§8e: one tensor split over ranks.  Three virtual ranks in one process
    run the per-pass histograms, their sum stands in for the all-reduce, and
    every rank's selection must give the single-device order statistic and
    the oracle's budget tau."""
    import torch
    from paper_2403_09603_b200 import dist as vd, protocol
    x = np.random.default_rng(90).normal(0.0, 0.4, size=250_001)
    x[::7] = np.round(x[::7] * 1000) / 1000  # some near-grid mass
    cuts = [0, 61_000, 190_017, x.size]
    shards = [torch.from_numpy(x[a:b].copy()).cuda() for a, b in zip(cuts, cuts[1:])]
    for B in (0, 1_250, 40_000):
        ks = [vd.ShardedKth(s, 32, tag=f"kth_v{r}") for r, s in enumerate(shards)]
        for k in ks:
            k.begin(B)
        for p in range(vd.ShardedKth.PASSES):
            hs = [k.local_hist(p) for k in ks]
            total = sum(h.to(torch.int64) for h in hs).to(torch.int32)
            for h in hs:
                h.copy_(total)
            for k in ks:
                k.select(p)
        vals = [k.value() for k in ks]
        want = protocol.kth_largest_distance(x, 32, B)
        assert all(v == want for v in vals), (B, vals, want)
        lower, upper = oracle.tau_bounds(32)
        for _ in range(30):
            t = (lower + upper) / 2.0
            if vals[0] <= t:
                upper = t
            else:
                lower = t
        assert upper == oracle.search_tau_budget(x, 32, B)
    # world of one: the sharded entry point equals the single-device search
    assert vd.search_tau_budget_sharded(torch.from_numpy(x).cuda(), 32, 1_250) == oracle.search_tau_budget(x, 32, 1_250)


def test_sharded_candidate_budget_search_virtual_ranks(oracle):
    """The candidate path over a tensor cut into uneven shards (virtual ranks
    on one GPU; the all-reduce is a sum of the exchange buffers, the
    all-gather a concatenation): tau equals the oracle's budget search for
    ordinary budgets, zero, a budget of 40% (candidate overflow -> the exact
    multi-pass fallback), a tensor of ties, values near the grid (v <= tau_lo)
    and an empty shard."""
    import torch
    from paper_2403_09603_b200 import dist as vd
    rng = np.random.default_rng(21)
    cases = [rng.normal(0.0, 3.0, 400_003), np.full(300_000, 1.0 + 0.4 * 2.0 ** -23),
             1.0 + rng.uniform(0, 0.2, size=200_000) * 2.0 ** -23,
             (rng.integers(1 << 23, 1 << 24, size=150_000) + 0.5) * 2.0 ** -23]
    cases[1][::3] = 1.0 + 0.45 * 2.0 ** -23
    for ci, x in enumerate(cases):
        n = x.size
        cuts = [0, n // 7, n // 7, n // 2 + 3, n]  # the second shard is empty
        shards = [torch.from_numpy(x[a:b].copy()).cuda() for a, b in zip(cuts, cuts[1:])]
        for B in (0, 1, int(0.005 * n), int(0.4 * n)):
            sbs = [vd.ShardedBudget(s, 32, n, B, tag=f"sb{r}") for r, s in enumerate(shards)]
            xsum = sum(sb.candidates() for sb in sbs)
            decisions = [sb.decide(xsum.cpu().numpy()) for sb in sbs]
            assert all(d[:2] == decisions[0][:2] for d in decisions)
            kind, val, rank = decisions[0]
            if kind == "value":
                v = val
            elif kind == "digit":
                keys = torch.cat([sb.digit_keys(val) for sb in sbs])
                assert keys.numel() == sbs[0].digit_count
                v = vd.ShardedBudget.finish(keys.cpu().numpy(), rank)
            else:
                v = protocol_kth(x, B)
            want = oracle.search_tau_budget(x, 32, B)
            assert vd._bisect_tau(v, 32, 30) == want, (ci, B, kind)
            if kind == "digit":  # the exact order statistic itself
                assert v == oracle.kth_largest(oracle.normalized_distance(x, 32), B), (ci, B)
    # the entry point on one process equals the single-device search
    x = cases[0]
    for B in (0, 2_000, int(0.4 * x.size)):
        assert vd.search_tau_budget_sharded(torch.from_numpy(x).cuda(), 32, B) == oracle.search_tau_budget(x, 32, B)


def protocol_kth(x, B):
    from paper_2403_09603_b200 import protocol
    return protocol.kth_largest_distance(x, 32, B)
