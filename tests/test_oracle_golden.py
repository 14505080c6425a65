"""Pin the CPU oracle to outputs of the real reference (tests/golden/*)."""

from __future__ import annotations

import hashlib
import zlib

import numpy as np
import pytest

from conftest import bits
from paper_2403_09603_b200 import workloads

B_VALUES = (10, 26, 29, 32)


@pytest.mark.parametrize("b_r", B_VALUES)
def test_fpround_matches_reference(golden, oracle, b_r):
    g = golden.fpround
    x = g[f"x_{b_r}"]
    assert np.array_equal(bits(oracle.rnd_array(x, b_r)), bits(g[f"rnd_{b_r}"]))
    lo, hi = oracle.grid_neighbors_array(x, b_r)
    assert np.array_equal(bits(lo), bits(g[f"below_{b_r}"]))
    assert np.array_equal(bits(hi), bits(g[f"above_{b_r}"]))
    assert np.array_equal(bits(oracle.exponent_scale_array(x)), bits(g[f"scale_{b_r}"]))
    assert np.array_equal(oracle.is_on_grid(x, b_r), g[f"ongrid_{b_r}"])
    assert np.array_equal(bits(oracle.rev_array(x, b_r, g[f"codes_{b_r}"])), bits(g[f"rev_{b_r}"]))
    for i, t in enumerate(g[f"taus_{b_r}"]):
        d = oracle.direction_array(x, b_r, float(t))
        assert np.array_equal(d, g[f"dir_{b_r}_{i}"]), (b_r, t)
        assert np.array_equal(bits(oracle.rev_array(x, b_r, d)), bits(g[f"revdir_{b_r}_{i}"]))


def _call(oracle, case):
    x = np.array([float.fromhex(v) for v in case["x"]])
    fn, b_r = case["fn"], case["b_r"]
    if fn == "rnd_array":
        return oracle.rnd_array(x, b_r)
    if fn == "grid_neighbors_array":
        return oracle.grid_neighbors_array(x, b_r)
    if fn == "rev_array":
        return oracle.rev_array(x, b_r, np.ones(x.shape, np.uint8))
    if fn == "direction_array":
        return oracle.direction_array(x, b_r, 2.0 ** -25)
    if fn == "exponent_scale_array":
        return oracle.exponent_scale_array(x)
    if fn.startswith("rev_array_badcode"):
        return oracle.rev_array(x, b_r, np.full(x.shape, 3, np.uint8))
    if fn == "rev_array_shape":
        return oracle.rev_array(x, b_r, np.ones(3, np.uint8))
    raise AssertionError(fn)


def test_error_semantics_match_reference(golden, oracle):
    for case in golden.errors:
        if case["error"] is None:
            _call(oracle, case)
        else:
            with pytest.raises(ValueError) as ei:
                _call(oracle, case)
            assert str(ei.value) == case["error"], case


def test_known_answers(oracle):
    # test_fpround.py:65-67, 153-162, 222-230 of the reference
    assert oracle.rnd_array(1.0 + 2.0 ** -24, 32)[0] == 1.0
    t = 0.25 * 2.0 ** -23
    assert oracle.direction_array(1.0 + 0.75 * 2.0 ** -23, 32, t)[0] == 1
    assert oracle.direction_array(1.0 + 0.6 * 2.0 ** -23, 32, t)[0] == 2
    assert oracle.direction_array(1.0 + 0.4 * 2.0 ** -23, 32, t)[0] == 0
    assert oracle.rev_array(1.0 + 0.4 * 2.0 ** -23, 32, [2])[0] == 1.0 + 2.0 ** -23
    assert oracle.rev_array(1.0 + 0.6 * 2.0 ** -23, 32, [0])[0] == 1.0
    assert bits(oracle.rnd_array(-(2.0 ** -151), 32))[0] == bits(np.array([-0.0]))[0]


def test_roundlog_matches_reference(golden, oracle):
    for i, case in enumerate(golden.roundlog["cases"]):
        digits = golden.roundlog_digits[f"d{i}"]
        assert hashlib.sha256(digits.tobytes()).hexdigest() == case["digits_sha"]
        chunks, prev = [], 0
        for c in case["cuts"] + [case["n"]]:
            chunks.append(digits[prev:c])
            prev = c
        raw = oracle.vtrl_bytes(chunks, case["b_r"], case["compress"])
        assert hashlib.sha256(raw).hexdigest() == case["file_sha"]
        assert len(raw) == case["file_len"]
        if case["compress"]:
            assert len(zlib.decompress(raw[15:])) == (case["n"] + 4) // 5
        if case["payload_hex"] is not None:
            assert raw[15:].hex() == case["payload_hex"]
        assert oracle.unpack_groups(oracle.pack_groups(
            np.concatenate([digits, np.ones((-digits.size) % 5, np.uint8)])))[: digits.size].tolist() == digits.tolist()
    for digs, val in golden.roundlog["known"]["pack5"]:
        assert oracle.pack_groups(digs) == bytes([val])
    for b, digs in golden.roundlog["known"]["unpack5"]:
        assert oracle.unpack_groups(bytes([b])).tolist() == digs
    with pytest.raises(ValueError, match="corrupt log byte"):
        oracle.unpack_groups(bytes([243]))


def test_sparse_roundtrip(oracle):
    rng = np.random.default_rng(5)
    codes = rng.integers(0, 3, size=10007).astype(np.uint8)
    w = oracle.sparse_from_codes(codes, base=12345)
    assert np.all(np.diff((w >> np.uint64(1)).astype(np.int64)) > 0)
    assert np.array_equal(oracle.codes_from_sparse(w, codes.size, base=12345), codes)


def test_search_tau_matches_reference(golden, oracle):
    for case in golden.tau["search_tau"]:
        s = [float.fromhex(v) for v in case["samples"]]
        assert oracle.search_tau(s, case["b_r"], case["iters"]).hex() == case["tau"]


def test_budget_tau_restatement(golden, oracle):
    for case in golden.tau["budget"]:
        x = np.random.default_rng(case["seed"]).normal(0.0, 10.0 ** case["sigma_exp"], size=case["n"])
        t = oracle.search_tau_budget(x, 32, case["budget"])
        assert t.hex() == case["tau"]
        assert int(np.count_nonzero(oracle.direction_array(x, 32, t) != 1)) == case["logged"]


def test_merkle_matches_reference(golden, oracle):
    for case in golden.merkle["build"]:
        leaves = [hashlib.sha256(f"leaf-{i}".encode()).digest() for i in range(case["n"])]
        levels = oracle.merkle_levels(leaves)
        assert [[d.hex() for d in lvl] for lvl in levels] == case["levels"]
    ch = golden.merkle["chunked"]
    w = np.random.default_rng(ch["seed"]).normal(0.0, 0.02, size=ch["n_params"]).astype(np.float32)
    levels = oracle.merkle_levels(oracle.chunk_leaves(w.astype("<f4").tobytes(), ch["leaf_bytes"]))
    assert [[d.hex() for d in lvl] for lvl in levels] == ch["levels"]
    assert oracle.hash_weights([]).hex() == golden.merkle["hash_weights"]["empty"]
    assert oracle.hash_weights([np.arange(6.0).reshape(2, 3)]).hex() == golden.merkle["hash_weights"]["arange"]


def test_sha256_known_answers(oracle):
    # FIPS 180-4 example vectors
    assert oracle.sha256(b"abc").hex() == "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
    assert oracle.sha256(b"").hex() == "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"
    assert oracle.sha256(b"abcdbcdecdefdefgefghfghighijhijkijkljklmklmnlmnomnopnopq").hex() == \
        "248d6a61d20638b8e5c026930c3e6039a33ce45964ff2167f6ecedd419db06c1"


def test_config_digests(golden, oracle):
    c0 = golden.configs["config0"]
    x = workloads.config0_x(c0["n"], c0["seed"])
    assert hashlib.sha256(x.tobytes()).hexdigest() == c0["x_sha"]
    tau = float.fromhex(c0["tau"])
    assert tau == workloads.TAU_CONFIG0
    r = oracle.rnd_array(x, 32)
    assert hashlib.sha256(r.astype(np.float32).tobytes()).hexdigest() == c0["rnd_f32_sha"]
    d = oracle.direction_array(x, 32, tau)
    assert hashlib.sha256(d.tobytes()).hexdigest() == c0["codes_sha"]
    assert hashlib.sha256(oracle.sparse_from_codes(d).tobytes()).hexdigest() == c0["sparse_sha"]
    c1 = golden.configs["config1"]
    xt, xa = workloads.config1_pair(c1["n"], c1["seed"])
    assert hashlib.sha256(xa.tobytes()).hexdigest() == c1["xa_sha"]
    ya = oracle.rev_array(xa, 32, oracle.direction_array(xt, 32, tau))
    assert hashlib.sha256(ya.astype(np.float32).tobytes()).hexdigest() == c1["auditor_f32_sha"]


def test_oracle_hash_weights_game_golden(oracle):
    """The oracle's hash_weights restatement against the reference's digests
    (merkle.py:155-166): FP64 pair, FP32 specials / overflow, FP32 input."""
    import json
    from conftest import GOLDEN
    hw = json.loads((GOLDEN / "merkle_game_golden.json").read_text())["hash_weights"]
    rng = np.random.default_rng(17)
    w1 = rng.normal(0.0, 0.02, size=(37, 41))
    w2 = rng.normal(0.0, 1.0, size=100_003)
    assert oracle.hash_weights([w1, w2]).hex() == hw["pair"]
    w3 = np.array([1e300, -1e300, 3.4028235e38, 1e-45, -0.0, 2.0 ** -149, 2.0 ** -150], dtype=np.float64)
    with np.errstate(over="ignore"):
        assert oracle.hash_weights([w3]).hex() == hw["specials"]
    assert oracle.hash_weights([w1.astype(np.float32)]).hex() == hw["f32_input"]
    bad = np.zeros(50, dtype=np.float64)
    bad[17] = np.inf
    with pytest.raises(ValueError) as e:
        oracle.hash_weights([w1, bad])
    assert str(e.value) == hw["nonfinite_error"]


@pytest.mark.parametrize("name", ["tiny", "logreg", "trend"])
def test_oracle_replays_reference_channel_traces(oracle, name):
    """The oracle restatement over the recorded channel calls of real
    reference runs: trainer outputs, directed counts and .vtrl bytes;
    auditor outputs and corrections (trend's prefix carries 77)."""
    import json
    from conftest import GOLDEN
    arr = np.load(GOLDEN / "channel_traces.npz")
    m = json.loads((GOLDEN / "channel_traces.json").read_text())[name]
    sizes = [int(np.prod(s)) for s in m["shapes"]]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    t_in, t_out = arr[f"{name}_t_in"], arr[f"{name}_t_out"]
    a_in, a_out = arr[f"{name}_a_in"], arr[f"{name}_a_out"]
    codes_all = []
    for i, tau in enumerate(m["taus"]):
        x = t_in[offs[i]:offs[i + 1]]
        c = oracle.direction_array(x, m["b_r"], tau)
        codes_all.append(c)
        assert np.array_equal(bits(oracle.rnd_array(x, m["b_r"]).astype(np.float32)), bits(t_out[offs[i]:offs[i + 1]]))
        assert int(np.count_nonzero(c != 1)) == m["directed"][i]
        xa = a_in[offs[i]:offs[i + 1]]
        ya = oracle.rev_array(xa, m["b_r"], c)
        assert np.array_equal(bits(ya.astype(np.float32)), bits(a_out[offs[i]:offs[i + 1]]))
        assert int(np.count_nonzero(ya != oracle.rnd_array(xa, m["b_r"]))) == m["corrections"][i]
    assert hashlib.sha256(oracle.vtrl_bytes(codes_all, m["b_r"])).hexdigest() == m["vtrl_sha"]
    if name == "trend":
        assert sum(m["corrections"]) == 77


def test_order_statistic_budget_search_equals_counting_search(oracle):
    """search_tau_budget_kth (np.partition, used at full BASELINE sizes) is the
    counting bisection of search_tau_budget, bit for bit, incl. budget >= n,
    budget 0, ties and magnitudes across the FP32 range."""
    from paper_2403_09603_b200 import workloads
    rng = np.random.default_rng(123)
    cases = [rng.normal(0, 10.0 ** s, size=n) for s, n in ((-3, 5000), (0, 20_001), (1, 777))]
    cases += [workloads.config0_x(30_000, 5), np.full(4096, 1.0 + 0.4 * 2.0 ** -23),
              (rng.integers(1 << 23, 1 << 24, size=3000) + 0.5) * 2.0 ** -23, np.zeros(0)]
    for b_r in (32, 26):
        for x in cases:
            for B in sorted({0, 1, 17, int(0.005 * x.size), x.size // 3, x.size, x.size + 5}):
                assert oracle.search_tau_budget_kth(x, b_r, B) == oracle.search_tau_budget(x, b_r, B), (b_r, x.size, B)


def test_parallel_oracle_driver(oracle):
    """vt_parallel (the chunked, all-cores driver of the full-size GPU parity
    tests) agrees with the sequential oracle, and detects a flipped bit."""
    import vt_parallel as P
    from paper_2403_09603_b200 import workloads
    n = 300_007
    xt, xa = workloads.config1_pair(n, 77)
    tau = workloads.TAU_CONFIG0
    codes = oracle.direction_array(xt, 32, tau)
    words = oracle.sparse_from_codes(codes, base=1000)
    yt = oracle.rnd_array(xt, 32).astype(np.float32)
    ya = oracle.rev_array(xa, 32, codes).astype(np.float32)
    r = P.check_round_and_log(xt, 32, tau, words, yt, xa, ya, base=1000, chunk=1 << 15, procs=4)
    assert r["n_log"] == r["words"] == words.size
    assert r["log_mismatches"] == r["yt_mismatches"] == r["ya_mismatches"] == 0
    assert r["corrections"] == int(np.count_nonzero(ya != oracle.rnd_array(xa, 32).astype(np.float32)))
    ya2 = ya.copy()
    ya2[123_456] = np.nextafter(ya2[123_456], np.float32(np.inf))
    words2 = words.copy()
    words2[5] ^= np.uint64(1)
    r2 = P.check_round_and_log(xt, 32, tau, words2, yt, xa, ya2, base=1000, chunk=1 << 15, procs=4)
    assert r2["ya_mismatches"] == 1 and r2["ya_first_bad"] == 123_456 and r2["log_mismatches"] == 1
    # exact top-k over chunks == the sequential order-statistic search
    xs = [np.random.default_rng(s).normal(0, 10.0 ** (s - 3), size=m) for s, m in ((1, 100_000), (2, 5), (3, 70_001))]
    Bs = [500, 5, 350]
    assert P.search_tau_budget_many(xs, 32, Bs, chunk=1 << 14, procs=4) == \
        [oracle.search_tau_budget(x, 32, B) for x, B in zip(xs, Bs)]
    # Merkle levels over all cores == merkle.build over the chunked leaves
    w = np.random.default_rng(4).normal(0, 0.02, size=1_000_003).astype(np.float32)
    lv = P.merkle_levels_bytes(w, 4096, procs=4)
    ref = oracle.merkle_levels(oracle.chunk_leaves(w.tobytes(), 4096))
    assert [b"".join(level) for level in ref] == lv
