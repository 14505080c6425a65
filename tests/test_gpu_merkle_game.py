"""GPU parity of the verification-game queries answered from device levels
(merkle.node / path / verify_path / first_divergence, reference
pkg/src/vtrain/merkle.py:75-152) and of the canonical checkpoint digest
merkle.hash_weights (merkle.py:155-166), against fixtures produced by the
real reference (tests/golden/make_golden.py: golden_merkle_game)."""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def game():
    return json.loads((GOLDEN / "merkle_game_golden.json").read_text())


@pytest.fixture(scope="module")
def mk():
    from paper_2403_09603_b200 import merkle
    return merkle


def _leaves(case):
    return [hashlib.sha256(f"{case['seed_tag']}-{i}".encode()).digest() for i in range(case["n"])]


def test_node_and_path(game, mk):
    for case in game["trees"]:
        t = mk.build(_leaves(case))
        for lv, ix, want in case["nodes"]:
            assert mk.node(t, lv, ix).hex() == want
        for p in case["paths"]:
            got = mk.path(t, p["leaf_index"])
            assert got.leaf.hex() == p["leaf"]
            assert [[d.hex(), side] for d, side in got.siblings] == p["siblings"]
            assert mk.verify_path(got, t.root) == p["verifies"]
            assert not mk.verify_path(got, hashlib.sha256(b"other").digest())


def test_first_divergence(game, mk):
    for case in game["trees"]:
        t = mk.build(_leaves(case))
        assert mk.first_divergence(t, mk.build(_leaves(case))) is None
        for d in case["divergence"]:
            other = mk.build([bytes.fromhex(h) for h in d["other"]])
            assert mk.first_divergence(t, other) == d["first"]
    a = mk.build(_leaves(game["trees"][3]))
    with pytest.raises(ValueError, match="checkpoint schedule mismatch"):
        mk.first_divergence(a, mk.build(_leaves(game["trees"][4])))


def test_query_errors(game, mk):
    t3 = mk.build([hashlib.sha256(b"e%d" % i).digest() for i in range(3)])
    with pytest.raises(IndexError) as e:
        mk.node(t3, 5, 0)
    assert str(e.value) == game["errors"]["level"]
    with pytest.raises(IndexError) as e:
        mk.node(t3, 1, 2)
    assert str(e.value) == game["errors"]["index"]
    with pytest.raises(IndexError) as e:
        mk.path(t3, 3)
    assert str(e.value) == game["errors"]["path"]


def test_paths_on_chunked_tree(oracle, mk):
    """Paths of the 4 KiB-chunk checkpoint tree verify against its root and
    match the oracle's levels (the game's leaf queries on a device tree)."""
    w = np.random.default_rng(4).normal(0, 0.02, size=300_001).astype(np.float32)
    tree = mk.merkle_chunked(w)
    levels = oracle.merkle_levels(oracle.chunk_leaves(w.tobytes(), 4096))
    assert tree.root == levels[-1][0]
    for li in (0, 1, 146, len(levels[0]) - 1):
        p = mk.path(tree, li)
        assert p.leaf == levels[0][li]
        assert mk.verify_path(p, levels[-1][0])


def test_hash_weights_golden(game, mk, golden):
    import torch
    hw = game["hash_weights"]
    rng = np.random.default_rng(17)
    w1 = rng.normal(0.0, 0.02, size=(37, 41))
    w2 = rng.normal(0.0, 1.0, size=100_003)
    assert hashlib.sha256(w1.tobytes()).hexdigest() == hw["w1_sha"]
    assert hashlib.sha256(w2.tobytes()).hexdigest() == hw["w2_sha"]
    assert mk.hash_weights([w1, w2]).hex() == hw["pair"]
    # device tensors in, small chunks (the pipelined path crosses tensor and chunk edges)
    assert mk.hash_weights([torch.from_numpy(w1).cuda(), torch.from_numpy(w2).cuda()], chunk=4096).hex() == hw["pair"]
    w3 = np.array([1e300, -1e300, 3.4028235e38, 1e-45, -0.0, 2.0 ** -149, 2.0 ** -150], dtype=np.float64)
    assert mk.hash_weights([w3]).hex() == hw["specials"]  # overflow -> inf, FP32 subnormals, -0.0
    assert mk.hash_weights([w1.astype(np.float32)]).hex() == hw["f32_input"]
    assert mk.hash_weights([]).hex() == golden.merkle["hash_weights"]["empty"]
    assert mk.hash_weights([np.arange(6, dtype=np.float64).reshape(2, 3)]).hex() == \
        golden.merkle["hash_weights"]["arange"]


def test_hash_weights_errors(game, mk):
    hw = game["hash_weights"]
    rng = np.random.default_rng(17)
    w1 = rng.normal(0.0, 0.02, size=(37, 41))
    bad = np.zeros(50, dtype=np.float64)
    bad[17] = np.inf
    bad[31] = np.nan
    with pytest.raises(ValueError) as e:
        mk.hash_weights([w1, bad])
    assert str(e.value) == hw["nonfinite_error"]
    with pytest.raises(ValueError) as e:  # the first bad index survives chunking
        mk.hash_weights([w1, bad], chunk=16)
    assert str(e.value) == hw["nonfinite_error"]
    with pytest.raises(ValueError) as e:
        mk.hash_weights([w1], b_m=16)
    assert str(e.value) == hw["b_m_error"]


def test_hash_weights_large_vs_oracle(oracle, mk):
    """Tens of millions of parameters over several chunks vs the reference
    restatement (hashlib over numpy's astype('<f4'))."""
    import torch
    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    ws = [torch.randn(n, dtype=torch.float64, device="cuda", generator=g) * 0.05
          for n in (5_000_000, 17, 3 * (1 << 22) + 5)]
    want = oracle.hash_weights([w.cpu().numpy() for w in ws])
    assert mk.hash_weights(ws, chunk=1 << 22) == want
