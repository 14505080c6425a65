"""Host-side multi-GPU plans (no GPU): LPT assignment of independent
tensors for the adaptive threshold (SURVEY.md §8e, configs[2])."""

from __future__ import annotations

import numpy as np


def test_lpt_assign_balances_resnet_tensors():
    from paper_2403_09603_b200 import dist as vd, workloads
    sizes = [int(np.prod(s)) for _, s in workloads.resnet50_tensors()]
    for world in (1, 2, 4, 8):
        owner = vd.lpt_assign(sizes, world)
        assert len(owner) == len(sizes) and set(owner) <= set(range(world))
        loads = np.bincount(owner, weights=sizes, minlength=world)
        assert loads.sum() == sum(sizes)
        # LPT: the heaviest rank exceeds the ideal split by at most one tensor
        assert loads.max() <= sum(sizes) / world + max(sizes)
        assert owner == vd.lpt_assign(sizes, world)  # deterministic


def test_lpt_assign_small_cases():
    from paper_2403_09603_b200 import dist as vd
    assert vd.lpt_assign([], 3) == []
    assert vd.lpt_assign([5], 4) == [0]
    assert vd.lpt_assign([3, 3, 2, 2, 2], 2) == [0, 1, 0, 1, 0]


def test_sharded_budget_decision_logic_on_host():
    """The host half of the sharded budget search (ShardedBudget.decide /
    finish, the plan from vt_tau_shard_plan) on exchange buffers built here
    from oracle keys split over 3 virtual ranks: the bisected tau equals the
    oracle's budget search.  The device half is tested on the GPU."""
    import ctypes as C
    import sys
    from conftest import REPO
    sys.path.insert(0, str(REPO / "oracle"))
    import vt_oracle as O
    from paper_2403_09603_b200 import _lib
    from paper_2403_09603_b200 import dist as vd

    rng = np.random.default_rng(5)
    x = rng.normal(0.0, 2.0, 120_001)
    n = x.size
    keys = O.normalized_distance(x, 32).view(np.uint64)
    hi_key = int(np.array([2.0 ** -24]).view(np.uint64)[0])
    for B in (0, 7, int(0.005 * n), 3_000):
        L, s0 = C.c_uint64(0), C.c_int(0)
        _lib.call("vt_tau_shard_plan", n, 32, B, C.byref(L), C.byref(s0))
        L, s0 = int(L.value), int(s0.value)
        cand = keys[keys > np.uint64(L)]
        xsum = np.zeros(vd.SHARD_XWORDS, dtype=np.int64)
        inr = cand[cand <= np.uint64(hi_key)]
        np.add.at(xsum, ((inr - np.uint64(L + 1)) >> np.uint64(s0)).astype(np.int64), 1)
        xsum[vd.SHARD_BINS] = int(np.count_nonzero(cand > np.uint64(hi_key)))
        xsum[vd.SHARD_BINS + 1] = cand.size
        sb = vd.ShardedBudget.__new__(vd.ShardedBudget)
        sb.b_r, sb.n_global, sb.budget, sb.L_key, sb.s0, sb.digit_count = 32, n, B, L, s0, 0

        class _NoFlags:
            @staticmethod
            def read():
                return 0, [0, 0, 0, 0]

        class _D:
            @staticmethod
            def raise_fpround(err):
                assert err == 0

        sb.flags, sb.D = _NoFlags, _D
        kind, val, rank = sb.decide(xsum)
        assert kind == "digit", (B, kind)
        parts = np.array_split(inr[((inr - np.uint64(L + 1)) >> np.uint64(s0)) == np.uint64(val)], 3)
        assert sum(p.size for p in parts) == sb.digit_count
        v = vd.ShardedBudget.finish(np.concatenate(parts).view(np.int64), rank)
        assert vd._bisect_tau(v, 32, 30) == O.search_tau_budget(x, 32, B), B
