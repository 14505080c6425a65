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
