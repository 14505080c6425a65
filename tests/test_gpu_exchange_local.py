"""The peer-memory count exchange (dist.CountExchange) in a single process,
without a process group: the one-rank case on a plain device buffer."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu


def test_count_exchange_single_process():
    """Without a process group the exchange is the one-rank case (its own buffer)."""
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("a process group is active in this session")
    import torch
    from paper_2403_09603_b200 import dist as vdist
    from paper_2403_09603_b200 import ops, workloads
    ex = vdist.CountExchange()
    x = workloads.config0_x_torch(300_000, 70)
    y, slog = vdist.round_and_log_sharded(x, 32, workloads.TAU_CONFIG0, 0, exchange=ex)
    assert slog.counts.tolist() == [ops.round_and_log(x, 32, workloads.TAU_CONFIG0)[1].count]
    assert torch.equal(y.view(torch.int32), ops.round_and_log(x, 32, workloads.TAU_CONFIG0)[0].view(torch.int32))
