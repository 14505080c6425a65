"""The multi-GPU path of paper_2403_09603_b200/dist.py on a real NCCL
communicator (one rank: this pool's boxes have one GPU, and NCCL does not
put two ranks on one device).  The collectives -- the count all-gather, the
Merkle block-root all-gather, the corrections all-reduce -- run through
NCCL here; their multi-rank arithmetic is covered by the world-size-2 gloo
tests (tests/test_dist_gloo.py).  Results must equal the single-device
operators bit for bit."""

from __future__ import annotations

import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    import torch
    import torch.distributed as dist
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


def test_sharded_round_and_log_replay_nccl(nccl_group):
    import torch
    from paper_2403_09603_b200 import dist as vdist
    from paper_2403_09603_b200 import ops, workloads
    n = (1 << 20) + 777
    xt, xa = workloads.config1_pair_torch(n, seed=4, device=torch.device("cuda"))
    lo, hi = vdist.shard_range(n, 0, 1)
    assert (lo, hi) == (0, n)
    base = 5 * n
    y, slog = vdist.round_and_log_sharded(xt, 32, workloads.TAU_CONFIG0, base, group=nccl_group)
    y1, log1 = ops.round_and_log(xt, 32, workloads.TAU_CONFIG0, global_base=base)
    assert torch.equal(y.view(torch.int32), y1.view(torch.int32))
    assert torch.equal(slog.local.words, log1.words)
    assert slog.offset == 0 and slog.total == log1.count and slog.counts.tolist() == [log1.count]
    ya, corr = vdist.replay_sharded(xa, 32, slog, base, group=nccl_group)
    ya1, corr1 = ops.replay(xa, 32, log1, global_base=base)
    assert torch.equal(ya.view(torch.int32), ya1.view(torch.int32)) and corr == corr1
    assert torch.equal(ya.view(torch.int32), y.view(torch.int32))


def test_sharded_budget_search_nccl(nccl_group, oracle):
    import torch
    from paper_2403_09603_b200 import dist as vdist
    x = np.random.default_rng(12).normal(0.0, 3.0, 400_003)
    B = int(0.005 * x.size)
    tau = vdist.search_tau_budget_sharded(torch.from_numpy(x).cuda(), 32, B, group=nccl_group)
    assert tau == oracle.search_tau_budget(x, 32, B)


def test_merkle_sharded_nccl(nccl_group):
    import torch
    from paper_2403_09603_b200 import dist as vdist
    from paper_2403_09603_b200 import merkle
    g = torch.Generator(device="cuda")
    g.manual_seed(9)
    w = torch.randn(3 * (1 << 20) + 12345, dtype=torch.float32, device="cuda", generator=g) * 0.02
    b = w.view(torch.uint8)
    n_leaves = (b.numel() + 4095) // 4096
    lv, top = vdist.merkle_sharded(b, n_leaves, group=nccl_group, k=8)
    ref = merkle.merkle_chunked(w)
    assert bytes(top[-1][0].cpu().numpy()) == ref.root


def test_count_exchange_over_symmetric_memory(nccl_group):
    """The count exchange fused into the round-and-log kernel (last CTA ->
    every rank's symmetric-memory buffer; wait kernel) equals the NCCL
    all-gather, over repeated calls of varying size (the sequence number and
    slot parity advance), graph-captured as well."""
    import torch
    from paper_2403_09603_b200 import dist as vdist
    from paper_2403_09603_b200 import ops, workloads
    ex = vdist.CountExchange(nccl_group)
    for i, n in enumerate((5_000, (1 << 20) + 3, 70_001, 1 << 22, 640)):
        x = workloads.config0_x_torch(n, 50 + i)
        y, slog = vdist.round_and_log_sharded(x, 32, workloads.TAU_CONFIG0, 7 * n, group=nccl_group, exchange=ex)
        y1, log1 = ops.round_and_log(x, 32, workloads.TAU_CONFIG0, global_base=7 * n)
        assert slog.counts.tolist() == [log1.count] and slog.total == log1.count, i
        assert torch.equal(slog.local.words, log1.words) and torch.equal(y.view(torch.int32), y1.view(torch.int32))
    assert int(ex.buf[0].item()) == 5  # five exchanges, five sequence numbers
    # an empty shard still takes part: it publishes a count of 0
    p = ex.round_and_log(torch.empty(0, dtype=torch.float64, device="cuda"), 32, workloads.TAU_CONFIG0, 0)
    assert ex.wait().tolist() == [0] and p.finish()[1].count == 0
    ex.check()
    assert int(ex.buf[0].item()) == 6
    # graph-captured: the fused kernel + the wait kernel replayed
    n = 1 << 21
    x = workloads.config0_x_torch(n, 60)
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    words = torch.empty(n // 4, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    state = {}

    def step():
        state["p"] = ex.round_and_log(x, 32, workloads.TAU_CONFIG0, 0, out=y, log_out=words)
        state["c"] = ex.wait()

    with torch.cuda.stream(s):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    _, log1 = ops.round_and_log(x, 32, workloads.TAU_CONFIG0)
    assert state["c"].tolist() == [log1.count]
    ex.check()
    assert int(ex.buf[0].item()) == 6 + 1 + 3  # warm-up call, then 3 replays (capture runs nothing)



def test_digest_exchange_over_symmetric_memory(nccl_group):
    """merkle_sharded with the block roots over peer memory (the level kernel
    publishes them) equals the NCCL all-gather path and merkle_chunked."""
    import torch
    from paper_2403_09603_b200 import dist as vdist
    from paper_2403_09603_b200 import merkle
    g = torch.Generator(device="cuda")
    g.manual_seed(19)
    w = torch.randn(5 * (1 << 20) + 4321, dtype=torch.float32, device="cuda", generator=g)
    b = w.view(torch.uint8)
    n_leaves = (b.numel() + 4095) // 4096
    n_blocks = (n_leaves + (1 << 8) - 1) >> 8
    ex = vdist.DigestExchange(n_blocks, nccl_group)
    for _ in range(3):
        lv, top = vdist.merkle_sharded(b, n_leaves, group=nccl_group, k=8, exchange=ex)
    lv2, top2 = vdist.merkle_sharded(b, n_leaves, group=nccl_group, k=8)
    assert all(torch.equal(a, c) for a, c in zip(top, top2))
    assert bytes(top[-1][0].cpu().numpy()) == merkle.merkle_chunked(w).root
    ex.check()
    assert int(ex.buf[0].item()) == 3


def test_budget_exchange_over_symmetric_memory(nccl_group, oracle):
    """The sharded budget search with both exchanges over peer memory and
    the decision on the device equals the oracle (and the NCCL path)."""
    import torch
    from paper_2403_09603_b200 import dist as vdist
    ex = vdist.BudgetExchange(nccl_group)
    rng = np.random.default_rng(21)
    for k in range(3):
        x = rng.normal(0.0, 3.0, 400_003 + 11 * k)
        B = int(0.005 * x.size)
        xt = torch.from_numpy(x).cuda()
        tau = vdist.search_tau_budget_sharded(xt, 32, B, group=nccl_group, exchange=ex)
        assert tau == oracle.search_tau_budget(x, 32, B) == vdist.search_tau_budget_sharded(xt, 32, B,
                                                                                              group=nccl_group)
    assert int(ex.buf[0].item()) == 3
