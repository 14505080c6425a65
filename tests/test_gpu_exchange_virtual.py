"""The peer-memory count exchange with several ranks on ONE GPU, without
kernels that wait on one another: W virtual ranks, each with its own
exchange buffer (plain device memory standing in for the symmetric-memory
mapping), drive vt_round_log_exchange / vt_counts_wait on one stream in an
order where every wait is enqueued only after the publishes it needs, so no
kernel ever spins on work that has not already run (B200_PROFILING.md: no
mutually waiting ranks on one GPU).  This checks the multi-rank protocol
itself -- slot parity, sequence tags, every rank's counts in rank order, a
rank one exchange ahead of a peer, an empty shard -- bit for bit against
the single-device operator; tests/test_dist_gloo.py covers the process-group
plumbing, tests/test_gpu_dist_nccl.py the symmetric-memory buffer."""

from __future__ import annotations

import pytest

pytestmark = pytest.mark.gpu

W = 4


class _VirtualRanks:
    def __init__(self, world: int):
        import torch

        from paper_2403_09603_b200 import _device as D
        from paper_2403_09603_b200 import _lib
        self.D, self.lib, self.world = D, _lib, world
        words = int(_lib.lib().vt_exchange_words(world))
        self.bufs = [torch.zeros(words, dtype=torch.int64, device="cuda") for _ in range(world)]
        self.ptrs = torch.tensor([b.data_ptr() for b in self.bufs], dtype=torch.int64, device="cuda")
        self.counts = [torch.full((world,), -1, dtype=torch.int64, device="cuda") for _ in range(world)]
        self.flags = [torch.zeros(2, dtype=torch.int32, device="cuda") for _ in range(world)]
        self.pending = {}

    def publish(self, r: int, x, tau: float, base: int):
        import torch

        from paper_2403_09603_b200 import ops
        D, lib = self.D, self.lib
        n = x.numel()
        y = torch.empty(n, dtype=torch.float32, device="cuda")
        words = torch.empty(max(n, 1024), dtype=torch.int64, device="cuda")
        ws = D.workspace(int(lib.lib().vt_round_log_workspace(max(n, 1))), "round_log")
        f = D.Flags()
        lib.call("vt_round_log_exchange", D.ptr(x) if n else None, n, 32, float(tau), lib.OUT_F32, D.ptr(y),
                 D.ptr(words), words.numel(), int(base), f.cnt_ptr, f.err_ptr, D.ptr(ws), ws.numel(),
                 self.ptrs.data_ptr(), self.world, r, D.stream_ptr())
        self.pending[r] = ops.PendingRound(y, words, f)

    def wait(self, r: int):
        lib = self.lib
        lib.call("vt_counts_wait", self.ptrs.data_ptr(), self.world, r, self.D.ptr(self.counts[r]),
                 self.flags[r].data_ptr(), self.D.stream_ptr())
        return self.counts[r]


def _shards(round_no: int):
    from paper_2403_09603_b200 import workloads
    sizes = [(1 << 18) + 17 * round_no, 70_001, 0 if round_no % 2 else 5_000, (1 << 20) + 3]
    return [workloads.config0_x_torch(n, 100 * round_no + r) if n else None for r, n in enumerate(sizes)]


def test_virtual_ranks_exchange_counts_in_lockstep():
    """Rounds of publish-all then wait-all: every rank sees every rank's count."""
    import torch

    from paper_2403_09603_b200 import ops, workloads
    vr = _VirtualRanks(W)
    tau = workloads.TAU_CONFIG0
    for rnd in range(5):
        xs = _shards(rnd)
        want = []
        for r, x in enumerate(xs):
            xx = x if x is not None else torch.empty(0, dtype=torch.float64, device="cuda")
            vr.publish(r, xx, tau, 1_000 * r)
            want.append(ops.round_and_log(xx, 32, tau, global_base=1_000 * r)[1].count if xx.numel() else 0)
        for r in range(W):
            assert vr.wait(r).tolist() == want, (rnd, r)
        for r, x in enumerate(xs):
            y, log = vr.pending[r].finish()
            if x is not None:
                y1, log1 = ops.round_and_log(x, 32, tau, global_base=1_000 * r)
                assert torch.equal(y.view(torch.int32), y1.view(torch.int32))
                assert torch.equal(log.words, log1.words)
        torch.cuda.synchronize()
        assert all(int(f[0].item()) == 0 for f in vr.flags)
    # every rank's own sequence number counts the exchanges
    assert [int(b[0].item()) for b in vr.bufs] == [5] * W


def test_virtual_ranks_one_exchange_ahead():
    """A rank that publishes exchange k+1 before a peer has waited for
    exchange k must not overwrite what that peer still reads (the slots
    alternate by parity)."""
    import torch

    from paper_2403_09603_b200 import ops, workloads
    vr = _VirtualRanks(W)
    tau = workloads.TAU_CONFIG0
    xs0, xs1 = _shards(1), _shards(2)

    def count(x, r):
        return ops.round_and_log(x, 32, tau, global_base=7 * r)[1].count if x is not None else 0

    empty = torch.empty(0, dtype=torch.float64, device="cuda")
    want0 = [count(x, r) for r, x in enumerate(xs0)]
    want1 = [count(x, r) for r, x in enumerate(xs1)]
    for r, x in enumerate(xs0):  # exchange 0: everyone publishes
        vr.publish(r, x if x is not None else empty, tau, 7 * r)
    got0 = {}
    got0[0] = vr.wait(0).clone()  # rank 0 waits ...
    vr.publish(0, xs1[0], tau, 0)  # ... and runs ahead into exchange 1
    for r in range(1, W):  # the others only now read exchange 0
        got0[r] = vr.wait(r).clone()
    for r in range(1, W):
        vr.publish(r, xs1[r] if xs1[r] is not None else empty, tau, 7 * r)
    got1 = {r: vr.wait(r).clone() for r in range(W)}
    torch.cuda.synchronize()
    assert all(got0[r].tolist() == want0 for r in range(W)), (got0, want0)
    assert all(got1[r].tolist() == want1 for r in range(W)), (got1, want1)
    assert all(int(f[0].item()) == 0 for f in vr.flags)
