"""The peer-memory exchanges (round-and-log counts, Merkle block roots)
with several ranks on ONE GPU, without
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
        base0 = (1 << 33) + 17 if rnd == 4 else 0  # global indices past 32 bits in the last round
        for r, x in enumerate(xs):
            xx = x if x is not None else torch.empty(0, dtype=torch.float64, device="cuda")
            vr.publish(r, xx, tau, base0 + 1_000 * r)
            want.append(ops.round_and_log(xx, 32, tau, global_base=base0 + 1_000 * r)[1].count if xx.numel() else 0)
        for r in range(W):
            assert vr.wait(r).tolist() == want, (rnd, r)
        for r, x in enumerate(xs):
            y, log = vr.pending[r].finish()
            if x is not None:
                y1, log1 = ops.round_and_log(x, 32, tau, global_base=base0 + 1_000 * r)
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


# ---------------------------------------------------------------------------
# the Merkle block-root exchange (vt_merkle_level_exchange / vt_digests_publish
# / vt_digests_wait), W virtual ranks on one GPU in the same publish-then-wait
# order
# ---------------------------------------------------------------------------

def _virtual_merkle(w_bytes, n_leaves: int, world: int, k: int, rounds: int = 1):
    """Every virtual rank hashes its whole 2^k-leaf blocks; the level that
    yields its block roots publishes them; then every rank waits and builds
    the top levels.  Returns (per-rank local levels, per-rank roots, root)."""
    import torch

    from paper_2403_09603_b200 import _device as D
    from paper_2403_09603_b200 import _lib, merkle
    from paper_2403_09603_b200 import dist as vdist
    depth = vdist.local_depth(n_leaves, k)
    ranges = [vdist.leaf_block_range(n_leaves, r, world, k) for r in range(world)]
    n_blocks = [(hi - lo + (1 << k) - 1) >> k for lo, hi in ranges]
    n_total = sum(n_blocks)
    words = int(_lib.lib().vt_digest_exchange_words(world, n_total))
    bufs = [torch.zeros(words, dtype=torch.int64, device="cuda") for _ in range(world)]
    ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    flags = [torch.zeros(2, dtype=torch.int32, device="cuda") for _ in range(world)]
    out = None
    for _ in range(rounds):
        local = []
        for r, (lo, hi) in enumerate(ranges):
            dst = sum(n_blocks[:r])
            b = w_bytes[lo * 4096: min(hi * 4096, w_bytes.numel())]
            if hi <= lo:
                lv = [torch.zeros((0, 32), dtype=torch.uint8, device="cuda") for _ in range(depth + 1)]
                _lib.call("vt_digests_publish", None, 0, ptrs.data_ptr(), world, r, dst, n_total, D.stream_ptr())
                local.append(lv)
                continue
            cur = merkle.sha256_leaves(b, 4096)
            lv, published = [cur], False
            for L in range(depth):
                if cur.shape[0] > 1:
                    nxt = torch.empty(((cur.shape[0] + 1) // 2, 32), dtype=torch.uint8, device="cuda")
                    if L == depth - 1:
                        _lib.call("vt_merkle_level_exchange", D.ptr(cur), cur.shape[0], D.ptr(nxt), ptrs.data_ptr(),
                                  world, r, dst, n_total, D.stream_ptr())
                        published = True
                    else:
                        _lib.call("vt_merkle_level", D.ptr(cur), cur.shape[0], D.ptr(nxt), D.stream_ptr())
                    cur = nxt
                lv.append(cur)
            if not published:
                _lib.call("vt_digests_publish", D.ptr(lv[-1]), lv[-1].shape[0], ptrs.data_ptr(), world, r, dst,
                          n_total, D.stream_ptr())
            local.append(lv)
        roots = []
        for r in range(world):
            got = torch.empty((n_total, 32), dtype=torch.uint8, device="cuda")
            _lib.call("vt_digests_wait", ptrs.data_ptr(), world, r, n_total, D.ptr(got), flags[r].data_ptr(),
                      D.stream_ptr())
            roots.append(got)
        top = vdist.combine_top(roots[0], vdist._device_level)
        out = (local, roots, bytes(top[-1][0].cpu().numpy()))
    torch.cuda.synchronize()
    assert all(int(f[0].item()) == 0 for f in flags)
    return out


@pytest.mark.parametrize("n_params,k", [(3 * (1 << 20) + 12345, 4), ((1 << 18) + 7, 2), (9 * 1024, 4),
                                        (1024, 4), (5 * 1024, 12)])
def test_virtual_ranks_merkle_block_roots(n_params, k):
    """Every rank gathers the same block roots = level `depth` of the full
    tree, and the top levels give merkle_chunked's root; uneven, empty and
    single-block ranks included (k small so four ranks get blocks)."""
    import torch

    from paper_2403_09603_b200 import merkle
    from paper_2403_09603_b200 import dist as vdist
    g = torch.Generator(device="cuda")
    g.manual_seed(n_params)
    w = torch.randn(n_params, dtype=torch.float32, device="cuda", generator=g)
    n_leaves = (n_params * 4 + 4095) // 4096
    local, roots, root = _virtual_merkle(w.view(torch.uint8), n_leaves, W, k, rounds=3)
    ref = merkle.merkle_chunked(w)
    assert root == ref.root
    full = ref.levels_device
    depth = vdist.local_depth(n_leaves, k)
    for r in range(W):
        assert torch.equal(roots[r], full[depth])
    levels = vdist.assemble_levels(local, vdist.combine_top(roots[0], vdist._device_level))
    assert len(levels) == len(full) and all(torch.equal(a, b) for a, b in zip(levels, full))


def test_digest_exchange_single_process():
    """Without a process group DigestExchange is the one-rank case, and
    merkle_sharded through it equals merkle_chunked level for level."""
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("a process group is active in this session")
    import torch

    from paper_2403_09603_b200 import merkle
    from paper_2403_09603_b200 import dist as vdist
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    for n_params in (3 * (1 << 20) + 999, 1000):
        w = torch.randn(n_params, dtype=torch.float32, device="cuda", generator=g)
        n_leaves = (n_params * 4 + 4095) // 4096
        n_blocks = (n_leaves + (1 << vdist.BLOCK_LEAVES_LOG2) - 1) >> vdist.BLOCK_LEAVES_LOG2
        ex = vdist.DigestExchange(n_blocks)
        for _ in range(3):  # repeated exchanges: the parity alternates
            lv, top = vdist.merkle_sharded(w.view(torch.uint8), n_leaves, exchange=ex)
        ref = merkle.merkle_chunked(w)
        levels = vdist.assemble_levels([lv], top)
        assert len(levels) == len(ref.levels_device)
        assert all(torch.equal(a, b) for a, b in zip(levels, ref.levels_device))
        assert int(ex.buf[0].item()) == 3


# ---------------------------------------------------------------------------
# the sharded budget search with both exchanges over peer memory
# (vt_tau_shard_search_x): phase A for every virtual rank, then B, then C
# ---------------------------------------------------------------------------

def _virtual_budget(shards, b_r: int, budget: int, keys_cap: int = 1 << 16, iters: int = 30):
    import torch

    from paper_2403_09603_b200 import _device as D
    from paper_2403_09603_b200 import _lib
    world = len(shards)
    n_global = sum(int(s.numel()) for s in shards)
    words = int(_lib.lib().vt_tau_shard_exchange_words(world, keys_cap))
    bufs = [torch.zeros(words, dtype=torch.int64, device="cuda") for _ in range(world)]
    ptrs = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    outs = [torch.zeros(3, dtype=torch.int64, device="cuda") for _ in range(world)]
    wss = [torch.zeros(int(_lib.lib().vt_tau_shard_search_x_workspace(int(s.numel()))) + 256, dtype=torch.uint8,
                       device="cuda") for s in shards]
    wss = [w[(-w.data_ptr()) % 256:] for w in wss]  # 256-byte aligned views
    for phase in (1, 2, 4):
        for r, s in enumerate(shards):
            o = outs[r].data_ptr()
            _lib.call("vt_tau_shard_search_x", D.ptr(s) if s.numel() else None, int(s.numel()), b_r, n_global,
                      budget, iters, ptrs.data_ptr(), bufs[r].data_ptr(), world, r, keys_cap, o, o + 8, o + 16,
                      D.ptr(wss[r]), wss[r].numel(), phase, D.stream_ptr())
    torch.cuda.synchronize()
    res = []
    for o in outs:
        v = o.cpu()
        assert int(v[2]) & 0xFFFFFFFF == 0
        res.append((int(v[1]), float(v[0:1].view(torch.float64).item())))
    return res


@pytest.mark.parametrize("case", ["normal", "uneven_empty", "budget0", "wide", "tiny_budget_digit", "b_r26"])
def test_virtual_ranks_sharded_budget_search(case, oracle):
    """Every virtual rank gets the oracle's budget tau of the whole tensor,
    decided on the device (status 0), for uneven and empty shards and the
    decision's edge cases."""
    import numpy as np
    import torch
    rng = np.random.default_rng({"normal": 1, "uneven_empty": 2, "budget0": 3, "wide": 4,
                                 "tiny_budget_digit": 5, "b_r26": 6}[case])
    b_r = 26 if case == "b_r26" else 32
    if case == "uneven_empty":
        sizes = [300_001, 0, 77_777, 5]
    elif case == "wide":
        sizes = [200_000] * 4
    else:
        sizes = [250_000, 250_003, 249_999, 1]
    x = rng.normal(0.0, 3.0, sum(sizes))
    if case == "wide":
        x *= np.exp2(rng.integers(-60, 60, x.size))
    budget = {"budget0": 0, "tiny_budget_digit": 3}.get(case, int(0.005 * x.size))
    shards, lo = [], 0
    for n in sizes:
        shards.append(torch.from_numpy(x[lo:lo + n].copy()).cuda())
        lo += n
    res = _virtual_budget(shards, b_r, budget)
    want = oracle.search_tau_budget(x, b_r, budget)
    for status, tau in res:
        assert status == 0 and tau == want, (res, want)


def test_virtual_ranks_sharded_budget_fallback_flag(oracle):
    """More digit keys on a rank than keys_cap: status 1 on every rank (the
    host then runs the exact multi-pass path), never a wrong tau."""
    import numpy as np
    import torch
    rng = np.random.default_rng(9)
    x = rng.normal(0.0, 1.0, 800_000)
    # half the elements share one value just below an FP32 rounding midpoint:
    # the (B+1)-th largest distance is theirs, so its digit holds ~100 K keys per rank
    x[rng.random(x.size) < 0.5] = 1.0 + 2.0 ** -24 * (1.0 - 2.0 ** -12)
    shards = [torch.from_numpy(p.copy()).cuda() for p in np.array_split(x, 4)]
    B = int(0.005 * x.size)
    res = _virtual_budget(shards, 32, B, keys_cap=1024)
    assert all(status == 1 for status, _ in res), res
    # (with a larger keys_cap the candidates themselves overflow the shard
    # workspace here -- also status 1).  Through search_tau_budget_sharded the
    # host then runs the exact multi-pass path: the oracle's tau.
    import torch.distributed as dist
    if not dist.is_initialized():
        from paper_2403_09603_b200 import dist as vdist
        ex = vdist.BudgetExchange(keys_cap=1024)
        tau = vdist.search_tau_budget_sharded(torch.from_numpy(x).cuda(), 32, B, exchange=ex)
        assert tau == oracle.search_tau_budget(x, 32, B)


def test_budget_exchange_single_process(oracle):
    """BudgetExchange without a process group (the one-rank case) equals the
    oracle, repeated (the parity alternates), through search_tau_budget_sharded."""
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("a process group is active in this session")
    import numpy as np
    import torch

    from paper_2403_09603_b200 import dist as vdist
    ex = vdist.BudgetExchange()
    rng = np.random.default_rng(12)
    for k in range(3):
        x = rng.normal(0.0, 2.0, 300_003 + k)
        B = int(0.005 * x.size)
        tau = vdist.search_tau_budget_sharded(torch.from_numpy(x).cuda(), 32, B, exchange=ex)
        assert tau == oracle.search_tau_budget(x, 32, B)
    assert int(ex.buf[0].item()) == 3
