"""The public operators are reentrant across streams and host threads
(SURVEY.md §8b threading row; reference purity: fpround is pure and
thread-safe).  Each (device, stream) gets its own workspace, so two host
threads driving two streams at once through ``ops.round_and_log``,
``ops.replay`` and ``ops.round_and_log_adaptive`` must reproduce the
sequential results bit for bit.  Caller-supplied output buffers are
validated before their pointers reach the C ABI."""

from __future__ import annotations

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.timeout(300)
def test_two_threads_two_streams_public_api(oracle):
    import torch

    from paper_2403_09603_b200 import ops, workloads
    tau = workloads.TAU_CONFIG0
    sizes = [(1 << 23) + 4099, (1 << 22) + 77]
    pairs = [workloads.config1_pair(n, 40 + i) for i, n in enumerate(sizes)]
    xs = [(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()) for a, b in pairs]
    ref = []
    for (xt, xa), n in zip(xs, sizes):
        y, log = ops.round_and_log(xt, 32, tau)
        ya, corr = ops.replay(xa, 32, log)
        yad, logad, tauad = ops.round_and_log_adaptive(xt, 32, int(0.005 * n))
        ref.append((y.clone(), log.words.clone(), ya.clone(), corr, yad.clone(), logad.words.clone(), tauad))
    # the sequential results are the oracle's
    codes = oracle.direction_array(pairs[1][0], 32, tau)
    assert np.array_equal(ref[1][1].cpu().numpy().view(np.uint64), oracle.sparse_from_codes(codes))
    torch.cuda.synchronize()

    errors: list = []
    barrier = threading.Barrier(len(xs))

    def worker(i: int) -> None:
        try:
            s = torch.cuda.Stream()
            xt, xa = xs[i]
            n = sizes[i]
            with torch.cuda.stream(s):
                barrier.wait()
                for rep in range(12):
                    p = ops.round_and_log(xt, 32, tau, check=False)
                    y, log = p.finish()
                    ya, corr = ops.replay(xa, 32, log)
                    yad, logad, tauad = ops.round_and_log_adaptive(xt, 32, int(0.005 * n))
                    r = ref[i]
                    ok = (torch.equal(y.view(torch.int32), r[0].view(torch.int32)) and torch.equal(log.words, r[1])
                          and torch.equal(ya.view(torch.int32), r[2].view(torch.int32)) and corr == r[3]
                          and torch.equal(yad.view(torch.int32), r[4].view(torch.int32))
                          and torch.equal(logad.words, r[5]) and tauad == r[6])
                    if not ok:
                        errors.append((i, rep))
                        return
        except Exception as e:  # pragma: no cover - reported below
            errors.append((i, repr(e)))

    th = [threading.Thread(target=worker, args=(i,)) for i in range(len(xs))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=240)
    assert not errors, errors


def test_workspaces_are_per_stream():
    import torch

    from paper_2403_09603_b200 import _device as D
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        a = D.workspace(4096, "t_ws")
        a2 = D.workspace(4096, "t_ws")
    with torch.cuda.stream(s2):
        b = D.workspace(4096, "t_ws")
    assert a.data_ptr() == a2.data_ptr() and a.data_ptr() != b.data_ptr()
    with torch.cuda.stream(s1):
        big = D.workspace(8 << 20, "t_ws")  # grows: the old buffer is retired, not freed
    assert big.numel() >= 8 << 20 and any(r.data_ptr() == a.data_ptr() for r in D._RETIRED)


def test_workspace_growth_is_geometric():
    """A run of ever larger calls retires O(log) buffers, not one per call."""
    import torch

    from paper_2403_09603_b200 import _device as D
    s = torch.cuda.Stream()
    before = len(D._RETIRED)
    with torch.cuda.stream(s):
        for k in range(1, 201):
            ws = D.workspace(k * (1 << 20) + 7, "t_ws_geo")
            assert ws.numel() >= k * (1 << 20) + 7
    retired = D._RETIRED[before:]
    assert len(retired) <= 16, len(retired)
    assert sum(r.numel() for r in retired) <= 2 * ws.numel()


def test_out_buffers_are_validated():
    import torch

    from paper_2403_09603_b200 import ops, workloads
    x = torch.from_numpy(workloads.config0_x(4096, 5)).cuda()
    tau = workloads.TAU_CONFIG0
    bad = [
        dict(out=torch.empty(4096, dtype=torch.float64, device="cuda")),           # dtype
        dict(out=torch.empty(4095, dtype=torch.float32, device="cuda")),           # too short
        dict(out=torch.empty(8192, dtype=torch.float32, device="cuda")[::2]),      # strided
        dict(out=torch.empty(4096, dtype=torch.float32)),                          # host
        dict(log_out=torch.empty(4096, dtype=torch.int32, device="cuda")),         # log dtype
        dict(codes_out=torch.empty(100, dtype=torch.uint8, device="cuda")),        # codes too short
    ]
    for kw in bad:
        with pytest.raises(ValueError):
            ops.round_and_log(x, 32, tau, **kw)
    with pytest.raises(ValueError):
        ops.round_and_log(x, 32, tau, out_dtype=torch.float16)
    _, log = ops.round_and_log(x, 32, tau)
    with pytest.raises(ValueError):
        ops.replay(x, 32, log, out=torch.empty(4096, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        ops.round_and_log_adaptive(x, 32, 20, out=torch.empty(10, dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        ops.round_and_log_adaptive_batch([x], 32, [20], outs=[torch.empty(4096, dtype=torch.float64, device="cuda")])
    with pytest.raises(ValueError):
        ops.round_and_log_adaptive_batch([x], 32, [20], log_outs=[torch.empty(21, dtype=torch.float32,
                                                                              device="cuda")])


def test_default_log_capacity_grows_when_needed(oracle):
    """round_and_log without log_out sizes the log at n/8 and re-runs once
    with the exact size when more is logged (tau = 0 logs every off-grid
    element)."""
    import torch

    from paper_2403_09603_b200 import ops, workloads
    xh = workloads.config0_x(200_003, 8)
    x = torch.from_numpy(xh).cuda()
    assert ops.default_log_capacity(200_003) == 1 << 16
    y, log = ops.round_and_log(x, 32, 0.0)
    want = oracle.sparse_from_codes(oracle.direction_array(xh, 32, 0.0))
    assert log.count == want.size > 200_003 // 2
    assert np.array_equal(log.words.cpu().numpy().view(np.uint64), want)
    with pytest.raises(ops.LogOverflow):
        ops.round_and_log(x, 32, 0.0, check=False).finish()


def test_flags_out_arena_for_round_and_log_and_replay(oracle):
    """flags_out: caller-owned zeroed flag rows instead of a per-call
    allocation -- same outputs, counts and corrections; a graph of both
    operators on arena rows allocates nothing per replay."""
    import numpy as np
    import torch

    from paper_2403_09603_b200 import ops, workloads
    n = (1 << 20) + 33
    xt, xa = workloads.config1_pair(n, 5)
    tau = workloads.TAU_CONFIG0
    t, a = torch.from_numpy(xt).cuda(), torch.from_numpy(xa).cuda()
    arena = torch.zeros((2, 6), dtype=torch.int64, device="cuda")
    y, log = ops.round_and_log(t, 32, tau, flags_out=arena[0])
    ya, corr = ops.replay(a, 32, log, flags_out=arena[1])
    y1, log1 = ops.round_and_log(t, 32, tau)
    ya1, corr1 = ops.replay(a, 32, log1)
    assert torch.equal(log.words, log1.words) and torch.equal(y.view(torch.int32), y1.view(torch.int32))
    assert torch.equal(ya.view(torch.int32), ya1.view(torch.int32)) and corr == corr1
    assert int(arena[0, 2]) == log.count and int(arena[1, 2]) == corr
    codes = oracle.direction_array(xt, 32, tau)
    assert np.array_equal(log.words.cpu().numpy().view(np.uint64), oracle.sparse_from_codes(codes))
    # graph-captured on arena rows (zeroed inside the graph, no allocation per replay)
    yo = torch.empty(n, dtype=torch.float32, device="cuda")
    yao = torch.empty(n, dtype=torch.float32, device="cuda")
    words = torch.empty(n // 4, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())

    def step():
        arena.zero_()
        p = ops.round_and_log(t, 32, tau, out=yo, log_out=words, check=False, flags_out=arena[0])
        ops.replay(a, 32, words[:log.count], out=yao, check=False, flags_out=arena[1])
        return p

    with torch.cuda.stream(s):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    assert int(arena[0, 2]) == log.count and int(arena[1, 2]) == corr
    assert torch.equal(yao.view(torch.int32), ya1.view(torch.int32))
