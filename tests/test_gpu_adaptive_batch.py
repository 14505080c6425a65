"""GPU parity of the batched adaptive round-and-log
(ops.round_and_log_adaptive_batch -> vt_round_log_adaptive_batch): many
independent tensors in one fused rounding pass plus batched selection and
filter kernels.  Per tensor the result must equal the oracle's budget search
(protocol.search_tau skeleton, pkg/src/vtrain/protocol.py:494-506, budget
form of SURVEY.md A.4), the oracle's direction codes at that tau
(fpround.py:164-177) as sparse words, and rnd_array (fpround.py:127-135)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu


def _inputs(seed: int):
    """Ragged sizes (tile / super-tile edges), magnitudes from 1e-3 to 10,
    and tensors that take each exact-fallback trigger."""
    from paper_2403_09603_b200 import workloads
    rng = np.random.default_rng(seed)
    xs = []
    for n in [1, 5, 2047, 2048, 2049, 8191, 8192, 8193, 10_000, 100_003, 1 << 20]:
        xs.append(rng.normal(0.0, 10.0 ** rng.uniform(-3, 1), n))
    n = 200_000
    xs.append(np.where(rng.random(n) < 0.9, np.round(rng.normal(0, 100, n)), rng.normal(0, 1, n)))  # few cands
    xs.append(workloads.config0_x(n, 8))                                                       # midpoints
    xs.append(rng.normal(0, 1, 50_000) * np.exp2(rng.integers(-160, 4, 50_000)))            # tiny values
    return xs


def _check_all(oracle, xs, res, b_r, budgets, bases=None):
    for i, (x, (y, log, tau)) in enumerate(zip(xs, res)):
        t_or = oracle.search_tau_budget(x, b_r, budgets[i])
        assert tau == t_or, (i, tau.hex(), t_or.hex())
        want = oracle.sparse_from_codes(oracle.direction_array(x, b_r, t_or), base=0 if bases is None else bases[i])
        assert log.count == want.size, i
        assert np.array_equal(log.words.cpu().numpy().view(np.uint64), want), i
        r = oracle.rnd_array(x, b_r)
        got = y.cpu().numpy()
        assert np.array_equal(bits(got), bits(r if got.dtype == np.float64 else r.astype(np.float32))), i


def test_batch_matches_oracle(oracle):
    import torch
    from paper_2403_09603_b200 import ops
    xs = _inputs(1)
    budgets = [int(0.005 * x.size) for x in xs]
    budgets[-2] = int(0.4 * xs[-2].size)  # a 40 % budget: too many candidates
    bases = [1000 * i for i in range(len(xs))]
    res = ops.round_and_log_adaptive_batch([torch.from_numpy(x).cuda() for x in xs], 32, budgets,
                                           global_bases=bases)
    _check_all(oracle, xs, res, 32, budgets, bases)


@pytest.mark.parametrize("b_r", [26, 10])
def test_batch_general_grid_fp64_out(oracle, b_r):
    import torch
    from paper_2403_09603_b200 import ops
    rng = np.random.default_rng(b_r)
    xs = [rng.normal(0.0, 2.0, n) for n in (3, 4099, 123_457, 40_000)]
    budgets = [max(1, int(0.005 * x.size)) for x in xs]
    res = ops.round_and_log_adaptive_batch([torch.from_numpy(x).cuda() for x in xs], b_r, budgets,
                                           out_dtype=torch.float64)
    _check_all(oracle, xs, res, b_r, budgets)


def test_batch_equals_single_calls_and_chunks():
    """More tensors than one launch's table (224) and every size twice:
    the batch equals the per-tensor single calls bit for bit; repeated and
    re-shaped batches on one workspace stay exact."""
    import torch
    from paper_2403_09603_b200 import ops
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    sizes = [int(s) for s in np.random.default_rng(5).integers(1, 40_000, 300)]
    xs = [torch.randn(n, dtype=torch.float64, device="cuda", generator=g) * (1 + i % 7) for i, n in enumerate(sizes)]
    budgets = [int(0.01 * n) for n in sizes]
    for rep in range(2):
        sub = xs if rep == 0 else xs[::-1][:150]
        bud = budgets if rep == 0 else budgets[::-1][:150]
        res = ops.round_and_log_adaptive_batch(sub, 32, bud)
        for x, B, (y, log, tau) in zip(sub, bud, res):
            y1, log1, tau1 = ops.round_and_log_adaptive(x, 32, B)
            assert tau == tau1
            assert torch.equal(log.words, log1.words)
            assert torch.equal(y.view(torch.int32), y1.view(torch.int32))


def test_batch_graph_replay_and_empty():
    """Graph-captured batch (the configs[2] bench form) replays to the eager
    results; an empty tensor gets the host search's tau and an empty log."""
    import torch
    from paper_2403_09603_b200 import ops, protocol
    g = torch.Generator(device="cuda")
    g.manual_seed(6)
    xs = [torch.randn(n, dtype=torch.float64, device="cuda", generator=g) for n in (70_000, 0, 1 << 18, 12_345)]
    budgets = [int(0.005 * x.numel()) for x in xs]
    want = ops.round_and_log_adaptive_batch(xs, 32, budgets)
    assert want[1][1].count == 0
    assert want[1][2] == protocol.search_tau_budget(xs[1], 32, budgets[1])
    ys = [torch.empty(x.numel(), dtype=torch.float32, device="cuda") for x in xs]
    ws = [torch.empty(b + 1, dtype=torch.int64, device="cuda") for b in budgets]
    holder = {}

    def run():
        holder["p"] = ops.round_and_log_adaptive_batch(xs, 32, budgets, outs=ys, log_outs=ws, check=False)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        run()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        run()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    got = holder["p"].finish()
    for (y0, l0, t0), (y1, l1, t1) in zip(want, got):
        assert t0 == t1
        assert torch.equal(l0.words, l1.words)
        assert torch.equal(y0.reshape(-1).view(torch.int32), y1.view(torch.int32))


def test_batch_errors():
    import torch
    from paper_2403_09603_b200 import ops
    a = torch.randn(10_000, dtype=torch.float64, device="cuda")
    b = torch.randn(20_000, dtype=torch.float64, device="cuda")
    b[777] = float("nan")
    with pytest.raises(ValueError, match="non-finite value"):
        ops.round_and_log_adaptive_batch([a, b], 32, [50, 100])
    c = torch.randn(20_000, dtype=torch.float64, device="cuda")
    c[5] = 1e300
    with pytest.raises(ValueError, match="out of representable range"):
        ops.round_and_log_adaptive_batch([a, c], 32, [50, 100])
    with pytest.raises(ValueError, match="in-place"):
        ops.round_and_log_adaptive_batch([a], 32, [50], out_dtype=torch.float64, outs=[a])
    with pytest.raises(ValueError, match="one budget per tensor"):
        ops.round_and_log_adaptive_batch([a, b], 32, [50])
    with pytest.raises(ValueError, match="global_bases: one entry per tensor"):
        ops.round_and_log_adaptive_batch([a, c], 32, [50, 100], global_bases=[0])
    small = torch.empty(3, dtype=torch.int64, device="cuda")
    with pytest.raises(ops.LogOverflow):
        ops.round_and_log_adaptive_batch([torch.randn(100_000, dtype=torch.float64, device="cuda")], 32, [500],
                                         log_outs=[small])


@pytest.mark.parametrize("frac", [0.02, 0.1])
def test_batch_dense_candidates(oracle, frac):
    """Budgets of 2 % and 10 %: at the candidate threshold many 256-element
    rows hold more candidates than the rounding pass stages keys for (12),
    so those keys are gathered from x by the histogram pass; mixed with
    staged rows the result still equals the oracle."""
    import torch
    from paper_2403_09603_b200 import ops
    rng = np.random.default_rng(int(frac * 1000))
    xs = [rng.normal(0.0, 1.0, n) for n in (300_001, 65_536, 9_999)]
    xs.append(rng.normal(0.0, 1.0, 100_000) * np.exp2(rng.integers(-140, -120, 100_000)))  # FP32-subnormal zone
    budgets = [int(frac * x.size) for x in xs]
    res = ops.round_and_log_adaptive_batch([torch.from_numpy(x).cuda() for x in xs], 32, budgets)
    _check_all(oracle, xs, res, 32, budgets)
