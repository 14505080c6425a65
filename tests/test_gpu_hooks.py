"""Round-and-log hooks on a torch FP64 model: every leaf output and input
gradient lands on the FP32 grid with its adaptive tau, in place."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_hooks_tiny_gpt2(oracle):
    import torch
    from paper_2403_09603_b200 import hooks, workloads
    model = workloads.gpt2_small_fp64(vocab=97, d=64, layers=2, heads=4, ctx=32)
    idx = torch.randint(0, 97, (2, 32), device="cuda")
    seen = []

    def spy(mod, inp, out):
        seen.append(out.detach().clone())

    hk = hooks.RoundAndLogHooks(model)
    # runs after the rounding hook (registered later): sees the rounded output
    for mod in model.modules():
        if not any(True for _ in mod.children()):
            mod.register_forward_hook(spy)
    logits = model(idx)
    loss = torch.nn.functional.cross_entropy(logits.view(-1, 97), idx.view(-1))
    loss.backward()
    info = hk.collect()
    assert info["fwd"] == 2 + 2 * 7 + 2 and info["bwd"] > 0
    for t in seen:
        a = t.cpu().numpy().reshape(-1)
        assert np.array_equal(a.view(np.uint64), oracle.rnd_array(a, 32).view(np.uint64))
    for p in model.parameters():
        assert p.grad is not None and torch.isfinite(p.grad).all()
    hk.remove()


def test_hooks_arena_growth_and_reuse(oracle):
    """More hooked tensors than the first result arena (64 slots): the slots
    grow during the first step while earlier calls are still pending, and a
    second step reuses them; per-tensor taus equal the oracle's search and
    every rounded output is on the grid."""
    import torch
    from paper_2403_09603_b200 import hooks, ops
    torch.manual_seed(0)
    model = torch.nn.Sequential(*[torch.nn.Linear(48, 48, dtype=torch.float64) for _ in range(45)]).cuda()
    x = torch.randn(64, 48, dtype=torch.float64, device="cuda")
    seen = []
    orig = ops.round_and_log_adaptive

    def spy(t, b_r, budget, **kw):
        seen.append((t.detach().clone().cpu().numpy(), b_r, budget))
        return orig(t, b_r, budget, **kw)

    ops.round_and_log_adaptive = spy
    try:
        hk = hooks.RoundAndLogHooks(model)
        infos = []
        for step in range(2):
            seen.clear()
            model(x).sum().backward()
            taus = hk._taus[:len(hk.records)].cpu().tolist()
            counts = [int(c) for c in hk._flags[:len(hk.records), 2].cpu().tolist()]
            infos.append(hk.collect())
            assert infos[-1]["tensors"] == len(seen) > 64
            for (a, b_r, budget), tau, cnt in zip(seen, taus, counts):
                t_or = oracle.search_tau_budget(a.reshape(-1), b_r, budget)
                assert tau == t_or
                assert cnt == int(np.count_nonzero(oracle.direction_array(a.reshape(-1), b_r, t_or) != 1))
        assert infos[0]["tensors"] == infos[1]["tensors"]
        hk.remove()
    finally:
        ops.round_and_log_adaptive = orig


def test_hooks_error_then_clean_step():
    """A non-finite activation raises the reference's error at collect();
    the next step starts from cleared slots."""
    import torch
    from paper_2403_09603_b200 import hooks
    model = torch.nn.Sequential(torch.nn.Linear(16, 16, dtype=torch.float64),
                                torch.nn.Linear(16, 16, dtype=torch.float64)).cuda()
    hk = hooks.RoundAndLogHooks(model)
    x = torch.randn(8, 16, dtype=torch.float64, device="cuda")
    bad = x.clone()
    bad[0, 0] = float("inf")
    model(bad)
    with pytest.raises(ValueError, match="non-finite value"):
        hk.collect()
    model(x).sum().backward()
    info = hk.collect()
    assert info["tensors"] > 0
    hk.remove()


@pytest.mark.parametrize("b_r", [32, 26])
def test_auditor_replay_hooks_reproduce_the_trainer(oracle, b_r):
    """Trainer: RoundAndLogHooks on a small FP64 GPT-2 step, logs kept.
    Auditor: the same step on a copy of the model whose every hooked tensor
    is perturbed (a stand-in for other hardware: 5% of the elements moved by
    up to 2^-34 relative, inside the logged band) and then replayed with the
    trainer's logs -- every hooked tensor, the loss and every gradient equal
    the trainer's bit for bit, with corrections where plain rounding of the
    perturbed values would have diverged (protocol._AuditorChannel on a
    torch model)."""
    import copy
    import torch
    from paper_2403_09603_b200 import hooks, workloads
    torch.manual_seed(4)
    model = workloads.gpt2_small_fp64(vocab=97, d=64, layers=2, heads=4, ctx=32)
    with torch.no_grad():  # full 53-bit FP64 parameters: an FP32-derived init puts 1/64 of the embedding
        for prm in model.parameters():  # rows exactly on b_r = 26 midpoints, which no budget tau logs
            prm.add_(torch.randn_like(prm) * 1e-9)
    model_a = copy.deepcopy(model)
    idx = torch.randint(0, 97, (4, 32), device="cuda")

    def run(m, hk_factory):
        seen = []
        hk = hk_factory(m)
        hs = [mod.register_forward_hook(lambda mod, i, o: seen.append(o.detach().clone()))
              for mod in m.modules() if not any(True for _ in mod.children())]
        logits = hk.loss_grad(m(idx))  # the loss gradient goes through the channel too (protocol.py:277-280)
        loss = torch.nn.functional.cross_entropy(logits.view(-1, 97), idx.view(-1))
        loss.backward()
        for h in hs:
            h.remove()
        return hk, seen, loss.detach().clone(), [p.grad.clone() for p in m.parameters()]

    hk_t, seen_t, loss_t, grads_t = run(model, lambda m: hooks.RoundAndLogHooks(m, b_r=b_r))
    info = hk_t.collect(keep_logs=True)
    hk_t.remove()
    assert len(info["logs"]) == info["tensors"] and info["logged"] > 0 and info["loss"] == 1

    g = torch.Generator(device="cuda")
    g.manual_seed(11)

    def perturb(flat):
        sel = torch.rand(flat.numel(), device="cuda", generator=g) < 0.05
        # below the budget tau's margin to the midpoint ((1 - tau / 2^-24) ~ 0.005 of the half-ulp):
        # an auditor deviation the trainer's log covers
        rel = (torch.rand(flat.numel(), device="cuda", dtype=torch.float64, generator=g) * 2 - 1) * \
            2.0 ** -(b_r + 2)  # the same fraction of a grid step (2^-(b_r - 9) relative) on every grid
        flat.add_(torch.where(sel, flat * rel, torch.zeros_like(flat)))

    hk_a, seen_a, loss_a, grads_a = run(model_a, lambda m: hooks.ReplayHooks(m, info["logs"], b_r=b_r,
                                                                              perturb=perturb))
    res = hk_a.collect()
    hk_a.remove()
    assert res["tensors"] == info["tensors"]
    assert sum(res["corrections"]) > 0
    assert len(seen_a) == len(seen_t)
    for a, t in zip(seen_a, seen_t):
        assert torch.equal(a.view(torch.int64), t.view(torch.int64))
    assert torch.equal(loss_a.view(torch.int64), loss_t.view(torch.int64))
    for a, t in zip(grads_a, grads_t):
        assert torch.equal(a.view(torch.int64), t.view(torch.int64))


def test_replay_hooks_out_of_step():
    """An auditor whose hooked tensors do not follow the trainer's order (or
    count) is refused, as protocol._run refuses an operation-count mismatch."""
    import torch
    from paper_2403_09603_b200 import hooks
    model = torch.nn.Sequential(torch.nn.Linear(16, 16, dtype=torch.float64),
                                torch.nn.Linear(16, 16, dtype=torch.float64)).cuda()
    x = torch.randn(8, 16, dtype=torch.float64, device="cuda")
    hk = hooks.RoundAndLogHooks(model)
    model(x)  # forward only: two hooked outputs
    logs = hk.collect(keep_logs=True)["logs"]
    hk.remove()
    ha = hooks.ReplayHooks(model, logs[::-1])  # wrong order
    with pytest.raises(RuntimeError, match="out of step"):
        model(x)
    ha.remove()
    ha = hooks.ReplayHooks(model, logs + logs)  # the trainer logged more
    model(x)
    with pytest.raises(RuntimeError, match="out of step"):
        ha.collect()
    ha.remove()


def test_loss_gradient_and_parameters_on_the_grid(oracle):
    """hooks.loss_grad: the gradient reaching the model output is rounded and
    logged with its own budget tau (protocol.py:277-280); round_parameters:
    every parameter lands on the grid after the update (protocol.py:286-293)."""
    import torch
    from paper_2403_09603_b200 import hooks, workloads
    torch.manual_seed(6)
    model = workloads.gpt2_small_fp64(vocab=97, d=64, layers=2, heads=4, ctx=32)
    idx = torch.randint(0, 97, (2, 32), device="cuda")
    hk = hooks.RoundAndLogHooks(model)
    seen, raw = [], []
    out = model(idx)
    out.register_hook(lambda g_: raw.append(g_.detach().clone()))  # tensor hooks run in order: the raw gradient
    logits = hk.loss_grad(out)
    logits.register_hook(lambda g_: seen.append(g_.detach().clone()))  # after the rounding hook
    torch.nn.functional.cross_entropy(logits.view(-1, 97), idx.view(-1)).backward()
    info = hk.collect(keep_logs=True)
    hk.remove()
    assert info["loss"] == 1 and len(seen) == 1 and len(raw) == 1
    k = [c[1] for c in info["calls"]].index("loss")
    g = seen[0].cpu().numpy().reshape(-1)
    assert np.array_equal(g.view(np.uint64), oracle.rnd_array(g, 32).view(np.uint64))
    # the loss gradient's log is the oracle's at the oracle's budget tau
    r = raw[0].cpu().numpy().reshape(-1)
    B = int(0.005 * r.size)
    tau = oracle.search_tau_budget(r, 32, B)
    assert info["taus"][k] == tau
    codes = oracle.direction_array(r, 32, tau)
    want = np.flatnonzero(codes != 1)
    words = info["logs"][k][2].cpu().numpy()
    assert np.array_equal(words >> 1, want) and np.array_equal(words & 1, (codes[want] == 2).astype(np.int64))
    # parameters after an SGD update
    with torch.no_grad():
        for p in model.parameters():
            p.add_(p.grad, alpha=-1e-3)
    hooks.round_parameters(model)
    for p in model.parameters():
        a = p.detach().cpu().numpy().reshape(-1)
        assert np.array_equal(a.view(np.uint64), oracle.rnd_array(a, 32).view(np.uint64))
