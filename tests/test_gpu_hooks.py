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
