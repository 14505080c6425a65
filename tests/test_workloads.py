"""The synthetic workloads match their BASELINE.json definitions (CPU)."""

from __future__ import annotations

from collections import Counter

import numpy as np
import pytest

from paper_2403_09603_b200 import workloads


def test_resnet50_tensor_list_matches_torchvision_meta():
    torchvision = pytest.importorskip("torchvision")
    import torch
    model = torchvision.models.resnet50().to("meta")
    outs, ins = [], []

    def hook(mod, inp, out):
        outs.append(tuple(out.shape))
        if isinstance(mod, (torch.nn.Conv2d, torch.nn.Linear)):
            ins.append(tuple(inp[0].shape))

    for m in model.modules():
        if isinstance(m, (torch.nn.Conv2d, torch.nn.BatchNorm2d, torch.nn.Linear)):
            m.register_forward_hook(hook)
    model(torch.empty(32, 3, 224, 224, device="meta"))
    mine = workloads.resnet50_tensors()
    assert len(mine) == 161
    assert Counter(s for n, s in mine if n.startswith("out")) == Counter(outs)
    assert Counter(s for n, s in mine if n.startswith("grad")) == Counter(ins)
    assert sum(int(np.prod(s)) for _, s in mine) == 1_052_589_312


def test_config0_distribution():
    x = workloads.config0_x(1 << 16, 0)
    f = x.astype(np.float32).astype(np.float64)
    # ~10% of values sit within 2^-40 (relative) of an FP32 midpoint
    up = np.nextafter(x.astype(np.float32), np.float32(np.inf)).astype(np.float64)
    dn = np.nextafter(x.astype(np.float32), np.float32(-np.inf)).astype(np.float64)
    lo = np.where(f <= x, f, dn)
    hi = np.where(f <= x, up, f)
    near = np.abs(x - (lo + hi) / 2) <= np.abs(x) * 2.0 ** -39
    assert 0.099 < near.mean() < 0.101
    xt, xa = workloads.config1_pair(1 << 16, 1)
    assert 0.049 < np.mean(xt != xa) < 0.051
    assert np.all(np.abs(xt - xa) <= np.abs(np.nextafter(xt, np.inf) - xt) * 1.0000001)
