"""Writes the pinned list of configs[3]'s hooked GPT-2 tensors (tests/golden/gpt2_hooked_tensors.json
is its formatted copy); needs a GPU.  Development aid."""
import json, sys
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import hooks, workloads
model = workloads.gpt2_small_fp64()
g = torch.Generator(device="cuda"); g.manual_seed(3)
idx = torch.randint(0, 50257, (8, 1024), device="cuda", generator=g)
tgt = torch.randint(0, 50257, (8, 1024), device="cuda", generator=g)
hk = hooks.RoundAndLogHooks(model)
logits = hk.loss_grad(model(idx))
torch.nn.functional.cross_entropy(logits.view(-1, logits.shape[-1]), tgt.view(-1)).backward()
info = hk.collect()
calls = [list(c) for c in info["calls"]]
out = {"about": "BASELINE configs[3]: every tensor the GPT-2-small FP64 step (batch 8 x 1024) passes through the "
                "adaptive round-and-log, in call order: [module, kind (fwd output / bwd input gradient / loss "
                "gradient), elements, budget]; written by tests/golden/make_golden.py --gpt2-list on a B200",
       "tensors": len(calls), "elements": int(sum(c[2] for c in calls)), "calls": calls}
json.dump(out, open("gpurun_out/gpt2_hooked_tensors.json", "w"), indent=0)
print(out["tensors"], out["elements"])
