"""Development aid: per-step and per-hook GPU time of the configs[3] GPT-2
FP64 step with the round-and-log hooks, over several steps (variance hunt)."""
import json
import sys
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import hooks, ops, workloads

model = workloads.gpt2_small_fp64()
opt = torch.optim.SGD(model.parameters(), lr=1e-4)
g = torch.Generator(device="cuda"); g.manual_seed(3)
idx = torch.randint(0, 50257, (8, 1024), device="cuda", generator=g)
tgt = torch.randint(0, 50257, (8, 1024), device="cuda", generator=g)
orig = ops.round_and_log_adaptive
ev = []


def wrapped(x, *a, **k):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    r = orig(x, *a, **k)
    e.record()
    ev.append((x.numel(), s, e, r))
    return r


ops.round_and_log_adaptive = wrapped
hk = hooks.RoundAndLogHooks(model)


def step():
    opt.zero_grad(set_to_none=True)
    logits = model(idx)
    loss = torch.nn.functional.cross_entropy(logits.view(-1, logits.shape[-1]), tgt.view(-1))
    loss.backward()
    opt.step()


for it in range(8):
    ev.clear()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); step(); b.record()
    torch.cuda.synchronize()
    per = sorted(((s.elapsed_time(e), n, r.tau.item(), r.flags.read()[1][0]) for n, s, e, r in ev), reverse=True)
    print(json.dumps({"step": it, "ms": round(a.elapsed_time(b), 2), "hooks_ms": round(sum(p[0] for p in per), 2),
                      "top": [[round(p[0], 3), p[1], p[2], p[3]] for p in per[:4]]}))
    hk.collect()
