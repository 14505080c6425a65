"""configs[3] hook cost breakdown (development aid): the adaptive round-and-log
alone on the 174 GPT-2 hooked tensor sizes, eager and graph-captured."""
import sys, json
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import hooks, ops, workloads

model = workloads.gpt2_small_fp64()
g = torch.Generator(device="cuda"); g.manual_seed(3)
idx = torch.randint(0, 50257, (8, 1024), device="cuda", generator=g)
tgt = torch.randint(0, 50257, (8, 1024), device="cuda", generator=g)
hk = hooks.RoundAndLogHooks(model)
logits = model(idx)
torch.nn.functional.cross_entropy(logits.view(-1, logits.shape[-1]), tgt.view(-1)).backward()
sizes = [r.numel for r in hk.records]
hk.collect(); hk.remove()
del model, logits
torch.cuda.empty_cache()
mx = max(sizes)
buf = torch.randn(mx, dtype=torch.float64, device="cuda", generator=g)
def run():
    for n in sizes:
        x = buf[:n]
        ops.round_and_log_adaptive(x, 32, int(0.005 * n), out_dtype=torch.float64, out=x, check=False, tag="hooks_fwd")
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps
ms = t(run)
print(json.dumps({"tensors": len(sizes), "elements": sum(sizes), "max": mx, "eager_ms": round(ms, 3),
                  "gb_28B": round(sum(sizes) * 28 / 1e9, 2)}))
