"""configs[3] hook cost breakdown (development aid): the adaptive round-and-log
alone on the 174 GPT-2 hooked tensor sizes -- in place on fresh data (the
hooks' call) and out of place -- timed with CUDA events around the ops only."""
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
src = torch.randn(mx, dtype=torch.float64, device="cuda", generator=g)
work = torch.empty_like(src)
out = torch.empty_like(src)


def timed(inplace: bool, reps: int = 3) -> float:
    res = []
    for r in range(reps + 1):
        evs = []
        for n in sizes:
            if inplace:
                work[:n].copy_(src[:n])  # fresh (unrounded) data, outside the timed spans
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            if inplace:
                ops.round_and_log_adaptive(work[:n], 32, int(0.005 * n), out_dtype=torch.float64, out=work[:n],
                                           check=False, tag="hooks_fwd")
            else:
                ops.round_and_log_adaptive(src[:n], 32, int(0.005 * n), out_dtype=torch.float64, out=out[:n],
                                           check=False, tag="hooks_fwd")
            e.record()
            evs.append((s, e))
        torch.cuda.synchronize()
        if r:
            res.append(sum(a.elapsed_time(b) for a, b in evs))
    return sum(res) / len(res)


print(json.dumps({"tensors": len(sizes), "elements": sum(sizes), "max": mx,
                  "in_place_ms": round(timed(True), 3), "out_of_place_ms": round(timed(False), 3)}))
