"""Quick CUDA-event timing of the fused kernels (development aid)."""
import sys, json
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import ops, workloads, merkle, protocol

def t(fn, reps=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps

res = {}
for lg in (26, 30):
    n = 1 << lg
    x, xa = workloads.config1_pair_torch(n, 1)
    tau = workloads.TAU_CONFIG0
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    words = torch.empty(n // 4, dtype=torch.int64, device="cuda")
    p = ops.round_and_log(x, 32, tau, out=y, log_out=words, check=False)
    _, log = p.finish()
    f = log.count / n
    ms = t(lambda: ops.round_and_log(x, 32, tau, out=y, log_out=words, check=False))
    gbs = n * (8 + 4 + 8 * f) / ms / 1e6
    ya = torch.empty_like(y)
    ms2 = t(lambda: ops.replay(xa, 32, log, out=ya, check=False))
    gbs2 = n * (8 + 4 + 8 * f) / ms2 / 1e6
    res[lg] = dict(frac_logged=f, rl_ms=ms, rl_gbs=gbs, rp_ms=ms2, rp_gbs=gbs2)
    del x, xa, y, ya, words, log
    torch.cuda.empty_cache()
w = torch.randn(375_000_000, device="cuda") * 0.02
ms = t(lambda: merkle.merkle_chunked(w), reps=3, warm=1)
res["merkle_1.5GB"] = dict(ms=ms, gbs=w.numel() * 4 / ms / 1e6)
x = torch.randn(1 << 26, dtype=torch.float64, device="cuda")
ms = t(lambda: protocol.kth_largest_distance(x, 32, int(0.005 * x.numel())), reps=3)
res["tau_2^26"] = dict(ms=ms, gbs=x.numel() * 8 * 5 / ms / 1e6)
print(json.dumps(res, indent=1))
