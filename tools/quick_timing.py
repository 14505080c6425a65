"""Quick CUDA-event timing of the hot kernels (development aid)."""
import json
import sys

sys.path.insert(0, ".")
import torch

from paper_2403_09603_b200 import merkle, ops, protocol, workloads


def t(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


res = {}
for lg in [int(a) for a in (sys.argv[1:] or ["26", "30"])]:
    n = 1 << lg
    x, xa = workloads.config1_pair_torch(n, 1)
    tau = workloads.TAU_CONFIG0
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    words = torch.empty(n // 4, dtype=torch.int64, device="cuda")
    p = ops.round_and_log(x, 32, tau, out=y, log_out=words, check=False)
    _, log = p.finish()
    f = log.count / n
    ms = t(lambda: ops.round_and_log(x, 32, tau, out=y, log_out=words, check=False))
    ya = torch.empty_like(y)
    ms2 = t(lambda: ops.replay(xa, 32, log, out=ya, check=False))
    b = n * (8 + 4 + 8 * f)
    res[lg] = dict(frac_logged=f, rl_ms=ms, rl_gbs=b / ms / 1e6, rp_ms=ms2, rp_gbs=b / ms2 / 1e6)
    B = int(0.005 * n)
    ms3 = t(lambda: protocol.budget_key(x, 32, B), reps=5)
    res[lg].update(budget_ms=ms3, budget_gbs_per_pass=n * 8 * 2 / ms3 / 1e6)
    del x, xa, y, ya, words, log
    torch.cuda.empty_cache()
w = torch.randn(375_000_000, device="cuda") * 0.02
ms = t(lambda: merkle.merkle_chunked(w), reps=3, warm=1)
res["merkle_1.5GB"] = dict(ms=ms, gbs=w.numel() * 4 / ms / 1e6)
print(json.dumps(res, indent=1))
