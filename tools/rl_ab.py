"""A/B timing of the round-and-log op at a few sizes (development aid; env vars pick variants)."""
import json, os, sys
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import ops, workloads


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


out = {}
for lg in [int(a) for a in sys.argv[1:]]:
    n = 1 << lg
    x, _ = workloads.config1_pair_torch(n, 1)
    tau = workloads.TAU_CONFIG0
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    words = torch.empty(n // 4, dtype=torch.int64, device="cuda")
    p = ops.round_and_log(x, 32, tau, out=y, log_out=words, check=False)
    _, log = p.finish()
    f = log.count / n
    ms = t(lambda: ops.round_and_log(x, 32, tau, out=y, log_out=words, check=False))
    out[lg] = dict(ms=round(ms, 4), gbs=round(n * (12 + 8 * f) / ms / 1e6, 1))
    del x, y, words, log
    torch.cuda.empty_cache()
print(os.environ.get("TAG", ""), json.dumps(out))
