"""e2e host pipeline vs chunk size (development aid)."""
import sys, json
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import ops, workloads
n = 1 << 26
xt_d, xa_d = workloads.config1_pair_torch(n, seed=1)
xt_h = torch.empty(n, dtype=torch.float64, pin_memory=True); xt_h.copy_(xt_d)
xa_h = torch.empty(n, dtype=torch.float64, pin_memory=True); xa_h.copy_(xa_d)
del xt_d, xa_d
yt_h = torch.empty(n, dtype=torch.float32, pin_memory=True)
ya_h = torch.empty(n, dtype=torch.float32, pin_memory=True)
log_h = torch.empty(n // 4, dtype=torch.int64, pin_memory=True)
res = {}
for lg in (21, 22, 23, 24):
    f = lambda: ops.round_and_log_replay_host(xt_h, xa_h, 32, workloads.TAU_CONFIG0, yt_h, ya_h, log_h, chunk=1 << lg)
    f(); f(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): f()
    e.record(); torch.cuda.synchronize()
    res[lg] = round(s.elapsed_time(e) / 5, 3)
print(json.dumps(res))
