"""Development aid: run-to-run spread of the fused round-and-log / replay at
2^30 (graph replays, CUDA events per replay)."""
import json, sys
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import ops, workloads
n = 1 << 30
x = workloads.config0_x_torch_bernoulli(n, seed=30)
TAU = 1.0 if "--nolog" in sys.argv else workloads.TAU_CONFIG0  # tau >= 2^-24: nothing is logged
y = torch.empty(n, dtype=torch.float32, device="cuda")
ya = torch.empty_like(y)
words = torch.empty(n // 4, dtype=torch.int64, device="cuda")
_, log = ops.round_and_log(x, 32, TAU, out=y, log_out=words, check=False).finish()
lw = log.words
graphs = []
for fn in (lambda: ops.round_and_log(x, 32, TAU, out=y, log_out=words, check=False),
           lambda: ops.replay(x, 32, lw, out=ya, check=False)):
    s_ = torch.cuda.Stream(); s_.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_):
        fn()
    torch.cuda.current_stream().wait_stream(s_)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    graphs.append(g)
b = n * (8 + 4 + 8 * log.count / n)
res = {"rl": [], "rp": []}
order = [("rl", graphs[0])] * 3 + [("rp", graphs[1])] * 3 if "--separate" in sys.argv else \
    [("rl", graphs[0]), ("rp", graphs[1])] * 3
import time
for name, g in order:
    if "--idle" in sys.argv:
        torch.cuda.synchronize()
        time.sleep(0.5)
    if True:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(8)]
        for a, e in evs:
            a.record(); g.replay(); e.record()
        torch.cuda.synchronize()
        res[name] += [round(b / a.elapsed_time(e) / 1e6 / 6537, 3) for a, e in evs]
print(json.dumps(res))

# the same spread for a plain device copy of the same size (hardware drift?)
dst = torch.empty_like(x)
cp = []
for _ in range(24):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); dst.copy_(x); e.record()
    torch.cuda.synchronize()
    cp.append(round(2 * n * 8 / a.elapsed_time(e) / 1e6 / 6537, 3))
print(json.dumps({"copy": cp}))
