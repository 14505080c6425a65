"""A/B of the bench's pair step (round-and-log then replay, graph-replayed
back to back) at a few sizes (development aid; VTRAIN_B200_LIB picks the build).
Prints per-size rl / rp / pair ms and fractions of the copy peak."""
import json, os, sys
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import ops, workloads

PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6537.0


def graph(fn, s):
    with torch.cuda.stream(s):
        fn(); fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        fn()
    return g


out = {}
s = torch.cuda.Stream()
for lg in [int(a) for a in sys.argv[1:]]:
    n = 1 << lg
    xt, xa = workloads.config1_pair_torch(n, 1)
    tau = workloads.TAU_CONFIG0
    y, ya = torch.empty(n, dtype=torch.float32, device="cuda"), torch.empty(n, dtype=torch.float32, device="cuda")
    words = torch.empty(n // 4, dtype=torch.int64, device="cuda")
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        _, log = ops.round_and_log(xt, 32, tau, out=y, log_out=words, check=False).finish()
    lw = words[:log.count]
    gt = graph(lambda: ops.round_and_log(xt, 32, tau, out=y, log_out=words, check=False), s)
    ga = graph(lambda: ops.replay(xa, 32, lw, out=ya, check=False), s)
    steps = 40 if lg <= 26 else 10
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    with torch.cuda.stream(s):
        for _ in range(5):
            gt.replay(); ga.replay()
        for e in ev:
            e[0].record(s); gt.replay(); e[1].record(s); ga.replay(); e[2].record(s)
    torch.cuda.synchronize()
    rl = sum(e[0].elapsed_time(e[1]) for e in ev) / steps
    rp = sum(e[1].elapsed_time(e[2]) for e in ev) / steps
    b = n * (12 + 8 * log.count / n)
    out[lg] = dict(rl_ms=round(rl, 4), rp_ms=round(rp, 4), rl=round(b / rl / 1e6 / PEAK, 4), rp=round(b / rp / 1e6 / PEAK, 4),
                   pair=round(2 * b / (rl + rp) / 1e6 / PEAK, 4))
    assert torch.equal(y.view(torch.int32), ya.view(torch.int32))
    del xt, xa, y, ya, words, lw, log, gt, ga
    torch.cuda.empty_cache()
print(os.environ.get("TAG", ""), json.dumps(out), flush=True)
