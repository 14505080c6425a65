"""Fixed-cost probe at mid sizes (2^22..2^28): per-launch time of the fused
round-and-log / replay when captured alone vs 16 back-to-back in one graph,
next to a plain FP64 -> FP32 conversion copy (torch) of the same bytes --
what any streaming kernel pays for its ramp and drain at that size."""

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2403_09603_b200 import ops, workloads  # noqa: E402

peak, _ = bench.peaks()
out = {}
for lg in [int(a) for a in sys.argv[1:]] or [22, 24, 26, 28]:
    n = 1 << lg
    x = workloads.config0_x_torch_bernoulli(n, seed=lg)
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    ya = torch.empty_like(y)
    words = torch.empty(max(n // 4, 1024), dtype=torch.int64, device="cuda")
    _, log = ops.round_and_log(x, 32, workloads.TAU_CONFIG0, out=y, log_out=words, check=False).finish()
    lw = log.words
    b = n * (8 + 4 + 8 * log.count / n)
    rl = lambda: ops.round_and_log(x, 32, workloads.TAU_CONFIG0, out=y, log_out=words, check=False)  # noqa: E731
    rp = lambda: ops.replay(x, 32, lw, out=ya, check=False)  # noqa: E731
    cp = lambda: y.copy_(x)  # noqa: E731
    r = {}
    for name, fn, bytes_ in (("round_log", rl, b), ("replay", rp, b), ("copy_f64_to_f32", cp, 12 * n)):
        g1 = bench._capture(fn)
        g16 = bench._capture(lambda: [fn() for _ in range(16)])
        ms1 = bench._time(g1.replay, 20)
        ms16 = bench._time(g16.replay, 5) / 16
        r[name] = {"ms_single": round(ms1, 4), "ms_in_16": round(ms16, 4),
                   "frac_single": round(bytes_ / ms1 / 1e6 / peak, 4), "frac_in_16": round(bytes_ / ms16 / 1e6 / peak, 4)}
    out[f"2^{lg}"] = r
    del x, y, ya, words, lw
    torch.cuda.empty_cache()
print(json.dumps(out, indent=1))
