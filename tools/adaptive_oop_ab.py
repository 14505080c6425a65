"""Out-of-place adaptive round-and-log (ops.round_and_log_adaptive), graph-timed at a few sizes (development aid; VTRAIN_B200_LIB picks the build)."""
import json, os, sys
sys.path.insert(0, ".")
import torch
import bench
from paper_2403_09603_b200 import ops
out = {}
for lg in [int(a) for a in sys.argv[1:]]:
    n = 1 << lg
    g = torch.Generator(device="cuda"); g.manual_seed(lg)
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    B = int(0.005 * n)
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    logw = torch.empty(B + 1, dtype=torch.int64, device="cuda")
    tau = torch.empty(1, dtype=torch.float64, device="cuda")
    fl = torch.zeros(6, dtype=torch.int64, device="cuda")
    call = lambda: ops.round_and_log_adaptive(x, 32, B, out=y, log_out=logw, check=False, tau_out=tau, flags_out=fl)  # noqa: E731
    gr = bench._capture(call)
    ms = bench._time(gr.replay, 20)
    out[lg] = round(ms * 1e3, 1)
print(os.environ.get("TAG", ""), json.dumps(out))
