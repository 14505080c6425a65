"""In-place adaptive round-and-log (the GPT-2 hooks' call) on GPT-2 tensor
sizes, graph-timed back to back (development aid; A/B via VTRAIN_B200_LIB)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2403_09603_b200 import ops  # noqa: E402

for n in (8 * 1024 * 768, 3 * 8 * 1024 * 768, 4 * 8 * 1024 * 768):
    g = torch.Generator(device="cuda")
    g.manual_seed(n)
    src = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    x = src.clone()
    B = int(0.005 * n)
    logw = torch.empty(B + 1, dtype=torch.int64, device="cuda")
    taus = torch.empty(1, dtype=torch.float64, device="cuda")
    fl = torch.zeros(6, dtype=torch.int64, device="cuda")

    def call():
        x.copy_(src)  # fresh FP64 values each time (in place rounds them)
        ops.round_and_log_adaptive(x, 32, B, out_dtype=torch.float64, out=x, log_out=logw, check=False,
                                   tau_out=taus, flags_out=fl)

    def copy_only():
        x.copy_(src)

    gc, g0 = bench._capture(call), bench._capture(copy_only)
    ms = bench._time(gc.replay, 20) - bench._time(g0.replay, 20)
    print(f"n={n}: in-place adaptive {ms * 1e3:.1f} us ({n * 24 / ms / 1e6:.0f} GB/s at 24 B/elem)")
