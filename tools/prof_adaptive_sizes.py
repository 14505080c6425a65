"""ncu driver: the adaptive chain at a few tensor sizes (development aid)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2403_09603_b200 import ops
g = torch.Generator(device="cuda"); g.manual_seed(5)
xs = [torch.randn(n, dtype=torch.float64, device="cuda", generator=g) for n in (1 << 17, 1 << 20, 6_291_456, 1 << 25)]
outs = [torch.empty_like(x) for x in xs]
for x, o in zip(xs, outs):
    ops.round_and_log_adaptive(x, 32, int(0.005 * x.numel()), out_dtype=torch.float64, out=o, check=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for x, o in zip(xs, outs):
    ops.round_and_log_adaptive(x, 32, int(0.005 * x.numel()), out_dtype=torch.float64, out=o, check=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
