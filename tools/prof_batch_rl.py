"""ncu driver (development aid): the batched rounding pass over the 161
configs[2] tensors vs the same pass over one flat tensor of the same total
size (batch of 1) and the single-tensor adaptive call on that flat tensor."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2403_09603_b200 import ops, workloads
shapes = workloads.resnet50_tensors()
sig = workloads.config2_sigmas(len(shapes))
g = torch.Generator(device="cuda")
g.manual_seed(2)
xs = [torch.randn(int(np.prod(s)), dtype=torch.float64, device="cuda", generator=g) * float(sig[i])
      for i, (_, s) in enumerate(shapes)]
budgets = [int(0.005 * x.numel()) for x in xs]
total = sum(x.numel() for x in xs)
flat = torch.randn(total, dtype=torch.float64, device="cuda", generator=g)
ys = [torch.empty(x.numel(), dtype=torch.float32, device="cuda") for x in xs]
yf = torch.empty(total, dtype=torch.float32, device="cuda")
runs = [lambda: ops.round_and_log_adaptive_batch(xs, 32, budgets, outs=ys, check=False),
        lambda: ops.round_and_log_adaptive_batch([flat], 32, [int(0.005 * total)], outs=[yf], check=False),
        lambda: ops.round_and_log_adaptive(flat, 32, int(0.005 * total), out=yf, check=False)]
for r in runs:
    r(); r()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for r in runs:
    r()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
