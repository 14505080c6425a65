"""ncu driver: one configs[2] batched adaptive sweep (development aid).
ncu --profile-from-start off --metrics gpu__time_duration.sum python tools/prof_batch.py"""
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
ys = [torch.empty(x.numel(), dtype=torch.float32, device="cuda") for x in xs]
ws = [torch.empty(b + 1, dtype=torch.int64, device="cuda") for b in budgets]
for _ in range(2):
    ops.round_and_log_adaptive_batch(xs, 32, budgets, outs=ys, log_outs=ws, check=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
ops.round_and_log_adaptive_batch(xs, 32, budgets, outs=ys, log_outs=ws, check=False)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
