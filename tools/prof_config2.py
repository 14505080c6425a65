"""ncu driver for configs[2]: one eager sweep of the 161-tensor adaptive round-and-log (development aid)."""
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
total = sum(x.numel() for x in xs)
ys = torch.empty(total, dtype=torch.float32, device="cuda")
budgets = [int(0.005 * x.numel()) for x in xs]
words = torch.empty(sum(budgets) + len(xs), dtype=torch.int64, device="cuda")


def run():
    off = woff = 0
    for x, B in zip(xs, budgets):
        n = x.numel()
        ops.round_and_log_adaptive(x, 32, B, out=ys[off:off + n], log_out=words[woff:woff + B + 1], check=False)
        off += n
        woff += B + 1


run()
torch.cuda.synchronize()
print("sizes: min", min(x.numel() for x in xs), "median", int(np.median([x.numel() for x in xs])), "max",
      max(x.numel() for x in xs), "total", total)
torch.cuda.cudart().cudaProfilerStart()
run()
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
