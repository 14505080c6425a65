"""ncu driver for the budget-search passes (config-0 data and N(0, sigma) data)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import protocol, workloads
n = 1 << 26
x0 = workloads.config0_x_torch_bernoulli(n, 1)
x1 = torch.randn(n, dtype=torch.float64, device="cuda") * 0.05
B = int(0.005 * n)
for _ in range(2):
    protocol.budget_key(x0, 32, B)
    protocol.budget_key(x1, 32, B)
torch.cuda.synchronize()
import time
for name, x in (("config0", x0), ("normal", x1)):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        protocol.budget_key(x, 32, B)
    e.record(); torch.cuda.synchronize()
    print(name, s.elapsed_time(e) / 5, "ms")
