"""Eager timing of one out-of-place adaptive call at 2^26 (development aid)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2403_09603_b200 import ops
n = 1 << 26
g = torch.Generator(device="cuda"); g.manual_seed(1)
x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
B = int(0.005 * n)
y = torch.empty(n, dtype=torch.float32, device="cuda")
for _ in range(3): ops.round_and_log_adaptive(x, 32, B)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20): ops.round_and_log_adaptive(x, 32, B)
b.record(); torch.cuda.synchronize()
print("single out-of-place adaptive 2^26 ms/call", a.elapsed_time(b) / 20)
