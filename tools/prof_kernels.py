"""Short driver for ncu: 2 warm-up + 2 profiled launches of each hot kernel at 2^26."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import merkle, ops, protocol, workloads

n = 1 << 26
x, xa = workloads.config1_pair_torch(n, 1)
tau = workloads.TAU_CONFIG0
y = torch.empty(n, dtype=torch.float32, device="cuda")
words = torch.empty(n // 4, dtype=torch.int64, device="cuda")
_, log = ops.round_and_log(x, 32, tau, out=y, log_out=words)
ya = torch.empty_like(y)
for _ in range(4):
    ops.round_and_log(x, 32, tau, out=y, log_out=words, check=False)
    ops.replay(xa, 32, log.words, out=ya, check=False)
w = torch.randn(1 << 26, device="cuda") * 0.02
for _ in range(3):
    merkle.merkle_chunked(w)
for _ in range(3):
    protocol.kth_largest_distance(x, 32, int(0.005 * n))
torch.cuda.synchronize()
print("ok")
