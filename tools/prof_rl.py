"""ncu driver: a few launches of the round-and-log op at 2^LOG2 (development aid)."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import ops, workloads

n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 26)
x, _ = workloads.config1_pair_torch(n, 1)
tau = workloads.TAU_CONFIG0
y = torch.empty(n, dtype=torch.float32, device="cuda")
words = torch.empty(n // 4, dtype=torch.int64, device="cuda")
for _ in range(4):
    ops.round_and_log(x, 32, tau, out=y, log_out=words, check=False)
torch.cuda.synchronize()
print("ok")
