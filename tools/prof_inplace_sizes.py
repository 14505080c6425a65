"""ncu driver (development aid): the in-place adaptive chain (the hooks'
call) at the GPT-2 configs[3] tensor sizes."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import ops
g = torch.Generator(device="cuda"); g.manual_seed(5)
sizes = [1 << 17, 6_291_456, 18_874_368, 25_165_824]
src = [torch.randn(n, dtype=torch.float64, device="cuda", generator=g) for n in sizes]
work = [s.clone() for s in src]
for w, s in zip(work, src):
    ops.round_and_log_adaptive(w, 32, int(0.005 * w.numel()), out_dtype=torch.float64, out=w, check=False, tag="ip")
    w.copy_(s)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for w in work:
    ops.round_and_log_adaptive(w, 32, int(0.005 * w.numel()), out_dtype=torch.float64, out=w, check=False, tag="ip")
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
