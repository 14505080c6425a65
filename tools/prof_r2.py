"""Round-2 profiling driver (run under ncu, one workload per invocation):
  merkle  -- configs[4] chunked Merkle over 1.5e9 FP32 params + both variants
             of the int-mix peak kernel (the roofline denominator)
  budget  -- protocol.search_tau_budget on 2^26 N(0,1) (vt_tau_budget:
             adapt_keys32_kernel + adapt_tail_kernel)
Development aid; a number printed under ncu is never a bench value."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2403_09603_b200 import _device as D  # noqa: E402
from paper_2403_09603_b200 import _lib, merkle, protocol, workloads  # noqa: E402

what = sys.argv[1]
if what == "merkle":
    w = workloads.config4_weights_torch()
    t = merkle.merkle_chunked(w)
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    for fma in (0, 1):
        _lib.call("vt_int_mix_peak_bench", D.ptr(sink), 148 * 8, 2048, fma, D.stream_ptr())
    torch.cuda.synchronize()
    print("root", t.root_hex[:16])
elif what == "budget":
    g = torch.Generator(device="cuda")
    g.manual_seed(26)
    x = torch.randn(1 << 26, dtype=torch.float64, device="cuda", generator=g)
    for _ in range(2):
        tau = protocol.search_tau_budget(x, 32, int(0.005 * x.numel()))
    print("tau", tau)
