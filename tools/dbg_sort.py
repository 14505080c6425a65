import sys
sys.path.insert(0, ".")
sys.path.insert(0, "oracle")
import numpy as np, torch
import vt_oracle as oracle
from paper_2403_09603_b200 import ops, workloads
for lg, seed in [(27, 5), (26, 5), (27, 5), (27, 6)]:
    n = 1 << lg
    x = workloads.config0_x_torch(n, seed)
    y, log = ops.round_and_log(x, 32, workloads.TAU_CONFIG0)
    idx = log.indices()
    bad = torch.nonzero(idx[1:] <= idx[:-1]).flatten()
    print(lg, seed, "count", log.count, "violations", bad.numel())
    if bad.numel():
        b = int(bad[0])
        print("first at", b, idx[max(0,b-3):b+4].tolist())
        # expected
        lo = max(0, int(idx[b - 3]) - 100) if b >= 3 else 0
        xs = x[lo: lo + 20000].cpu().numpy()
        want = oracle.sparse_from_codes(oracle.direction_array(xs, 32, workloads.TAU_CONFIG0), base=lo)
        wi = (want >> 1)
        print("expected near", wi[:12].tolist())
        # super-tile of the violation
        print("super-tile", int(idx[b]) // 8192, int(idx[b+1]) // 8192)
        # total expected count via torch-free check: compare count with oracle on a sample
    del x, y, log
