import sys, os
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import torch, bench
from paper_2403_09603_b200 import merkle, workloads
w = workloads.config4_weights_torch()
t = merkle.merkle_chunked(w)
ms = bench._time(lambda: merkle.merkle_chunked(w), reps=5, warm=2)
print(os.environ.get("VT_SHA_ALU_ADDS", "0"), "ms", round(ms, 3), "GB/s", round(6e9 / ms / 1e6, 1), "root", t.root_hex[:16])
