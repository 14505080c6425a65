"""Phase timeline of adapt_tail_kernel (the budget search's cooperative tail)
from a -DVT_TIMELINE debug build (development aid): per-CTA stamps after the
candidate histogram, each grid sync, the digit compaction and the exact
selection (block 0)."""
import ctypes, subprocess, sys
from pathlib import Path
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import _lib, build_lib

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
so = Path("paper_2403_09603_b200/build/libvt_tl.so")
objs = []
for src in build_lib.SOURCES:
    o = Path("paper_2403_09603_b200/build") / ("tl_" + Path(src).stem + ".o")
    subprocess.run([build_lib.NVCC, *build_lib.FLAGS, "-DVT_TIMELINE", "-c", str(build_lib.CSRC / src), "-o", str(o)], check=True)
    objs.append(str(o))
subprocess.run([build_lib.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(so), *objs], check=True)
_lib.LIB_PATH = so.resolve()  # the timeline build, loaded lazily by the first call
from paper_2403_09603_b200 import protocol  # noqa: E402
lib = _lib.lib()
lib.vt_debug_timeline_tail.argtypes = [ctypes.c_void_p]
g = torch.Generator(device="cuda")
g.manual_seed(lg)
x = torch.randn(1 << lg, dtype=torch.float64, device="cuda", generator=g)
for _ in range(3):
    tau = protocol.search_tau_budget(x, 32, int(0.005 * x.numel()))
torch.cuda.synchronize()
tl = np.zeros((1024, 8), dtype=np.uint64)
lib.vt_debug_timeline_tail(tl.ctypes.data)
cand2 = int(tl[1023, 0])
t = tl[:1023].astype(np.int64)
used = t[:, 0] > 0
t = t[used]
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0
print(f"CTAs {used.sum()}, digit keys (cand2) {cand2}, tau {tau!r}")
for i, name in enumerate(["start", "hist done", "sync1 out", "digit done", "sync2 out", "exact done"]):
    print(f"{name:11s} min/med/max us:", np.percentile(rel[:, i], [0, 50, 100]).round(2))
