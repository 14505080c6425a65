"""Per-CTA timeline of rp_fused_kernel from a -DVT_TIMELINE debug build (development aid)."""
import ctypes, subprocess, sys
from pathlib import Path
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import _device as D, _lib, build_lib, ops, workloads

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
so = Path("paper_2403_09603_b200/build/libvt_tl.so")
objs = []
for src in build_lib.SOURCES:
    o = Path("paper_2403_09603_b200/build") / ("tl_" + Path(src).stem + ".o")
    subprocess.run([build_lib.NVCC, *build_lib.FLAGS, "-DVT_TIMELINE", "-c", str(build_lib.CSRC / src), "-o", str(o)], check=True)
    objs.append(str(o))
subprocess.run([build_lib.NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(so), *objs], check=True)
lib = ctypes.CDLL(str(so.resolve()))
for name, (ret, args) in _lib.EXPORTS.items():
    fn = getattr(lib, name); fn.restype = ret; fn.argtypes = args
lib.vt_debug_timeline.argtypes = [ctypes.c_void_p]
n = 1 << lg
xt, xa = workloads.config1_pair_torch(n, 1)
tau = workloads.TAU_CONFIG0
_, log = ops.round_and_log(xt, 32, tau)
w = log.words[: log.count].contiguous()
y = torch.empty(n, dtype=torch.float32, device="cuda")
ws = torch.zeros(int(lib.vt_replay_workspace(n)), dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
for rep in range(4):
    f = D.Flags()
    lib.vt_replay(D.ptr(xa), n, 32, _lib.LOG_SPARSE, D.ptr(w), w.numel(), 0, _lib.OUT_F32, D.ptr(y), f.cnt_ptr,
                  f.err_ptr, D.ptr(ws), ws.numel(), D.stream_ptr())
    torch.cuda.synchronize()
tl = np.zeros((1024, 64), dtype=np.uint64)
lib.vt_debug_timeline(tl.ctypes.data)
G = 443
t = tl[:G].astype(np.int64)
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0
for name, i in (("CTA start", 0), ("first data", 1), ("CTA end", 3)):
    print(f"{name:10s} min/med/max us:", np.percentile(rel[:, i], [0, 5, 50, 95, 100]).round(2))
tw = t[:, 10:14].astype(np.float64)
print("compute thread 0 waits (us, min/5%/med/95%/max over CTAs):")
for name, col in (("ticket top (search result)", 0), ("next ticket (search result)", 1), ("TMA data (full)", 2)):
    print(f"  {name:28s}", np.percentile(tw[:, col] / 1000.0, [0, 5, 50, 95, 100]).round(2))
print("tiles per CTA min/med/max", tw[:, 3].min(), np.median(tw[:, 3]), tw[:, 3].max())
