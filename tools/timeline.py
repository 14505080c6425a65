"""Per-CTA timeline of rl_fused_kernel from a -DVT_TIMELINE debug build
(development aid): builds build/libvt_tl.so, runs one round-and-log, prints
when CTAs start, get data, finish ordinals, and end."""
import ctypes, subprocess, sys
from pathlib import Path
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import _device as D, _lib, build_lib, workloads

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
x = workloads.config0_x_torch(n, 1)
tau = workloads.TAU_CONFIG0
y = torch.empty(n, dtype=torch.float32, device="cuda")
words = torch.empty(n // 4, dtype=torch.int64, device="cuda")
ws = torch.zeros(int(lib.vt_round_log_workspace(n)), dtype=torch.uint8, device="cuda")
for rep in range(4):
    f = D.Flags()
    lib.vt_round_log(D.ptr(x), n, 32, float(tau), _lib.OUT_F32, D.ptr(y), D.ptr(words), words.numel(), 0, None, None,
                     None, None, 0, None, f.cnt_ptr, f.err_ptr, D.ptr(ws), ws.numel(), D.stream_ptr())
    torch.cuda.synchronize()
tl = np.zeros((1024, 64), dtype=np.uint64)
lib.vt_debug_timeline(tl.ctypes.data)
G = 444
t = tl[:G].astype(np.int64)
t0 = t[:, 0].min()
rel = (t - t0) / 1000.0  # us
print("CTA start  min/med/max us:", np.percentile(rel[:, 0], [0, 50, 100]).round(2))
print("first data min/med/max us:", np.percentile(rel[:, 1], [0, 50, 100]).round(2))
print("loop exit  min/med/max us:", np.percentile(rel[:, 2], [0, 50, 100]).round(2))
print("CTA end    min/med/max us:", np.percentile(rel[:, 3], [0, 50, 100]).round(2))
for k in range(0, 14):
    c = [rel[:, 4 + 4 * k + j] for j in range(4)]
    ok = (t[:, 4 + 4 * k] > t0) & (t[:, 7 + 4 * k] > t0)
    if ok.sum() < 10:
        break
    prev = rel[:, 3 + 4 * k] if k else rel[:, 1]
    w = (c[1] - c[0]) if k >= 3 else np.zeros(G)
    print(f"ordinal {k:2d}: top {np.median(c[0][ok]):7.2f}  ofull-wait {np.median(w[ok]):5.2f}  "
          f"writes {np.median((c[2] - (c[1] if k >= 3 else c[0]))[ok]):5.2f}  compute {np.median((c[3] - c[2])[ok]):5.2f}"
          f"  gap-from-prev {np.median((c[0] - prev)[ok]):5.2f}  n={ok.sum()}")

last = np.array([max(k for k in range(14) if t[c, 7 + 4 * k] > t0) if (t[c, 7] > t0) else 0 for c in range(G)])
print("sentinel seen  min/med/max:", np.percentile(rel[:, 60], [0, 50, 100]).round(2))
print("drain k-2 done min/med/max:", np.percentile(rel[:, 61], [0, 50, 100]).round(2))
print("drain k-1 done min/med/max:", np.percentile(rel[:, 62], [0, 50, 100]).round(2))

sm = t[:, 63]; nord = t[:, 56]; lastT = t[:, 55]
sent = rel[:, 60]; lastdone = rel[:, 58]
o = np.argsort(sent)
print("latest 12 CTAs: cta sm ordinals last_ticket last_compute_done sentinel")
for c in o[-12:]:
    print(f"  {c:4d} {sm[c]:4d} {nord[c]:3d} {lastT[c]:6d} {lastdone[c]:8.2f} {sent[c]:8.2f}")
print("earliest 6:")
for c in o[:6]:
    print(f"  {c:4d} {sm[c]:4d} {nord[c]:3d} {lastT[c]:6d} {lastdone[c]:8.2f} {sent[c]:8.2f}")
print("ordinals per CTA min/med/max", nord.min(), np.median(nord), nord.max())
# per-SM: mean sentinel by sm parity/half
for name, m in (("sm<74", sm < 74), ("sm>=74", sm >= 74), ("even", sm % 2 == 0), ("odd", sm % 2 == 1)):
    print(name, "sentinel med", np.median(sent[m]).round(2), "ordinals med", np.median(nord[m]))
# ordinals per CTA by launch wave (CTA id // 148: the first, second, third CTA
# placed on each SM), and when each wave's CTAs end
for w in range(3):
    m = (np.arange(G) // 148) == w
    print(f"CTA ids {148 * w}-{148 * w + 147}: ordinals min/med/max", nord[m].min(), np.median(nord[m]), nord[m].max(),
          " sentinel med", np.median(sent[m]).round(2))
