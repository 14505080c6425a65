"""Would zero-copy (kernels reading / writing pinned host memory through UVA)
cut the per-call latency of the small-tensor channel path? (development aid)"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2403_09603_b200 import _device as D, _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rng = np.random.default_rng(0)
x = rng.normal(0, 1, n)
xh = torch.empty(n, dtype=torch.float64, pin_memory=True); xh.numpy()[:] = x
yh = torch.empty(n, dtype=torch.float64, pin_memory=True)
ph = torch.empty(n // 5 + 16, dtype=torch.uint8, pin_memory=True)
eh = torch.zeros(16, dtype=torch.uint8, pin_memory=True)
flh = torch.zeros(8, dtype=torch.int64, pin_memory=True)
fld = torch.zeros(8, dtype=torch.int64, device="cuda")
lib = _lib.lib()


def zc_call():
    # inputs and outputs in pinned host memory, flags on the device (atomics), one 64 B D2H + wait;
    # the NumPy input copied into the pinned buffer and the result copied out, as the product must
    np.copyto(xh.numpy(), x)
    fld.zero_()
    _lib.call("vt_round_log", xh.data_ptr(), n, 32, 6e-8, _lib.OUT_F64, yh.data_ptr(), None, 0, 0, None, None,
              None, ph.data_ptr(), 0, eh.data_ptr(), fld.data_ptr() + 16, fld.data_ptr(), None, 0, D.stream_ptr())
    flh.copy_(fld, non_blocking=True)
    D.sync_stream()
    return yh.numpy().copy()


zc_call()
want = np.asarray(x, dtype=np.float32).astype(np.float64)
assert np.array_equal(yh.numpy(), want), "zero-copy output differs"
for f, name in ((zc_call, "zero-copy"),):
    for _ in range(50):
        f()
    t0 = time.perf_counter()
    for _ in range(2000):
        f()
    print(f"{name} n={n}: {(time.perf_counter() - t0) / 2000 * 1e6:.1f} us per call")
from paper_2403_09603_b200 import roundlog
w = roundlog.LogWriter("/tmp/zc.vtrl", 32)
for _ in range(50):
    w.write_values_host(x, 6e-8)
t0 = time.perf_counter()
for _ in range(2000):
    w.write_values_host(x, 6e-8)
print(f"staged (product) n={n}: {(time.perf_counter() - t0) / 2000 * 1e6:.1f} us per call")
