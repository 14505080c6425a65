"""Per-call latency of the reference-API channels on small NumPy tensors
(the f2 / trend regime: a few thousand elements per call) -- where the time
goes (development aid)."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2403_09603_b200 import protocol, roundlog

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
rng = np.random.default_rng(0)
xs = [rng.normal(0, 1, n) for _ in range(64)]
w = roundlog.LogWriter("/tmp/ch.vtrl", 32)
ch = protocol.GpuTrainerChannel(w, 32)
for x in xs[:8]:
    ch.process(x, 6e-8)
torch.cuda.synchronize()
reps = 2000
t0 = time.perf_counter()
for i in range(reps):
    ch.process(xs[i % 64], 6e-8)
dt = (time.perf_counter() - t0) / reps
print(f"trainer channel n={n}: {dt * 1e6:.1f} us per call")
pr = cProfile.Profile()
pr.enable()
for i in range(500):
    ch.process(xs[i % 64], 6e-8)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
