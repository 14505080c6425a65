"""configs[2] time breakdown (development aid): the 161-tensor adaptive sweep
against lower bounds -- plain round-and-log of the same tensors at a fixed tau
(8 streams / 1 stream) and one round-and-log over a flat buffer of the same
total size.  Every variant is one CUDA graph, timed by CUDA events."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_2403_09603_b200 import ops, workloads



def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


shapes = workloads.resnet50_tensors()
sig = workloads.config2_sigmas(len(shapes))
gen = torch.Generator(device="cuda")
gen.manual_seed(2)
xs = [torch.randn(int(np.prod(s)), dtype=torch.float64, device="cuda", generator=gen) * float(sig[i])
      for i, (_, s) in enumerate(shapes)]
total = sum(x.numel() for x in xs)
ys = torch.empty(total, dtype=torch.float32, device="cuda")
budgets = [int(0.005 * x.numel()) for x in xs]
words = torch.empty(sum(budgets) + len(xs), dtype=torch.int64, device="cuda")
big_words = torch.empty(total // 8, dtype=torch.int64, device="cuda")
tau = 0.995 * 2.0 ** -24


def multi(fn, n_streams):
    side = [torch.cuda.Stream() for _ in range(n_streams)]

    def run():
        off = woff = 0
        main = torch.cuda.current_stream()
        for s_ in side:
            s_.wait_stream(main)
        for i, (x, B) in enumerate(zip(xs, budgets)):
            n = x.numel()
            with torch.cuda.stream(side[i % n_streams]):
                fn(i, x, ys[off:off + n], words[woff:woff + B + 1], f"t{n_streams}_{i % n_streams}")
            off += n
            woff += B + 1
        for s_ in side:
            main.wait_stream(s_)
    return run


def adaptive(i, x, y, w, tag):
    ops.round_and_log_adaptive(x, 32, budgets[i], out=y, log_out=w, check=False, tag=tag)


def plain(i, x, y, w, tag):
    ops.round_and_log(x, 32, tau, out=y, log_out=big_words[:w.numel() * 4], check=False)


flat = torch.randn(total, dtype=torch.float64, device="cuda", generator=gen)
res = {
    "elements": total,
    "sizes": sorted(x.numel() for x in xs),
    "adaptive_8s_ms": timed(multi(adaptive, 8)),
    "adaptive_1s_ms": timed(multi(adaptive, 1)),
    "adaptive_16s_ms": timed(multi(adaptive, 16)),
    "plain_1s_ms": timed(multi(plain, 1)),
    "flat_plain_ms": timed(lambda: ops.round_and_log(flat, 32, tau, out=ys, log_out=big_words, check=False)),
}
print(json.dumps(res))
