"""Where the fused round-and-log's steady state goes (development aid):
graph-timed rl at 2^26 / 2^28 with (a) FP32 out + log (the product),
(b) no output stores (OUT_NONE), (c) nothing logged (tau = 1), (d) both,
next to the replay of the same tensor."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2403_09603_b200 import _device as D  # noqa: E402
from paper_2403_09603_b200 import _lib, ops, workloads  # noqa: E402

peak, _ = bench.peaks()
for lg in (26, 28):
    n = 1 << lg
    x = workloads.config0_x_torch_bernoulli(n, seed=lg)
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    words = torch.empty(n // 4, dtype=torch.int64, device="cuda")
    ws = torch.zeros(int(_lib.lib().vt_round_log_workspace(n)), dtype=torch.uint8, device="cuda")
    f = D.Flags()

    def rl(kind, tau):
        def fn():
            _lib.call("vt_round_log", D.ptr(x), n, 32, float(tau), kind, D.ptr(y), D.ptr(words), words.numel(), 0,
                      None, None, None, None, 0, None, f.cnt_ptr, f.err_ptr, D.ptr(ws), ws.numel(), D.stream_ptr())
        return fn

    res = {}
    for name, kind, tau in (("f32+log", _lib.OUT_F32, workloads.TAU_CONFIG0), ("none+log", _lib.OUT_NONE,
                            workloads.TAU_CONFIG0), ("f32+nolog", _lib.OUT_F32, 1.0), ("none+nolog", _lib.OUT_NONE, 1.0)):
        g = bench._capture(rl(kind, tau))
        ms = bench._time(g.replay, 10)
        res[name] = round(ms, 4)
    _, log = ops.round_and_log(x, 32, workloads.TAU_CONFIG0, out=y, log_out=words, check=False).finish()
    lw = log.words
    ya = torch.empty_like(y)
    g = bench._capture(lambda: ops.replay(x, 32, lw, out=ya, check=False))
    res["replay"] = round(bench._time(g.replay, 10), 4)
    ideal = n * (8 + 4 + 8 * log.count / n) / peak / 1e6
    print(f"2^{lg}: ms {res}  ideal(f32+log at copy peak) {ideal:.4f}  read-only ideal {8 * n / peak / 1e6:.4f}")
    del x, y, words, ws, ya, lw
    torch.cuda.empty_cache()
