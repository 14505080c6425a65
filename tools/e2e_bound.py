"""What bounds the e2e pair (development aid): the same bytes as
ops.round_and_log_replay_host moved with no kernels -- (a) the two FP64
inputs H2D alone, (b) the same with the two FP32 outputs + log D2H running
concurrently on another stream -- next to the e2e call itself."""
import json, sys
sys.path.insert(0, ".")
import torch
from paper_2403_09603_b200 import ops, workloads

n = 1 << 26
chunk = 1 << 22
xt_d, xa_d = workloads.config1_pair_torch(n, seed=1)
xt_h = torch.empty(n, dtype=torch.float64, pin_memory=True); xt_h.copy_(xt_d)
xa_h = torch.empty(n, dtype=torch.float64, pin_memory=True); xa_h.copy_(xa_d)
yt_h = torch.empty(n, dtype=torch.float32, pin_memory=True)
ya_h = torch.empty(n, dtype=torch.float32, pin_memory=True)
log_h = torch.empty(n // 4, dtype=torch.int64, pin_memory=True)
dx = torch.empty(n, dtype=torch.float64, device="cuda")
dy = torch.empty(n, dtype=torch.float32, device="cuda")
dlog = torch.empty(n // 8, dtype=torch.int64, device="cuda")
s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def h2d_only():
    with torch.cuda.stream(s_in):
        for src in (xt_h, xa_h):
            for lo in range(0, n, chunk):
                dx[lo:lo + chunk].copy_(src[lo:lo + chunk], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s_in)


def h2d_and_d2h():
    with torch.cuda.stream(s_out):
        for dst in (yt_h, ya_h):
            for lo in range(0, n, chunk):
                dst[lo:lo + chunk].copy_(dy[lo:lo + chunk], non_blocking=True)
        log_h[: n // 8].copy_(dlog, non_blocking=True)
    h2d_only()
    torch.cuda.current_stream().wait_stream(s_out)


def e2e():
    ops.round_and_log_replay_host(xt_h, xa_h, 32, workloads.TAU_CONFIG0, yt_h, ya_h, log_h, chunk=chunk)


res = {k: round(timed(f), 3) for k, f in (("h2d_only_ms", h2d_only), ("h2d_with_d2h_ms", h2d_and_d2h), ("e2e_ms", e2e))}
res["h2d_gbs"] = round(16 * n / res["h2d_only_ms"] / 1e6, 1)
print(json.dumps(res))
