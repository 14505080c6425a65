"""Benchmark of the vtrain hot path on B200 (driver contract: one JSON line).

Workload (BASELINE.json configs[1], the config the metric is quoted on):
trainer/auditor replay pair on 2^26 FP64 elements per GPU -- the trainer
tensor has the config-0 distribution (90% N(0,1), 10% exact FP32 midpoints
perturbed by 2^-40 relative), the auditor tensor is the trainer tensor with
a seeded 5% moved one FP64 ulp.  One step = fused round-and-log of the
trainer tensor (FP32 out + sparse log) + fused replay of the auditor tensor
with that log (FP32 out + correction count).  Multi-GPU: weak scaling,
every rank owns its own 2^26-element shard with global indices, and the
exchange step is the NCCL all-gather of per-rank log counts.

``value`` = algorithmic bytes of the step / device time, GB/s (whole job):
  per element  round-and-log 8 (x) + 4 (FP32 out) + 8 f (sparse words)
               replay        8 (x') + 4 (FP32 out) + 8 f (sparse words read)
with f the logged fraction.  Inputs are 4x L2 (no flush needed).

``--impl reference`` times the reference algorithm on the host cores
(the oracle port of vtrain's NumPy code, oracle/vt_oracle.py -- the
reference is pure Python and cannot travel to the GPU box) on a bounded
sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "round-and-log / replay GB/s (fraction of HBM peak) at 1/2/4/8 B200 vs CPU ref"
FALLBACK_HBM = 6650.0


def peaks() -> tuple[float, str]:
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


def traffic_for(kernel: str, n: int):
    """dram bytes per launch from the committed ncu --set full capture, scaled
    per element (the capture may use a smaller n); None if absent."""
    p = REPO / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())[kernel]
        return d["dram_bytes_per_elem"] * n
    except Exception:
        return None


class Clocks:
    """NVML sampler thread (every ~5 ms) running during the timed region:
    SM clock, max SM clock and the active throttle reasons."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.mask = [], 0
        self.max_mhz = None
        self._stop = False
        self.ok = False

    def _loop(self):
        import pynvml as N
        h = N.nvmlDeviceGetHandleByIndex(self.index)
        while not self._stop:
            try:
                self.sm.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                self.mask |= N.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        import threading
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            self.ok = True
            self.th = threading.Thread(target=self._loop, daemon=True)
            self.th.start()
        except Exception:
            self.ok = False
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop = True
            self.th.join(timeout=2)
        return False

    def summary(self) -> dict:
        if not self.ok or not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        reasons = sorted(k for k, bit in self.REASONS.items() if self.mask & bit)
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.sm), "sm_mhz_min": min(self.sm)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2403_09603_b200 import _lib, ops, workloads
    from paper_2403_09603_b200 import dist as vdist

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    n = 1 << args.log2n
    tau = workloads.TAU_CONFIG0
    base = rank * n
    xt, xa = workloads.config1_pair_torch(n, seed=1 + rank, device=dev)
    y_t = torch.empty(n, dtype=torch.float32, device=dev)
    y_a = torch.empty(n, dtype=torch.float32, device=dev)
    words = torch.empty(n // 4, dtype=torch.int64, device=dev)

    # the auditor receives the log with its length (as a file carries it);
    # take it from one untimed trainer pass
    p0 = ops.round_and_log(xt, 32, tau, out=y_t, log_out=words, global_base=base, check=False)
    _, log0 = p0.finish()
    count = log0.count
    log_words = words[:count]

    def trainer():
        return ops.round_and_log(xt, 32, tau, out=y_t, log_out=words, global_base=base, check=False)

    def auditor():
        return ops.replay(xa, 32, log_words, out=y_a, global_base=base, check=False)[1]

    def exchange(p):
        if world > 1:  # the exchange step: all-gather of per-rank log counts
            vdist.all_gather_counts(p.flags.buf[2:3])

    for _ in range(args.warmup):
        p = trainer()
        exchange(p)
        fl = auditor()
    torch.cuda.synchronize()
    # verify once (outside the timed region): auditor output == trainer output, no errors
    err_t, cnt_t = p.flags.read()
    err_a, cnt_a = fl.read()
    assert err_t == 0 and err_a == 0 and cnt_t[0] == count, (err_t, err_a, cnt_t, count)
    ok_equal = bool(torch.equal(y_t.view(torch.int32), y_a.view(torch.int32)))

    # Each operator is captured once into a CUDA graph (its kernels + flag
    # resets); the timed loop replays the graphs, so host launch latency does
    # not leak into the device timeline.
    graphs = None
    if not args.no_graph:
        g_t, g_a = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):
            trainer()
            auditor()
        torch.cuda.current_stream(dev).wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g_t):
            pg = trainer()
        with torch.cuda.graph(g_a):
            flg = auditor()
        g_t.replay()
        g_a.replay()
        torch.cuda.synchronize()
        assert pg.flags.read()[1][0] == count and flg.read()[0] == 0
        graphs = (g_t, g_a, pg)

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    mids = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for i in range(args.steps):
            starts[i].record()
            if graphs:
                graphs[0].replay()
                mids[i].record()
                exchange(graphs[2])
                graphs[1].replay()
            else:
                p = trainer()
                mids[i].record()
                exchange(p)
                auditor()
            ends[i].record()
        t1.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms_total = t0.elapsed_time(t1)
    rl_ms = statistics.mean(starts[i].elapsed_time(mids[i]) for i in range(args.steps))
    rp_ms = statistics.mean(mids[i].elapsed_time(ends[i]) for i in range(args.steps))
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    f = count / n
    per_elem = (8 + 4 + 8 * f) * 2
    value = world * n * per_elem / (ms_step * 1e-3) / 1e9
    rl_bytes = n * (8 + 4 + 8 * f)
    rp_bytes = n * (8 + 4 + 8 * f)
    peak, peak_src = peaks()

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, n, tau, base, dev, world)

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    cpu = None if (world > 1 or args.no_cpu) else cpu_baseline(args)
    rl_ach = rl_bytes / (rl_ms * 1e-3) / 1e9
    rp_ach = rp_bytes / (rp_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64->f32 (int64 log words)",
        "data": "synthetic (seeded, BASELINE configs[1] distribution, generated in HBM)",
        "config": {"workload": f"configs[1]: round-and-log + replay pair, 2^{args.log2n} FP64 elements per GPU, "
                               f"b_r=32, tau=0x1.ff7ced916872bp-25",
                   "n_per_gpu": n, "logged_fraction": round(f, 6), "parallelism": f"dp{world} (contiguous shards)",
                   "l2": "no flush: every step streams 2 x 512 MiB of FP64 (>= 4x the 126 MB L2)",
                   "auditor_equals_trainer_bitwise": ok_equal,
                   "launch": "cuda graphs (one per operator)" if graphs else "eager"},
        "roofline": {"bound": "hbm",
                     "kernel": "round-and-log op: rl_fused_kernel (single pass: TMA-pipelined rnd + direction + "
                               "ballot staging, in-kernel decoupled look-back, final log words)",
                     "achieved": round(rl_ach, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(rl_ach / peak, 4), "traffic": traffic_for("round_log", n),
                     "algorithmic_bytes_per_launch": int(rl_bytes), "avg_launch_ms": round(rl_ms, 4),
                     "peak_source": peak_src},
        "kernels": {"replay: rp_fused_kernel": {"achieved": round(rp_ach, 1), "frac": round(rp_ach / peak, 4),
                                      "avg_launch_ms": round(rp_ms, 4), "algorithmic_bytes_per_launch": int(rp_bytes),
                                      "traffic": traffic_for("replay", n)}},
        "clocks": clk.summary(),
        "gpu_launches": 2 * args.steps,  # rl_fused + rp_fused per step
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    if args.sweep:
        line["sweep"] = sweep(args.sweep)
    if args.extras and world == 1:
        line["extras"] = {"configs[4]_size_sweep": sweep([20, 24, 26, 28, 30, 32]),
                          "vtrl_codec_2^26": vtrl_codec(26),
                          "configs[2]_resnet50_budget": config2(),
                          "configs[3]_gpt2_fp64_step": config3_gpt2(),
                          "configs[4]_merkle_1.5B": config4_merkle()}
        if not args.no_cpu:
            cores = len(os.sched_getaffinity(0))
            line["extras"]["configs[4]_merkle_1.5B"]["cpu_baseline"] = cpu_merkle(1 << 16, cores)
            line["extras"]["configs[2]_resnet50_budget"]["cpu_baseline"] = cpu_adaptive(1 << 22)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, n, tau, base, dev, world: int = 1):
    """Same step through the public API with pinned host buffers: H2D of both
    FP64 inputs, both kernels, D2H of both FP32 outputs and the sparse log.
    Whole job: every rank's bytes over the slowest rank's time."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2403_09603_b200 import ops, workloads

    xt_d, xa_d = workloads.config1_pair_torch(n, seed=1, device=dev)
    xt_h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    xa_h = torch.empty(n, dtype=torch.float64, pin_memory=True)
    xt_h.copy_(xt_d)
    xa_h.copy_(xa_d)
    del xt_d, xa_d
    yt_h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    ya_h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    log_h = torch.empty(n // 4, dtype=torch.int64, pin_memory=True)
    res = {}

    def one():
        cnt, corr, log_bytes = ops.round_and_log_replay_host(xt_h, xa_h, 32, tau, yt_h, ya_h, log_h,
                                                             global_base=base)
        res["log"] = cnt
        res["corr"] = corr

    for _ in range(2):
        one()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    steps = max(3, min(args.steps, 10))
    s.record()
    for _ in range(steps):
        one()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / steps
    cnt = res["log"]
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        c = torch.tensor([cnt], dtype=torch.int64, device=dev)
        dist.all_reduce(c)
        cnt = int(c.item())
    f = cnt / (n * world)
    v = world * n * (8 + 4 + 8 * f) * 2 / (ms * 1e-3) / 1e9
    # the link this leg is bound by: a plain pinned 1 GiB host -> device copy on this box
    big_h = torch.empty(1 << 27, dtype=torch.float64, pin_memory=True)
    big_d = torch.empty(1 << 27, dtype=torch.float64, device=dev)
    big_d.copy_(big_h, non_blocking=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(3):
        big_d.copy_(big_h, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    h2d_peak = 3 * big_h.numel() * 8 / (s.elapsed_time(e) * 1e-3) / 1e9
    h2d_rate = 16 * n / (ms * 1e-3) / 1e9
    del big_h, big_d
    return {"value": round(v, 2), "unit": "GB/s", "ms_per_step": round(ms, 3),
            "h2d_bytes_per_step": 16 * n * world, "d2h_bytes_per_step": 8 * n * world + 8 * cnt,
            "h2d_gbs_per_gpu": round(h2d_rate, 1), "h2d_copy_peak_gbs": round(h2d_peak, 1),
            "h2d_frac_of_copy_peak": round(h2d_rate / h2d_peak, 3),
            "path": "ops.round_and_log_replay_host (chunked H2D / kernel / D2H on 3 streams)"}


def _time(fn, reps: int, warm: int = 2) -> float:
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def sweep(log2s) -> dict:
    """configs[4] size sweep: round-and-log and replay at 2^20 .. 2^32 (config-0
    distribution, Bernoulli 10% midpoints; 2^20 is L2-resident).  Each operator
    is captured in a CUDA graph and the graph replays are timed (as for the
    headline); the eager per-call time (host overhead included) is kept too."""
    import torch

    from paper_2403_09603_b200 import ops, workloads
    peak, _ = peaks()
    out = {}
    for lg in log2s:
        n = 1 << lg
        x = workloads.config0_x_torch_bernoulli(n, seed=lg)
        y = torch.empty(n, dtype=torch.float32, device="cuda")
        words = torch.empty(max(n // 4, 1024), dtype=torch.int64, device="cuda")
        _, log = ops.round_and_log(x, 32, workloads.TAU_CONFIG0, out=y, log_out=words, check=False).finish()
        reps = 10 if lg <= 30 else 4
        ya = torch.empty_like(y)
        lw = log.words
        rl = lambda: ops.round_and_log(x, 32, workloads.TAU_CONFIG0, out=y, log_out=words, check=False)  # noqa: E731
        rp = lambda: ops.replay(x, 32, lw, out=ya, check=False)  # noqa: E731
        ms_e, ms2_e = _time(rl, reps), _time(rp, reps)
        graphs = []
        for fn in (rl, rp):
            s_ = torch.cuda.Stream()
            s_.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s_):
                fn()
            torch.cuda.current_stream().wait_stream(s_)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            graphs.append(g)
        ms, ms2 = _time(graphs[0].replay, reps), _time(graphs[1].replay, reps)
        b = n * (8 + 4 + 8 * log.count / n)
        out[f"2^{lg}"] = {"round_log_gbs": round(b / ms / 1e6, 1), "round_log_frac": round(b / ms / 1e6 / peak, 4),
                          "replay_gbs": round(b / ms2 / 1e6, 1), "replay_frac": round(b / ms2 / 1e6 / peak, 4),
                          "round_log_ms": round(ms, 4), "replay_ms": round(ms2, 4),
                          "round_log_ms_eager": round(ms_e, 4), "replay_ms_eager": round(ms2_e, 4),
                          "logged_fraction": round(log.count / n, 5), "l2_resident": n * 8 < 126e6}
        del x, y, words, ya, lw, log, graphs
        torch.cuda.empty_cache()
    return out


def vtrl_codec(lg: int = 26) -> dict:
    """the reference's own log format end to end on the device --
    the fused round-and-log writing the packed `.vtrl` payload (5 base-3 codes
    per byte, roundlog.py:43-53) instead of sparse words, and the replay
    decoding it (roundlog.py:73-82 + fpround.rev_array).  Algorithmic bytes per
    element: 8 (x) + 4 (FP32 y) + 0.2 (payload).  Graph-timed."""
    import torch

    from paper_2403_09603_b200 import _device as D
    from paper_2403_09603_b200 import _lib, workloads
    peak, _ = peaks()
    n = 1 << lg
    x, xa = workloads.config1_pair_torch(n, seed=1)
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    ya = torch.empty_like(y)
    packed = torch.empty(n // 5 + 1, dtype=torch.uint8, device="cuda")
    edge = torch.empty(16, dtype=torch.uint8, device="cuda")
    f, fa = D.Flags(), D.Flags()
    ws = D.workspace(int(_lib.lib().vt_round_log_workspace(n)), "vtrl_bench")

    def rl():
        _lib.call("vt_round_log", D.ptr(x), n, 32, workloads.TAU_CONFIG0, _lib.OUT_F32, D.ptr(y), None, 0, 0,
                  None, None, None, D.ptr(packed), 0, D.ptr(edge), f.cnt_ptr, f.err_ptr, D.ptr(ws), ws.numel(),
                  D.stream_ptr())

    rl()
    torch.cuda.synchronize()
    nfull, rem = divmod(n, 5)
    if rem:  # the writer's pending codes (LogWriter.close pads with 1s)
        tail = edge[:rem].tolist() + [1] * (5 - rem)
        packed[nfull] = sum(c * 3 ** k for k, c in enumerate(tail))
    nbytes = nfull + (1 if rem else 0)

    def rp():
        _lib.call("vt_replay", D.ptr(xa), n, 32, _lib.LOG_PACKED, D.ptr(packed), nbytes, 0, _lib.OUT_F32,
                  D.ptr(ya), fa.cnt_ptr, fa.err_ptr, None, 0, D.stream_ptr())

    rp()
    torch.cuda.synchronize()
    ok = bool(torch.equal(y.view(torch.int32), ya.view(torch.int32))) and f.read()[0] == 0 and fa.read()[0] == 0
    graphs = []
    for fn in (rl, rp):
        s_ = torch.cuda.Stream()
        s_.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_):
            fn()
        torch.cuda.current_stream().wait_stream(s_)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        graphs.append(g)
    ms, ms2 = _time(graphs[0].replay, 10), _time(graphs[1].replay, 10)
    b = n * (8 + 4 + 0.2)
    return {"n": n, "round_log_packed_gbs": round(b / ms / 1e6, 1), "round_log_packed_frac": round(b / ms / 1e6 / peak, 4),
            "replay_packed_gbs": round(b / ms2 / 1e6, 1), "replay_packed_frac": round(b / ms2 / 1e6 / peak, 4),
            "auditor_equals_trainer_bitwise": ok,
            "kernels": "round_log_kernel<PACKED> (codes packed 5 per byte in the same pass), replay_kernel<PACKED>"}


def config2() -> dict:
    """configs[2]: 161 ResNet-50-shaped FP64 tensors (N(0, sigma_t), sigma_t
    log-uniform in [1e-3, 10]); per tensor the budget search (B = 0.5% of n)
    then round-and-log at that tau."""
    import numpy as np
    import torch

    from paper_2403_09603_b200 import ops, protocol, workloads
    xs = workloads.config2_tensors_torch()
    total = sum(x.numel() for x in xs)
    ys = torch.empty(total, dtype=torch.float32, device="cuda")
    budgets = workloads.config2_budgets([x.numel() for x in xs])
    words = torch.empty(sum(budgets) + len(xs), dtype=torch.int64, device="cuda")
    state = {}

    def run_batch():
        # the whole sweep in one batched call: one fused rounding pass over all
        # 161 tensors + batched selection / filter kernels (fixed launch count)
        state["batch"] = ops.round_and_log_adaptive_batch(
            xs, 32, budgets, outs=[ys[o:o + x.numel()] for o, x in zip(offs, xs)],
            log_outs=[words[w:w + B + 1] for w, B in zip(woffs, budgets)], check=False)

    offs = np.concatenate([[0], np.cumsum([x.numel() for x in xs])[:-1]]).tolist()
    woffs = np.concatenate([[0], np.cumsum([B + 1 for B in budgets])[:-1]]).tolist()
    n_streams = 8  # per-tensor calls: kernels of different tensors overlap (own workspace per stream)
    side = [torch.cuda.Stream() for _ in range(n_streams)]

    def run():
        off = woff = 0
        pend = []
        main = torch.cuda.current_stream()
        for s_ in side:
            s_.wait_stream(main)
        for i, (x, B) in enumerate(zip(xs, budgets)):
            n = x.numel()
            with torch.cuda.stream(side[i % n_streams]):
                pend.append(ops.round_and_log_adaptive(x, 32, B, out=ys[off:off + n],
                                                       log_out=words[woff:woff + B + 1], check=False,
                                                       tag=f"adaptive{i % n_streams}"))
            off += n
            woff += B + 1
        for s_ in side:
            main.wait_stream(s_)
        state["pend"] = pend

    def graphed(fn):
        fn()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph):
            fn()
        return graph

    g_calls = graphed(run)
    ms_calls = _time(g_calls.replay, reps=5, warm=1)
    ms_calls_eager = _time(run, reps=2, warm=0)
    counts_calls = [p.flags.read()[1][0] for p in state["pend"]]
    taus_calls = [float(p.tau.item()) for p in state["pend"]]
    g_batch = graphed(run_batch)
    ms = _time(g_batch.replay, reps=5, warm=1)
    ms_eager = _time(run_batch, reps=2, warm=0)
    res = state["batch"].finish()
    counts = [r[1].count for r in res]
    taus = [r[2] for r in res]
    assert all(c <= B for c, B in zip(counts, budgets))
    # the batch equals the per-tensor calls, and the device tau the host search
    assert counts == counts_calls and taus == taus_calls
    k = int(np.argmin([x.numel() for x in xs]))
    assert taus[k] == protocol.search_tau_budget(xs[k], 32, budgets[k])
    t = np.array(taus) / 2.0 ** -24
    logged = sum(counts)
    return {"tensors": len(xs), "elements": total, "ms_per_sweep": round(ms, 3), "ms_per_sweep_eager": round(ms_eager, 3),
            "g_elements_per_s": round(total / ms / 1e6, 2),
            "round_log_gbs_equiv": round(total * (8 + 4 + 8 * logged / total) / ms / 1e6, 1),
            "ms_per_tensor_calls_8_streams": round(ms_calls, 3), "ms_per_tensor_calls_eager": round(ms_calls_eager, 3),
            "logged_fraction": round(logged / total, 6), "tau_over_2^-24": [round(float(t.min()), 6), round(float(t.max()), 6)],
            "note": "ops.round_and_log_adaptive_batch: one fused rounding pass over all 161 tensors (candidates "
                    "above a per-tensor threshold below tau) + batched exact selection, device bisection and "
                    "ordered filter; CUDA graph. Per-tensor calls (8 streams, one graph) kept for comparison"}


def config3_gpt2(steps: int = 3) -> dict:
    """configs[3]: one GPT-2-small FP64 training step (batch 8 x 1024 tokens,
    random init, SGD) with every leaf-module output and input gradient passed
    through the adaptive round-and-log (hooks.RoundAndLogHooks), against the
    same step without the hooks."""
    import torch

    from paper_2403_09603_b200 import hooks, workloads
    model = workloads.gpt2_small_fp64()
    opt = torch.optim.SGD(model.parameters(), lr=1e-4)
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    idx = torch.randint(0, 50257, (8, 1024), device="cuda", generator=g)
    tgt = torch.randint(0, 50257, (8, 1024), device="cuda", generator=g)

    def step():
        opt.zero_grad(set_to_none=True)
        logits = model(idx)
        loss = torch.nn.functional.cross_entropy(logits.view(-1, logits.shape[-1]), tgt.view(-1))
        loss.backward()
        opt.step()
        return loss

    ms_plain = _time(step, reps=steps, warm=1)
    hk = hooks.RoundAndLogHooks(model)
    step()
    info = hk.collect()

    def step_hooked():  # the trainer reads the step's taus and log sizes (one copy) every step
        step()
        hk.collect()

    ms_hooked = _time(step_hooked, reps=steps, warm=1)
    step()
    logs = hk.collect(keep_logs=True)["logs"]
    hk.remove()
    # the auditor's step: the same hook points replay a trainer step's logs in place
    ha = hooks.ReplayHooks(model, logs)

    def step_audited():
        step()
        ha.collect()

    ms_audited = _time(step_audited, reps=steps, warm=1)
    ha.remove()
    return {"model": "GPT-2 small FP64 (12x768, 12 heads, vocab 50257), random init", "batch": [8, 1024],
            "step_ms_plain": round(ms_plain, 2), "step_ms_round_and_log": round(ms_hooked, 2),
            "trainer_overhead": round(ms_hooked / ms_plain, 4), "step_ms_replay": round(ms_audited, 2),
            "auditor_overhead": round(ms_audited / ms_plain, 4), "hooked_tensors": info["tensors"],
            "hooked_fwd": info["fwd"], "hooked_bwd": info["bwd"], "hooked_elements": info["elements"],
            "logged_entries": info["logged"], "budget": "0.5% per tensor",
            "paper_trainer_overhead": "1.2-1.4x (PAPER.md:402, A40 / Titan XP / 2080 Ti)"}


def config4_merkle() -> dict:
    """configs[4]: SHA-256 Merkle tree over 1.5e9 FP32 params (4 KiB leaves)."""
    import torch

    from paper_2403_09603_b200 import _device as D
    from paper_2403_09603_b200 import _lib, merkle, workloads
    n = workloads.CONFIG4_PARAMS
    w = workloads.config4_weights_torch(n)
    ms = _time(lambda: merkle.merkle_chunked(w), reps=3, warm=1)
    t = merkle.merkle_chunked(w)
    sizes = [int(l.shape[0]) for l in t.levels_device]
    leaves = sizes[0]
    nodes = sum(m // 2 for m in sizes[:-1])  # hashed internal nodes (promoted copies excluded)
    comps = leaves * (4096 // 64 + 1) + nodes * 2
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    blocks, reps = 148 * 32, 64
    pk_ms = _time(lambda: _lib.call("vt_sha256_peak_bench", D.ptr(sink), blocks, reps, D.stream_ptr()), reps=3)
    peak_cps = blocks * 128 * reps / (pk_ms * 1e-3)
    cps = comps / (ms * 1e-3)
    return {"params": n, "leaves": int(leaves), "hashed_internal_nodes": int(nodes), "levels": len(sizes),
            "ms": round(ms, 3), "hashed_gbs": round(n * 4 / ms / 1e6, 1),
            "compressions_per_s": round(cps / 1e9, 3), "unit_cps": "G compressions/s",
            "int_ops_per_s": round(cps * 1400 / 1e12, 2), "unit_ops": "T int ops/s (analytic 1400 / compression)",
            "sha256_compute_ceiling_cps": round(peak_cps / 1e9, 3),
            "frac_of_sha256_int_peak": round(cps / peak_cps, 4),
            "peak_note": "ceiling = the same compress() on register-resident messages (vt_sha256_peak_bench)",
            "root": t.root_hex[:16]}


# ---------------------------------------------------------------------------
# CPU: the reference algorithm (oracle port) on the host cores
# ---------------------------------------------------------------------------

def _cpu_chunk(args):
    lo, hi, seed = args
    sys.path.insert(0, str(REPO / "oracle"))
    import numpy as np

    import vt_oracle as O
    from paper_2403_09603_b200 import workloads
    n = hi - lo
    xt, xa = workloads.config1_pair(n, seed)
    tau = workloads.TAU_CONFIG0
    t0 = time.perf_counter()
    # trainer channel (protocol.py:198-202): direction + rnd + pack
    codes = O.direction_array(xt, 32, tau)
    O.rnd_array(xt, 32)
    O.pack_groups(np.concatenate([codes, np.ones((-codes.size) % 5, np.uint8)]))
    # auditor channel (protocol.py:212-216): rev + rnd for the correction count
    ya = O.rev_array(xa, 32, codes)
    int(np.count_nonzero(ya != O.rnd_array(xa, 32)))
    dt = time.perf_counter() - t0
    return n, int(np.count_nonzero(codes != 1)), dt


def cpu_measure(total: int, chunk: int, procs: int):
    import multiprocessing as mp
    jobs = [(i * chunk, min(total, (i + 1) * chunk), 100 + i) for i in range((total + chunk - 1) // chunk)]
    t0 = time.perf_counter()
    if procs > 1:
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_cpu_chunk, jobs)
    else:
        res = [_cpu_chunk(j) for j in jobs]
    wall = time.perf_counter() - t0
    n = sum(r[0] for r in res)
    logged = sum(r[1] for r in res)
    compute = sum(r[2] for r in res)
    f = logged / n
    # input generation is excluded: the timed region is the reference calls,
    # spread perfectly over the processes (compute / procs)
    eff = compute / max(1, min(procs, len(jobs)))
    gbs = n * (8 + 4 + 8 * f) * 2 / eff / 1e9
    return {"gbs": gbs, "n": n, "wall_s": wall, "compute_s": compute, "eff_s": eff, "f": f}


def _cpu_leaf_chunk(args):
    lo, hi, leaf = args
    import hashlib

    import numpy as np
    w = np.random.default_rng(lo).normal(0.0, 0.02, size=(hi - lo) * leaf // 4).astype("<f4").tobytes()
    t0 = time.perf_counter()
    out = [hashlib.sha256(w[i:i + leaf]).digest() for i in range(0, len(w), leaf)]
    return out, time.perf_counter() - t0


def cpu_merkle(n_leaves: int, procs: int, leaf: int = 4096) -> dict:
    """Reference Merkle path on the host: hashlib (OpenSSL) SHA-256 of each
    4 KiB leaf over all cores, then merkle.build's levels (one process)."""
    import multiprocessing as mp
    sys.path.insert(0, str(REPO / "oracle"))
    import vt_oracle as O
    per = (n_leaves + procs - 1) // procs
    jobs = [(i * per, min(n_leaves, (i + 1) * per), leaf) for i in range(procs) if i * per < n_leaves]
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_cpu_leaf_chunk, jobs)
    leaves = [d for r in res for d in r[0]]
    hash_s = max(r[1] for r in res)
    t0 = time.perf_counter()
    O.merkle_levels(leaves)
    build_s = time.perf_counter() - t0
    return {"value": round(n_leaves * leaf / (hash_s + build_s) / 1e9, 3), "unit": "GB/s hashed",
            "cores": procs, "kind": "port", "sample": f"{n_leaves} leaves of {leaf} B (hashlib over {procs} "
                                                       f"processes, then the level build)"}


def cpu_adaptive(n: int) -> dict:
    """Reference budget search + trainer channel on one host core: the
    oracle's search_tau_budget (bisection on the exact order statistic) then
    direction_array + rnd_array at that tau, on one N(0,1) tensor."""
    import numpy as np
    sys.path.insert(0, str(REPO / "oracle"))
    import vt_oracle as O
    x = np.random.default_rng(2).normal(0.0, 1.0, n)
    t0 = time.perf_counter()
    tau = O.search_tau_budget(x, 32, int(0.005 * n))
    O.direction_array(x, 32, tau)
    O.rnd_array(x, 32)
    dt = time.perf_counter() - t0
    return {"value": round(n / dt / 1e9, 4), "unit": "G elements/s", "cores": 1, "kind": "port",
            "sample": f"one tensor of {n} elements"}


def cpu_baseline(args):
    cores = len(os.sched_getaffinity(0))
    total = 1 << args.cpu_log2n
    r = cpu_measure(total, 1 << 20, cores)
    r1 = cpu_measure(1 << 22, 1 << 20, 1)
    return {"value": round(r["gbs"], 4), "unit": "GB/s", "cores": cores, "kind": "port",
            "value_1core": round(r1["gbs"], 4),
            "sample": f"2^{args.cpu_log2n} elements of the configs[1] pair (trainer channel: direction_array + "
                      f"rnd_array + pack; auditor: rev_array + rnd_array count), chunks of 2^20 over "
                      f"{cores} processes, wall {r['wall_s']:.1f}s",
            "cpu_model": _cpu_model()}


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args) -> None:
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    total = 1 << args.cpu_log2n
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_measure(1 << 20, 1 << 20, 1)
    vals = []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_measure(total, 1 << 20, cores))
    wall = time.perf_counter() - t_all
    gbs = statistics.mean(v["gbs"] for v in vals)
    ms = wall / args.steps * 1e3
    line = {
        "impl": "reference",
        "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 1), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64->f32 (uint8 ternary codes)",
        "data": "synthetic (seeded, BASELINE configs[1] distribution)",
        "config": {"workload": f"configs[1]: round-and-log + replay pair, 2^{args.log2n} FP64 elements per GPU, "
                               f"b_r=32, tau=0x1.ff7ced916872bp-25",
                   "n_per_gpu": 1 << args.log2n, "parallelism": f"{cores} host processes",
                   "sample": f"each step times a bounded sample of 2^{args.cpu_log2n} elements of that pair"},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"2^{args.cpu_log2n} elements per step in 2^20 chunks",
                         "cpu_model": _cpu_model()},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--log2n", type=int, default=26)
    ap.add_argument("--cpu-log2n", type=int, default=25)
    ap.add_argument("--sweep", type=int, nargs="*", default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-extras", dest="extras", action="store_false",
                    help="skip configs[2], configs[4] and the 2^20..2^32 size sweep (run by default at N=1)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
