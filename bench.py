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


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_spawn(args) -> None:
    """``--gpus N`` without a launcher: re-execute this command under
    torch.distributed.run with N ranks on this node (rendezvous on 127.0.0.1,
    NCCL_DEBUG=INFO for the INIT lines that show the communicator's nranks)
    and exit with its status.  Under the driver's torchrun (WORLD_SIZE set)
    this does nothing."""
    if "WORLD_SIZE" in os.environ or args.gpus <= 1:
        return
    if args.dist_backend == "nccl" and not args.harness_check:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:  # NCCL puts one rank on one GPU; say so instead of a communicator error
            print(f"[bench] --gpus {args.gpus} needs {args.gpus} visible GPUs, this node has {have} "
                  f"(--dist-backend gloo runs the N-rank code path on one GPU)", file=sys.stderr)
            sys.exit(2)
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd, env=env))


def _graph(fn, stream):
    """Capture fn (already warmed on ``stream``) into a CUDA graph on that stream."""
    import torch
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        fn()
    return g


def _capture(fn):
    """Warm fn up on a side stream, then capture it on THAT stream: the
    operators' workspaces are per stream, so the graph reuses the warmed one
    (a workspace first allocated inside a capture would put its zero-fill in
    the graph)."""
    import torch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    return _graph(fn, s)


def run_harness_check(args) -> None:
    """CPU self-test of the launcher path (no GPU, no kernels; tests only):
    gloo ranks, the barrier + max-over-ranks timing and rank 0's single JSON
    line with n_gpus = world size.  Its value is not a measurement."""
    import torch
    import torch.distributed as dist
    world, rank, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    t0 = time.perf_counter()
    for _ in range(args.warmup + args.steps):
        torch.ones(1024).sum()
    ms = (time.perf_counter() - t0) * 1e3 / max(1, args.steps)
    t = torch.tensor([ms], dtype=torch.float64)
    ranks = torch.tensor([1], dtype=torch.int64)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(ranks)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "GB/s", "n_gpus": world,
                          "ranks_reporting": int(ranks.item()), "steps": args.steps, "warmup": args.warmup,
                          "ms_per_step": round(float(t.item()), 4), "harness_check": True}), flush=True)


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2403_09603_b200 import ops, workloads
    from paper_2403_09603_b200 import dist as vdist

    world, rank, local = dist_env()
    # --dist-backend gloo (tests only): every rank on GPU 0 with host-side
    # collectives, to exercise the multi-rank code paths on a one-GPU box --
    # its numbers are not measurements (ranks share one GPU)
    gloo = args.dist_backend == "gloo"
    if gloo:
        local = local % torch.cuda.device_count()
        args.no_graph = True  # host-side collectives cannot be captured
    torch.cuda.set_device(local)
    # under a launcher (WORLD_SIZE set, even 1) the NCCL path runs: process
    # group, count all-gather captured in the step's graph, max over ranks
    ddp = "WORLD_SIZE" in os.environ
    if ddp:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    n = 1 << args.log2n
    tau = workloads.TAU_CONFIG0
    base = rank * n
    xt, xa = workloads.config1_pair_torch(n, seed=1 + rank, device=dev)
    y_t = torch.empty(n, dtype=torch.float32, device=dev)
    y_a = torch.empty(n, dtype=torch.float32, device=dev)
    words = torch.empty(n // 4, dtype=torch.int64, device=dev)
    counts = torch.empty(max(world, 1), dtype=torch.int64, device=dev)
    stream = torch.cuda.Stream(dev)  # every operator runs (and is captured) on this stream
    stream.wait_stream(torch.cuda.current_stream(dev))

    # the exchange step at N ranks: the per-rank log counts, fused into the
    # round-and-log kernel over peer memory (symmetric memory over NVLink:
    # the kernel's last CTA stores its count into every rank's buffer, a wait
    # kernel collects them) -- or an NCCL all-gather if that cannot be set up
    xchg, xchg_kind = None, None
    if gloo:
        xchg_kind = "gloo all-gather (multi-rank code-path check on one GPU)"
    elif ddp:
        try:
            xchg = vdist.CountExchange(device=dev)
            xchg_kind = "peer-memory stores fused into rl_fused_kernel + counts_wait_kernel (symmetric memory)"
        except Exception as e:  # noqa: BLE001
            print(f"[bench] symmetric-memory exchange unavailable, using NCCL all-gather: {e!r}", file=sys.stderr)
            xchg_kind = "NCCL all-gather of the counts"
    with torch.cuda.stream(stream):
        # the auditor receives the log with its length (as a file carries it);
        # take it from one untimed trainer pass
        p0 = ops.round_and_log(xt, 32, tau, out=y_t, log_out=words, global_base=base, check=False)
        _, log0 = p0.finish()
    count = log0.count
    log_words = words[:count]
    state = {}
    if xchg is not None:  # once, untimed: the fused exchange equals the NCCL all-gather
        with torch.cuda.stream(stream):
            pe = xchg.round_and_log(xt, 32, tau, base, out=y_t, log_out=words)
            got = xchg.wait().clone()
            pe.finish()
        xchg.check()
        want = vdist.all_gather_counts(count, device=dev)
        if not torch.equal(got, want):
            raise RuntimeError(f"peer-memory count exchange {got.tolist()} != NCCL all-gather {want.tolist()}")

    def trainer():
        if xchg is not None:
            state["p"] = xchg.round_and_log(xt, 32, tau, base, out=y_t, log_out=words)
        else:
            state["p"] = ops.round_and_log(xt, 32, tau, out=y_t, log_out=words, global_base=base, check=False)

    def exchange():
        if xchg is not None:
            xchg.wait()
        elif ddp:  # the exchange step: all-gather of per-rank log counts (device-resident)
            vdist._all_gather_flat(counts, state["p"].flags.buf[2:3])

    def auditor():
        state["fa"] = ops.replay(xa, 32, log_words, out=y_a, global_base=base, check=False)[1]

    def step():
        trainer()
        exchange()
        auditor()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize()
    # verify once (outside the timed region): auditor output == trainer output, no errors
    if xchg is not None:
        xchg.check()
    err_t, cnt_t = state["p"].flags.read()
    err_a, cnt_a = state["fa"].read()
    assert err_t == 0 and err_a == 0 and cnt_t[0] == count, (err_t, err_a, cnt_t, count)
    ok_equal = bool(torch.equal(y_t.view(torch.int32), y_a.view(torch.int32)))

    # The step (both operators and, at N > 1, the NCCL count all-gather between
    # them) is captured once into CUDA graphs on `stream`; the timed loop
    # replays them, so host launch latency does not leak into the timeline.
    graphs = None
    if not args.no_graph:
        try:
            g_t = _graph(lambda: (trainer(), exchange()), stream)
            pg = state["p"]
            g_a = _graph(auditor, stream)
            flg = state["fa"]
            with torch.cuda.stream(stream):
                g_t.replay()
                g_a.replay()
            torch.cuda.synchronize()
            assert pg.flags.read()[1][0] == count and flg.read()[0] == 0
            graphs = (g_t, g_a)
        except Exception as e:  # e.g. a communicator that cannot be captured: eager steps
            print(f"[bench] graph capture failed, timing eager steps: {e!r}", file=sys.stderr)
            torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    mids = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if ddp:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk, torch.cuda.stream(stream):
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for i in range(args.steps):
            starts[i].record(stream)
            if graphs:
                graphs[0].replay()
                mids[i].record(stream)
                graphs[1].replay()
            else:
                trainer()
                exchange()
                mids[i].record(stream)
                auditor()
            ends[i].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
    if ddp:
        dist.barrier()
    if xchg is not None:
        xchg.check()
    ms_total = t0.elapsed_time(t1)
    rl_ms = statistics.mean(starts[i].elapsed_time(mids[i]) for i in range(args.steps))
    rp_ms = statistics.mean(mids[i].elapsed_time(ends[i]) for i in range(args.steps))
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if ddp:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    f = count / n
    per_elem = (8 + 4 + 8 * f) * 2
    value = world * n * per_elem / (ms_step * 1e-3) / 1e9
    rl_bytes = n * (8 + 4 + 8 * f)
    rp_bytes = n * (8 + 4 + 8 * f)
    peak, peak_src = peaks()
    del xt, xa
    torch.cuda.empty_cache()

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, n, tau, base, dev, world)

    strong = None
    if args.extras or ddp:
        strong = strong_scaling(args, world, rank, dev)

    extras = None
    if args.extras and world == 1:
        extras = {"configs[4]_size_sweep": sweep([20, 24, 26, 28, 30, 32]),
                  "vtrl_codec_2^26": vtrl_codec(26),
                  "configs[2]_resnet50_budget": config2(),
                  "configs[3]_gpt2_fp64_step": config3_gpt2(),
                  "configs[4]_merkle_1.5B": config4_merkle(),
                  "budget_search_standalone": budget_search(),
                  "f2_reference_loop_trend": f2_trend()}

    cpu = cpu_extra = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args)
        if args.extras:
            cpu_extra = cpu_legs()
    if ddp:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
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
                   "launch": ("cuda graphs (trainer + count exchange, auditor)" if ddp else
                              "cuda graphs (one per operator)") if graphs else "eager",
                   "exchange": xchg_kind},
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
    if strong is not None:
        line["strong_scaling"] = strong
    if args.sweep:
        line["sweep"] = sweep(args.sweep)
    if extras is not None:
        if cpu_extra is not None:
            extras["cpu_legs"] = cpu_extra
        line["extras"] = extras
    print(json.dumps(line), flush=True)


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
        graphs = [_capture(fn) for fn in (rl, rp)]
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

    ws_rp = D.workspace(int(_lib.lib().vt_replay_workspace(n)), "vtrl_bench_rp")

    def rp():
        _lib.call("vt_replay", D.ptr(xa), n, 32, _lib.LOG_PACKED, D.ptr(packed), nbytes, 0, _lib.OUT_F32,
                  D.ptr(ya), fa.cnt_ptr, fa.err_ptr, D.ptr(ws_rp), ws_rp.numel(), D.stream_ptr())

    rp()
    torch.cuda.synchronize()
    ok = bool(torch.equal(y.view(torch.int32), ya.view(torch.int32))) and f.read()[0] == 0 and fa.read()[0] == 0
    graphs = [_capture(fn) for fn in (rl, rp)]
    ms, ms2 = _time(graphs[0].replay, 10), _time(graphs[1].replay, 10)
    b = n * (8 + 4 + 0.2)
    return {"n": n, "round_log_packed_gbs": round(b / ms / 1e6, 1), "round_log_packed_frac": round(b / ms / 1e6 / peak, 4),
            "replay_packed_gbs": round(b / ms2 / 1e6, 1), "replay_packed_frac": round(b / ms2 / 1e6 / peak, 4),
            "auditor_equals_trainer_bitwise": ok,
            "kernels": "round_log_kernel<PACKED> (codes packed 5 per byte in the same pass), rp_fused_kernel<PACKED> "
                       "(persistent TMA pipeline, payload decoded a tile ahead into the code map)"}


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
        return _capture(fn)

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


def config3_gpt2(steps: int = 6) -> dict:
    """configs[3]: one GPT-2-small FP64 training step (batch 8 x 1024 tokens,
    random init, SGD) with every leaf-module output and input gradient, and
    the loss gradient, passed through the adaptive round-and-log
    (hooks.RoundAndLogHooks, protocol.py:264-285) and the updated parameters
    rounded onto the grid (hooks.round_parameters, protocol.py:286-293),
    against the same step without any of it."""
    import torch

    from paper_2403_09603_b200 import hooks, workloads
    model = workloads.gpt2_small_fp64()
    opt = torch.optim.SGD(model.parameters(), lr=1e-4)
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    idx = torch.randint(0, 50257, (8, 1024), device="cuda", generator=g)
    tgt = torch.randint(0, 50257, (8, 1024), device="cuda", generator=g)

    cur = {"hk": None}

    def step():
        opt.zero_grad(set_to_none=True)
        logits = model(idx)
        if cur["hk"] is not None:
            cur["hk"].loss_grad(logits)
        loss = torch.nn.functional.cross_entropy(logits.view(-1, logits.shape[-1]), tgt.view(-1))
        loss.backward()
        opt.step()
        if cur["hk"] is not None:
            hooks.round_parameters(model)
        return loss

    ms_plain = _time(step, reps=steps, warm=1)
    hk = cur["hk"] = hooks.RoundAndLogHooks(model)
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
    ha = cur["hk"] = hooks.ReplayHooks(model, logs)

    def step_audited():
        step()
        ha.collect()

    ms_audited = _time(step_audited, reps=steps, warm=1)
    ha.remove()
    return {"model": "GPT-2 small FP64 (12x768, 12 heads, vocab 50257), random init", "batch": [8, 1024],
            "step_ms_plain": round(ms_plain, 2), "step_ms_round_and_log": round(ms_hooked, 2),
            "trainer_overhead": round(ms_hooked / ms_plain, 4), "step_ms_replay": round(ms_audited, 2),
            "auditor_overhead": round(ms_audited / ms_plain, 4), "hooked_tensors": info["tensors"],
            "hooked_fwd": info["fwd"], "hooked_bwd": info["bwd"], "hooked_loss_grad": info["loss"],
            "parameters_rounded": True, "hooked_elements": info["elements"],
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
    # independent denominator: the SHF/LOP3/add mix on register-only chains,
    # adds on the ALU pipe (IADD3) or on the FMA pipe (IMAD); the faster is the peak
    mix_blocks, mix_reps = 148 * 8, 2048
    per = mix_blocks * 256 * mix_reps * int(_lib.lib().vt_int_mix_ops_per_thread_rep())
    mix = {}
    for fma in (0, 1):
        mix_ms = _time(lambda: _lib.call("vt_int_mix_peak_bench", D.ptr(sink), mix_blocks, mix_reps, fma,
                                         D.stream_ptr()), reps=3)
        mix["fma_adds" if fma else "iadd3_adds"] = per / (mix_ms * 1e-3)
    mix_ops = max(mix.values())
    cps = comps / (ms * 1e-3)
    return {"params": n, "leaves": int(leaves), "hashed_internal_nodes": int(nodes), "levels": len(sizes),
            "ms": round(ms, 3), "hashed_gbs": round(n * 4 / ms / 1e6, 1),
            "compressions_per_s": round(cps / 1e9, 3), "unit_cps": "G compressions/s",
            "int_ops_per_s": round(cps * 1400 / 1e12, 2), "unit_ops": "T int ops/s (analytic 1400 / compression)",
            "int_mix_peak_ops_per_s": round(mix_ops / 1e12, 2),
            "int_mix_variants_ops_per_s": {k: round(v / 1e12, 2) for k, v in mix.items()},
            "frac_of_sha256_int_peak": round(cps * 1400 / mix_ops, 4),
            "peak_note": "denominator = int_mix_peak_kernel: register-only chains of the SHA-256 op mix (6 SHF : "
                         "4 LOP3 : 4 three-input adds), not compress(); the faster of adds-as-IADD3 (ALU pipe) and "
                         "adds-as-2xIMAD (FMA pipe); numerator = compressions/s x 1400 analytic ops",
            "sha256_compress_ceiling_cps": round(peak_cps / 1e9, 3),
            "frac_of_compress_ceiling": round(cps / peak_cps, 4),
            "root": t.root_hex[:16]}


def budget_search() -> dict:
    """The standalone budget search (protocol.search_tau_budget ->
    vt_tau_budget: one read of x + the cooperative selection / bisection) at
    2^26 and 2^30 N(0,1) elements, 0.5% budget; algorithmic bytes = 8 per
    element (one read of x).  The sharded form (dist.search_tau_budget_sharded
    on one process: candidate pass, exchange buffer, digit keys, host
    selection -- host wall time incl. its syncs) and one pass of its exact
    5-pass fallback are timed beside it."""
    import torch

    from paper_2403_09603_b200 import _device as D
    from paper_2403_09603_b200 import _lib, protocol
    from paper_2403_09603_b200 import dist as vdist
    peak, _ = peaks()
    out = {}
    for lg in (26, 30):
        n = 1 << lg
        g = torch.Generator(device="cuda")
        g.manual_seed(lg)
        x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
        B = int(0.005 * n)
        ws = D.workspace(int(_lib.lib().vt_tau_budget_workspace(n)), "bench_tau")
        res = torch.empty(2, dtype=torch.float64, device="cuda")
        fl = D.Flags()

        def run():
            _lib.call("vt_tau_budget", D.ptr(x), n, 32, B, 30, D.ptr(res), res.data_ptr() + 8, fl.err_ptr, D.ptr(ws),
                      ws.numel(), D.stream_ptr())

        ms = _time(run, reps=10)
        tau = float(res[0].item())
        assert tau == protocol.search_tau_budget(x, 32, B)
        ms5 = _time(lambda: vdist.ShardedKth(x, 32).local_hist(0), reps=5)  # one of the 5 exact passes
        # the sharded form on one process: candidates + exchange buffer + digit keys + host selection
        t_sh = []
        for _ in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tau_sh = vdist.search_tau_budget_sharded(x, 32, B)
            t_sh.append(time.perf_counter() - t0)
        assert tau_sh == tau
        # the same with both exchanges over peer memory and the decision on the device
        ex = vdist.BudgetExchange()
        t_x = []
        for _ in range(4):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            tau_x = vdist.search_tau_budget_sharded(x, 32, B, exchange=ex, n_global=n)
            t_x.append(time.perf_counter() - t0)
        assert tau_x == tau
        out[f"2^{lg}"] = {"ms": round(ms, 4), "gbs": round(8 * n / ms / 1e6, 1), "frac": round(8 * n / ms / 1e6 / peak, 4),
                          "tau_over_2^-24": round(tau / 2.0 ** -24, 6),
                          "sharded_candidate_path_ms_wall": round(1e3 * min(t_sh[1:]), 3),
                          "sharded_peer_exchange_path_ms_wall": round(1e3 * min(t_x[1:]), 3),
                          "sharded_exact_select_pass_ms": round(ms5, 4),
                          "sharded_exact_select_5_passes_ms_est": round(5 * ms5, 4)}
        del x, ws
        torch.cuda.empty_cache()
    out["kernels"] = "adapt_keys32_kernel (candidate values, one read of x) + adapt_tail_kernel (cooperative selection, " \
                     "device FP64 bisection)"
    return out


def f2_trend() -> dict:
    """the reference's own loop (vtrain.protocol._run, unmodified,
    from baseline/_ref) on the shipped ``trend`` config, trainer then auditor,
    with the reference's NumPy channels and with the GPU channels in the seam;
    wall time of each run and of the channel calls inside it (a timing proxy
    around process()), after an untimed warm-up of both arms on the `tiny`
    config.  Roots / .vtrl / corrections must agree."""
    ref = REPO / "baseline" / "_ref"
    if not (ref / "vtrain" / "protocol.py").exists():
        return {"skipped": "reference not installed (tools/install_reference.sh)"}
    import hashlib
    import tempfile
    sys.path.insert(0, str(ref))
    from vtrain import cli
    from vtrain import protocol as pr
    from vtrain import roundlog as rrl

    from paper_2403_09603_b200 import protocol as gp
    from paper_2403_09603_b200 import roundlog

    class Timed:
        def __init__(self, inner):
            self.inner, self.s, self.calls = inner, 0.0, 0

        def process(self, values, tau):
            t0 = time.perf_counter()
            r = self.inner.process(values, tau)
            self.s += time.perf_counter() - t0
            self.calls += 1
            return r

    cfg = cli.load_config(ref / "vtrain_configs" / "trend.json")
    out = {}
    with tempfile.TemporaryDirectory() as td:
        # warm-up, untimed: the shipped `tiny` config through both arms (first
        # kernel launches, staging buffers, NumPy paths), as every timed leg here
        warm = cli.load_config(ref / "vtrain_configs" / "tiny.json")
        for W, R, T, A in ((rrl.LogWriter, rrl.LogReader, pr._TrainerChannel, pr._AuditorChannel),
                           (roundlog.LogWriter, roundlog.LogReader, gp.GpuTrainerChannel, gp.GpuAuditorChannel)):
            wl = Path(td) / "warm.vtrl"
            w = W(wl, warm.b_r)
            pr._run(warm, pr.get_profile(warm.trainer_profile), T(w, warm.b_r), False)
            w.close()
            pr._run(warm, pr.get_profile("pairwise"), A(R(wl), warm.b_r), False)
        for side, W, R, T, A in (("reference_numpy", rrl.LogWriter, rrl.LogReader, pr._TrainerChannel,
                                  pr._AuditorChannel),
                                 ("gpu", roundlog.LogWriter, roundlog.LogReader, gp.GpuTrainerChannel,
                                  gp.GpuAuditorChannel)):
            log = Path(td) / f"{side}.vtrl"
            w = W(log, cfg.b_r)
            tc = Timed(T(w, cfg.b_r))
            t0 = time.perf_counter()
            tree_t, *_ = pr._run(cfg, pr.get_profile(cfg.trainer_profile), tc, False)
            w.close()
            t1 = time.perf_counter()
            ac = Timed(A(R(log), cfg.b_r))
            tree_a, _, _, per_step, _, _ = pr._run(cfg, pr.get_profile("pairwise"), ac, False)
            t2 = time.perf_counter()
            out[side] = {"train_s": round(t1 - t0, 3), "audit_s": round(t2 - t1, 3),
                         "train_channel_s": round(tc.s, 3), "audit_channel_s": round(ac.s, 3), "calls": tc.calls,
                         "root": tree_t.root.hex()[:16], "audit_root": tree_a.root.hex()[:16],
                         "vtrl_sha": hashlib.sha256(log.read_bytes()).hexdigest()[:16],
                         "corrections": int(sum(s.forward_corrections + s.backward_corrections for s in per_step))}
    r, g = out["reference_numpy"], out["gpu"]
    out["same_results"] = all(r[k] == g[k] for k in ("root", "audit_root", "vtrl_sha", "corrections"))
    out["speedup_train_audit"] = round((r["train_s"] + r["audit_s"]) / (g["train_s"] + g["audit_s"]), 3)
    out["speedup_channels"] = round((r["train_channel_s"] + r["audit_channel_s"]) /
                                    (g["train_channel_s"] + g["audit_channel_s"]), 3)
    return out


def strong_scaling(args, world: int, rank: int, dev) -> dict:
    """Strong-scaling legs (fixed total work over the N ranks),
    device-timed with a barrier on both sides, max over ranks:
      * the 2^32 size-sweep point: round-and-log + count all-gather + replay
        over contiguous shards (dist.shard_range; global indices);
      * configs[4]: the 1.5e9-parameter Merkle tree, whole 2^12-leaf blocks
        per rank + block-root exchange (peer memory at N > 1 on NCCL) + top
        levels (dist.merkle_sharded); its root is checked equal to the
        single-GPU root;
      * the budget search of one 2^30-element N(0,1) tensor sharded over the
        ranks (dist.search_tau_budget_sharded with a BudgetExchange);
      * configs[2]: the 161 ResNet-50 tensors LPT-assigned to ranks, each rank
        one batched adaptive call; taus checked against the single-GPU batch."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2403_09603_b200 import merkle, ops, workloads
    from paper_2403_09603_b200 import dist as vdist

    def tmax(ms: float) -> float:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        if dist.is_initialized():
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, reps: int) -> float:
        fn()
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        if dist.is_initialized():
            dist.barrier()
        return tmax(s.elapsed_time(e) / reps)

    out = {"n_gpus": world, "scaling": "strong"}
    peak, _ = peaks()
    # --- 2^32 round-and-log + replay, sharded
    total = 1 << 32
    lo, hi = vdist.shard_range(total, rank, world)
    n = hi - lo
    x = workloads.config0_x_torch_bernoulli(n, seed=32 + rank, device=dev)
    y = torch.empty(n, dtype=torch.float32, device=dev)
    ya = torch.empty(n, dtype=torch.float32, device=dev)
    words = torch.empty(n // 8 + 4096, dtype=torch.int64, device=dev)
    counts = torch.empty(world, dtype=torch.int64, device=dev)
    tau = workloads.TAU_CONFIG0
    st = {}

    def rl():
        st["p"] = ops.round_and_log(x, 32, tau, out=y, log_out=words, global_base=lo, check=False)
        if dist.is_initialized():
            vdist._all_gather_flat(counts, st["p"].flags.buf[2:3])

    rl()
    _, log = st["p"].finish()
    lw = words[:log.count]

    def rp():
        ops.replay(x, 32, lw, out=ya, global_base=lo, check=False)

    ms_rl, ms_rp = timed(rl, 4), timed(rp, 4)
    logged = torch.tensor([log.count], dtype=torch.int64, device=dev)
    if dist.is_initialized():
        dist.all_reduce(logged)
    f = int(logged.item()) / total
    b = total * (8 + 4 + 8 * f)
    out["round_log_replay_2^32"] = {"round_log_ms": round(ms_rl, 3), "replay_ms": round(ms_rp, 3),
                                     "round_log_gbs": round(b / ms_rl / 1e6, 1), "replay_gbs": round(b / ms_rp / 1e6, 1),
                                     "pair_gbs": round(2 * b / (ms_rl + ms_rp) / 1e6, 1),
                                     "frac_per_gpu": round(2 * b / (ms_rl + ms_rp) / 1e6 / peak / world, 4),
                                     "logged_fraction": round(f, 5)}
    del x, y, ya, words, lw, log, st
    torch.cuda.empty_cache()
    # --- configs[4] Merkle, sharded by whole 2^12-leaf blocks
    nparam = workloads.CONFIG4_PARAMS
    n_leaves = (nparam * 4 + 4095) // 4096
    l0, l1 = vdist.leaf_block_range(n_leaves, rank, world)
    p0, p1 = l0 * 1024, min(nparam, l1 * 1024)
    w = workloads.config4_weights_torch(nparam, device=dev, lo=p0, hi=p1) if p1 > p0 else \
        torch.empty(0, device=dev)
    wb = w.view(torch.uint8)
    res = {}
    dx = None  # N > 1 over NCCL: the block roots travel over peer memory (DigestExchange)
    if dist.is_initialized() and args.dist_backend == "nccl":
        try:
            n_blocks = (n_leaves + (1 << vdist.BLOCK_LEAVES_LOG2) - 1) >> vdist.BLOCK_LEAVES_LOG2
            dx = vdist.DigestExchange(n_blocks, device=dev)
        except Exception as e:  # noqa: BLE001
            print(f"[bench] symmetric-memory block-root exchange unavailable, using NCCL: {e!r}", file=sys.stderr)

    def mk():
        res["lv"], res["top"] = vdist.merkle_sharded(wb, n_leaves, exchange=dx, check=False)

    ms_m = timed(mk, 3)
    if dx is not None:
        dx.check()
    root = bytes(res["top"][-1][0].cpu().numpy())
    del w, wb, res
    torch.cuda.empty_cache()
    same = None
    if rank == 0:  # the single-GPU tree over the whole checkpoint (untimed)
        wall = workloads.config4_weights_torch(nparam, device=dev)
        same = merkle.merkle_chunked(wall).root == root
        del wall
        torch.cuda.empty_cache()
    out["merkle_1.5B"] = {"ms": round(ms_m, 3), "hashed_gbs": round(nparam * 4 / ms_m / 1e6, 1),
                          "root": root.hex()[:16], "root_equals_single_gpu": same,
                          "block_roots": ("peer memory (vt_merkle_level_exchange + vt_digests_wait)" if dx is not None
                                          else "all-gather" if world > 1 else "local")}
    # --- one 2^30-element tensor's budget search, sharded (SURVEY §8e tau search)
    total_b = 1 << 30
    lo_b, hi_b = vdist.shard_range(total_b, rank, world)
    gx = torch.Generator(device=dev)
    gx.manual_seed(30 + rank)
    xb_ = torch.randn(hi_b - lo_b, dtype=torch.float64, device=dev, generator=gx)
    Bb = int(0.005 * total_b)
    bx = None
    if args.dist_backend == "nccl" or not dist.is_initialized():
        try:
            bx = vdist.BudgetExchange(device=dev)
        except Exception as e:  # noqa: BLE001
            print(f"[bench] symmetric-memory budget exchange unavailable, using NCCL: {e!r}", file=sys.stderr)
    rb = {}

    def bs():
        rb["tau"] = vdist.search_tau_budget_sharded(xb_, 32, Bb, exchange=bx, n_global=total_b)

    ms_b = timed(bs, 3)  # wall-inclusive: each search ends in one host read of (status, tau)
    out["budget_search_2^30_sharded"] = {"ms": round(ms_b, 3), "gbs": round(8 * total_b / ms_b / 1e6, 1),
                                         "tau_over_2^-24": round(rb["tau"] / 2.0 ** -24, 6),
                                         "exchange": "peer memory (vt_tau_shard_search_x)" if bx is not None
                                         else "NCCL + host decision"}
    del xb_
    torch.cuda.empty_cache()
    # --- configs[2], LPT over ranks
    xs = workloads.config2_tensors_torch(device=dev)
    sizes = [t.numel() for t in xs]
    budgets = workloads.config2_budgets(sizes)
    owner = vdist.lpt_assign(sizes, world)
    mine = [i for i in range(len(xs)) if owner[i] == rank]
    mx = [xs[i] for i in mine]
    mb = [budgets[i] for i in mine]
    ys = [torch.empty(t.numel(), dtype=torch.float32, device=dev) for t in mx]
    lws = [torch.empty(B + 1, dtype=torch.int64, device=dev) for B in mb]
    r2 = {}

    def c2():
        r2["b"] = ops.round_and_log_adaptive_batch(mx, 32, mb, outs=ys, log_outs=lws, check=False)

    ms_c2 = timed(c2, 3)
    taus = torch.zeros(len(xs), dtype=torch.float64, device=dev)
    if mine:
        taus[torch.tensor(mine, device=dev)] = r2["b"].taus
    if dist.is_initialized():
        dist.all_reduce(taus)
    same2 = None
    if rank == 0 and dist.is_initialized():
        full = ops.round_and_log_adaptive_batch(xs, 32, budgets, check=False)
        same2 = bool(torch.equal(full.taus, taus))
    out["configs[2]_lpt"] = {"ms": round(ms_c2, 3), "elements": int(sum(sizes)),
                             "g_elements_per_s": round(sum(sizes) / ms_c2 / 1e6, 2),
                             "max_rank_elements": int(max(np.bincount(owner, weights=sizes, minlength=world))),
                             "taus_equal_single_gpu": same2}
    del xs, mx, ys, lws, r2
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------------------
# CPU: the reference algorithm on the host cores
#
# The reference's own functions (vtrain 0.1.0 from baseline/_ref, installed
# by tools/install_reference.sh) when present -- kind "reference" -- else the
# oracle port of them (oracle/vt_oracle.py) -- kind "port".  Inputs are
# generated before the timed region and shared with a forked process pool
# (copy-on-write, no pickling); every timing is same-run WALL clock around the
# pool's map (the pool is started and warmed first), at P = 1 and P = all
# host cores, with the core count and CPU model stated.
# ---------------------------------------------------------------------------

_CPU: dict = {}


class _Impl:
    """direction_array / rnd_array / rev_array / exponent_scale_array / pack."""

    def __init__(self):
        ref = REPO / "baseline" / "_ref"
        if (ref / "vtrain" / "fpround.py").exists():
            sys.path.insert(0, str(ref))
            from vtrain import fpround as F
            from vtrain import roundlog as R
            self.direction_array, self.rnd_array, self.rev_array = F.direction_array, F.rnd_array, F.rev_array
            self.exponent_scale_array, self.pack = F.exponent_scale_array, R._pack_block
            self.kind = "reference"
            self.what = "vtrain 0.1.0 functions (baseline/_ref, unmodified)"
        else:
            sys.path.insert(0, str(REPO / "oracle"))
            import vt_oracle as O
            self.direction_array, self.rnd_array, self.rev_array = O.direction_array, O.rnd_array, O.rev_array
            self.exponent_scale_array, self.pack = O.exponent_scale_array, O.pack_groups
            self.kind = "port"
            self.what = "oracle/vt_oracle.py (NumPy restatement of the reference functions)"


def _impl() -> _Impl:
    if "impl" not in _CPU:
        _CPU["impl"] = _Impl()
    return _CPU["impl"]


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _pool(procs: int):
    import multiprocessing as mp
    pool = mp.get_context("fork").Pool(procs)
    pool.map(abs, range(4 * procs))  # workers up before any timing
    return pool


def _timed_map(fn, jobs, procs: int):
    """(results, wall seconds): in process for P = 1, else a warmed pool."""
    if procs <= 1:
        t0 = time.perf_counter()
        res = [fn(j) for j in jobs]
        return res, time.perf_counter() - t0
    with _pool(procs) as pool:
        t0 = time.perf_counter()
        res = pool.map(fn, jobs)
        wall = time.perf_counter() - t0
    return res, wall


def _pair_job(job):
    """The trainer channel (protocol.py:198-202: direction_array, write_array's
    _pack_block, rnd_array) and the auditor channel (protocol.py:212-216:
    rev_array, rnd_array for the correction count) on one chunk."""
    import numpy as np
    lo, hi = job
    F = _impl()
    xt, xa = _CPU["xt"][lo:hi], _CPU["xa"][lo:hi]
    tau = _CPU["tau"]
    codes = F.direction_array(xt, 32, tau)
    F.pack(np.concatenate([codes, np.ones((-codes.size) % 5, np.uint8)]))
    F.rnd_array(xt, 32)
    ya = F.rev_array(xa, 32, codes)
    corr = int(np.count_nonzero(ya != F.rnd_array(xa, 32)))
    return hi - lo, int(np.count_nonzero(codes != 1)), corr


def cpu_pair(total: int, procs: int, chunk: int | None = None, seed: int = 100) -> dict:
    """configs[1] pair over ``total`` elements: GB/s of the step's algorithmic
    bytes (both channels, the GPU formula) over the same-run wall clock.
    Chunks of 2^22 elements, smaller when needed so every
    process has at least two."""
    from paper_2403_09603_b200 import workloads
    if chunk is None:
        chunk = max(1 << 16, min(1 << 22, total // (2 * max(procs, 1))))
    key = ("pair", total, seed)
    if _CPU.get("pair_key") != key:  # inputs generated once per size, outside every timed region
        _CPU["pair_inputs"] = workloads.config1_pair(total, seed)
        _CPU["pair_key"] = key
    xt, xa = _CPU["pair_inputs"]
    _CPU.update(xt=xt, xa=xa, tau=workloads.TAU_CONFIG0)
    jobs = [(lo, min(total, lo + chunk)) for lo in range(0, total, chunk)]
    try:
        res, wall = _timed_map(_pair_job, jobs, procs)
    finally:
        for k in ("xt", "xa"):
            _CPU.pop(k, None)
    n = sum(r[0] for r in res)
    f = sum(r[1] for r in res) / n
    return {"gbs": n * (8 + 4 + 8 * f) * 2 / wall / 1e9, "n": n, "wall_s": wall, "f": f, "procs": procs,
            "chunk": chunk}


def _budget_job(job):
    """Budget search (the search_tau skeleton of protocol.py:494-506
    with predicate count(p > tau) <= B on the exact p = |x - rnd(x)| /
    max(scale, 2^-126), fpround.py:171-173) then the trainer channel at tau."""
    import numpy as np
    i = job
    F = _impl()
    x = _CPU["tensors"][i]
    B = int(0.005 * x.size)
    r = F.rnd_array(x, 32)
    p = np.abs(x - r) / np.maximum(F.exponent_scale_array(x), 2.0 ** -126)
    lo, hi = 2.0 ** -25, 2.0 ** -24
    for _ in range(30):
        t = (lo + hi) / 2.0
        if int(np.count_nonzero(p > t)) <= B:
            hi = t
        else:
            lo = t
    codes = F.direction_array(x, 32, hi)
    F.pack(np.concatenate([codes, np.ones((-codes.size) % 5, np.uint8)]))
    F.rnd_array(x, 32)
    return x.size, int(np.count_nonzero(codes != 1))


def cpu_budget(sizes: list[int], procs: int, seed: int) -> dict:
    """Per-tensor budget search + round-and-log over independent tensors
    (one tensor per job), x ~ N(0, sigma_t), sigma_t log-uniform [1e-3, 10]."""
    import numpy as np
    rng = np.random.default_rng(seed)
    _CPU["tensors"] = [rng.standard_normal(int(n)) * 10.0 ** rng.uniform(-3, 1) for n in sizes]
    try:
        res, wall = _timed_map(_budget_job, list(range(len(sizes))), procs)
    finally:
        _CPU.pop("tensors", None)
    n = sum(r[0] for r in res)
    return {"elements": n, "wall_s": round(wall, 3), "g_elements_per_s": round(n / wall / 1e9, 5), "procs": procs}


def _leaf_job(job):
    import hashlib
    lo, hi = job
    raw, lb = _CPU["w"], 4096
    return b"".join(hashlib.sha256(raw[i * lb:(i + 1) * lb]).digest() for i in range(lo, hi))


def cpu_merkle(n_leaves: int, procs: int) -> dict:
    """hashlib (OpenSSL, the reference's SHA-256, merkle.py:24-25) over 4 KiB
    leaves of FP32 N(0, 0.02) weights on ``procs`` processes, then the level
    build of merkle.build (merkle.py:55-72) in one process; wall clock."""
    import hashlib

    import numpy as np
    _CPU["w"] = memoryview(np.random.default_rng(4).normal(0.0, 0.02, size=n_leaves * 1024).astype("<f4")).cast("B")
    per = max(1, n_leaves // (4 * max(procs, 1)))
    jobs = [(lo, min(n_leaves, lo + per)) for lo in range(0, n_leaves, per)]
    try:
        res, wall = _timed_map(_leaf_job, jobs, procs)
    finally:
        _CPU.pop("w", None)
    leaves = b"".join(res)
    t0 = time.perf_counter()
    cur = [leaves[i:i + 32] for i in range(0, len(leaves), 32)]
    while len(cur) > 1:
        nxt = [hashlib.sha256(cur[i] + cur[i + 1]).digest() for i in range(0, len(cur) - 1, 2)]
        if len(cur) % 2:
            nxt.append(cur[-1])
        cur = nxt
    wall += time.perf_counter() - t0
    return {"gbs_hashed": round(n_leaves * 4096 / wall / 1e9, 4), "wall_s": round(wall, 3), "procs": procs,
            "leaves": n_leaves}


def _cores() -> int:
    return len(os.sched_getaffinity(0))


def cpu_baseline(args) -> dict:
    """The headline's cpu_baseline: the configs[1] pair at P = all (bounded
    sample of 2^cpu_log2n elements) and P = 1 (2^22 elements)."""
    cores = _cores()
    F = _impl()
    r = cpu_pair(1 << args.cpu_log2n, cores)
    r1 = cpu_pair(1 << 22, 1)
    return {"value": round(r["gbs"], 4), "unit": "GB/s", "cores": cores, "kind": F.kind,
            "value_1core": round(r1["gbs"], 4),
            "sample": f"2^{args.cpu_log2n} elements of the configs[1] pair in chunks of {r['chunk']} over {cores} "
                      f"processes (P=1: 2^22 elements in process); trainer channel: direction_array + _pack_block + "
                      f"rnd_array; "
                      f"auditor: rev_array + rnd_array count; same-run wall clock {r['wall_s']:.2f}s / "
                      f"{r1['wall_s']:.2f}s; {F.what}",
            "cpu_model": _cpu_model()}


def cpu_legs() -> dict:
    """CPU rows for the other configs, P = 1 and P = all."""
    import numpy as np

    from paper_2403_09603_b200 import workloads
    cores = _cores()
    F = _impl()
    out = {"cores": cores, "cpu_model": _cpu_model(), "kind": F.kind, "functions": F.what}
    shapes = [int(np.prod(s)) for _, s in workloads.resnet50_tensors()]
    sample = shapes[::8]  # every 8th of the 161 tensors (1/8 of the elements, all layer kinds)
    c2 = cpu_budget(sample, cores, 2)
    c2_1 = cpu_budget([1 << 22], 1, 2)
    out["configs[2]_budget_round_log"] = {
        "P_all": c2, "P_1": c2_1, "unit": "G elements/s",
        "sample": f"{len(sample)} of the 161 ResNet-50 tensors (every 8th, {sum(sample)} elements), one tensor per "
                  f"process; P=1: one 2^22-element tensor",
        "sweep_s_extrapolated_P_all": round(1_052_589_312 / (c2["g_elements_per_s"] * 1e9), 2)}
    # GPT-2 small, batch 8 x 1024: the hooked tensors' sizes (d = 768, 4d MLP)
    d_act, mlp_act = 8 * 1024 * 768, 8 * 1024 * 3072
    sample3 = [d_act] * 12 + [mlp_act] * 4
    c3 = cpu_budget(sample3, cores, 3)
    c3_1 = cpu_budget([d_act], 1, 3)
    out["configs[3]_gpt2_hooked_trainer_channel"] = {
        "P_all": c3, "P_1": c3_1, "unit": "G elements/s",
        "sample": "16 hooked-tensor shapes of the GPT-2-small step (12 x 8x1024x768, 4 x 8x1024x3072), budget "
                  "search + trainer channel each; P=1: one 8x1024x768 tensor",
        # 2.96e9 hooked elements per step: 88 outputs, 86 input gradients, the loss gradient
        "step_s_extrapolated_P_all": round(2.96e9 / (c3["g_elements_per_s"] * 1e9), 2)}
    m_all = cpu_merkle(1 << 18, cores)
    m_1 = cpu_merkle(1 << 15, 1)
    out["configs[4]_merkle"] = {"P_all": m_all, "P_1": m_1, "unit": "GB/s hashed",
                                "sample": "2^18 leaves (1 GiB) at P=all, 2^15 leaves at P=1; hashlib leaves + "
                                          "merkle.build levels",
                                "tree_s_extrapolated_P_all": round(6e9 / (m_all["gbs_hashed"] * 1e9), 2)}
    return out


def run_reference(args) -> None:
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cores = _cores()
    F = _impl()
    total = 1 << args.cpu_log2n
    for _ in range(min(args.warmup, 1)):
        cpu_pair(1 << 20, 1)
    vals = []
    t_all = time.perf_counter()
    for _ in range(args.steps):
        vals.append(cpu_pair(total, cores))
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
                   "sample": (f"each step times the whole pair (2^{args.cpu_log2n} elements)"
                              if args.cpu_log2n == args.log2n else
                              f"each step times a bounded sample of 2^{args.cpu_log2n} elements of that pair")},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": cores, "kind": F.kind,
                         "sample": f"2^{args.cpu_log2n} elements per step in chunks of {vals[-1]['chunk']} over {cores} "
                                   f"processes, wall clock; {F.what}",
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
    ap.add_argument("--cpu-log2n", type=int, default=26)  # the reference arm times the whole configs[1] pair per step
    ap.add_argument("--sweep", type=int, nargs="*", default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-extras", dest="extras", action="store_false",
                    help="skip the configs[2]/[3]/[4] extras, the size sweep and the strong-scaling legs at N=1")
    ap.add_argument("--harness-check", action="store_true",
                    help="CPU self-test of the multi-rank launcher (gloo, no kernels; tests only)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: every rank on GPU 0, host collectives -- a code-path check, not a measurement")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    maybe_spawn(args)
    if args.harness_check:
        run_harness_check(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
