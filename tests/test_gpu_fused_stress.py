"""GPU stress of the single-pass round-and-log kernel (rl_fused_kernel):
super-tile / tile boundaries, dense logs (the staged-row overflow paths),
repeated calls on one workspace (epoch + ticket reset), and two streams
running the kernel concurrently (ticketed super-tiles must not deadlock or
mix when the grids are not co-resident).  Everything is checked against the
oracle (vtrain fpround.direction_array / rnd_array restated) bit for bit."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu

SUPER = 8192  # elements per look-back super-tile
TILE = 2048


def _check(oracle, x, tau, base, y, log):
    codes = oracle.direction_array(x, 32, tau)
    want = oracle.sparse_from_codes(codes, base=base)
    assert log.count == want.size
    assert np.array_equal(log.words[: log.count].cpu().numpy().view(np.uint64), want)
    assert np.array_equal(bits(y.cpu().numpy()), bits(oracle.rnd_array(x, 32).astype(np.float32)))


@pytest.mark.parametrize("n", [TILE - 1, TILE, TILE + 1, SUPER - 1, SUPER, SUPER + 1, 3 * SUPER + 5,
                               444 * SUPER - 1, 450 * SUPER + TILE + 17])
def test_super_tile_boundaries(oracle, n):
    import torch
    from paper_2403_09603_b200 import ops, workloads
    x = workloads.config0_x(n, seed=n % 1000)
    tau = workloads.TAU_CONFIG0
    y, log = ops.round_and_log(torch.from_numpy(x).cuda(), 32, tau, global_base=3 * n + 1)
    _check(oracle, x, tau, 3 * n + 1, y, log)


@pytest.mark.parametrize("frac", [1.0, 0.3, 0.2, 0.15])
def test_dense_logs(oracle, frac):
    """Logged fractions whose 256-element warp-tiles overflow the 64-entry
    staged rows (frac >= 0.3) or need their second half (0.15-0.2)."""
    import torch
    from paper_2403_09603_b200 import ops
    n = 37 * SUPER + 1234
    x = np.random.default_rng(11).normal(0.0, 3.0, n)
    # p ~ U[0, 2^-24] for N(0, s) data: logged iff p > tau
    tau = 0.0 if frac == 1.0 else (1.0 - frac) * 2.0 ** -24
    y, log = ops.round_and_log(torch.from_numpy(x).cuda(), 32, tau, global_base=5)
    _check(oracle, x, tau, 5, y, log)
    assert abs(log.count / n - frac) < 0.02


def test_dense_general_grid(oracle):
    """b_r < 32 (non-fast path) with a dense log."""
    import torch
    from paper_2403_09603_b200 import ops
    n = 9 * SUPER + 77
    x = np.random.default_rng(12).normal(0.0, 1.0, n)
    y, log = ops.round_and_log(torch.from_numpy(x).cuda(), 26, 0.0, out_dtype=torch.float64)
    codes = oracle.direction_array(x, 26, 0.0)
    assert np.array_equal(log.words[: log.count].cpu().numpy().view(np.uint64), oracle.sparse_from_codes(codes))
    assert np.array_equal(bits(y.cpu().numpy()), bits(oracle.rnd_array(x, 26)))


def test_repeated_calls_one_workspace(oracle):
    """Epoch-tagged status words and the ticket counter survive many calls of
    varying size on the same workspace."""
    import torch
    from paper_2403_09603_b200 import ops, workloads
    tau = workloads.TAU_CONFIG0
    sizes = [SUPER * 600 + 3, 5000, SUPER * 17, 1, SUPER * 600 + 3, 123457]
    xs = [workloads.config0_x(n, seed=i) for i, n in enumerate(sizes)]
    want = [oracle.sparse_from_codes(oracle.direction_array(x, 32, tau)) for x in xs]
    xd = [torch.from_numpy(x).cuda() for x in xs]
    for rep in range(40):
        i = rep % len(sizes)
        _, log = ops.round_and_log(xd[i], 32, tau)
        assert log.count == want[i].size, (rep, i)
        if rep % 7 == 0 or sizes[i] < 10000:
            assert np.array_equal(log.words[: log.count].cpu().numpy().view(np.uint64), want[i])
        else:
            w = log.words[: log.count]
            assert int(w[0]) == int(want[i][0]) and int(w[-1]) == int(want[i][-1])
            assert bool((w[1:] > w[:-1]).all())


@pytest.mark.timeout(300)
def test_two_streams_concurrent():
    """Two grids of resident size on two streams at once: CTAs of one grid may
    wait for SMs held by the other, so super-tiles are handed out by ticket
    and a CTA only ever waits on lower tickets.  Results must equal the
    sequential ones."""
    import torch
    from paper_2403_09603_b200 import _device as D
    from paper_2403_09603_b200 import _lib, ops, workloads
    tau = workloads.TAU_CONFIG0
    n = 1 << 24
    xs = [workloads.config0_x_torch(n, s) for s in (21, 22)]
    ref = []
    for x in xs:
        y, log = ops.round_and_log(x, 32, tau)
        ref.append((y.clone(), log.words[: log.count].clone()))
    lib = _lib.lib()
    streams = [torch.cuda.Stream() for _ in xs]
    wss = [torch.zeros(int(lib.vt_round_log_workspace(n)), dtype=torch.uint8, device="cuda") for _ in xs]
    ys = [torch.empty(n, dtype=torch.float32, device="cuda") for _ in xs]
    words = [torch.empty(n // 4, dtype=torch.int64, device="cuda") for _ in xs]
    flags = [D.Flags() for _ in xs]
    torch.cuda.synchronize()
    for rep in range(25):
        for fl in flags:
            fl.buf.zero_()
        torch.cuda.synchronize()
        for i, x in enumerate(xs):
            with torch.cuda.stream(streams[i]):
                _lib.call("vt_round_log", D.ptr(x), n, 32, float(tau), _lib.OUT_F32, D.ptr(ys[i]),
                          D.ptr(words[i]), words[i].numel(), 0, None, None, None, None, 0, None,
                          flags[i].cnt_ptr, flags[i].err_ptr, D.ptr(wss[i]), wss[i].numel(),
                          streams[i].cuda_stream)
        torch.cuda.synchronize()
        for i in range(len(xs)):
            err, cnt = flags[i].read()
            assert err == 0 and cnt[0] == ref[i][1].numel(), (rep, i, cnt[0])
            assert torch.equal(words[i][: cnt[0]], ref[i][1])
            assert torch.equal(ys[i].view(torch.int32), ref[i][0].view(torch.int32))


def test_epoch_wrap_clears_stale_status(oracle):
    """The look-back status words carry a 20-bit epoch.  Plant words that
    would pass for the first epoch after the wrap (as a call 2^20 calls
    earlier could have left them) and run across the wrap: the call holding
    the last epoch value must clear them first."""
    import torch
    from paper_2403_09603_b200 import _device as D
    from paper_2403_09603_b200 import _lib, workloads
    lib = _lib.lib()
    tau = workloads.TAU_CONFIG0
    big, small = 300 * SUPER + 77, 3 * SUPER
    ws = torch.zeros(int(lib.vt_round_log_workspace(big)), dtype=torch.uint8, device="cuda")
    hdr = ws[:64].view(torch.int32)
    status = ws[64:64 + 8 * 320].view(torch.int64)
    mask = (1 << 20) - 1
    hdr[0] = mask - 1        # the next call runs with the last epoch value
    hdr[3] = 320             # high-water mark: some earlier call wrote 320 words
    status[:] = (1 << 44) | (2 << 42) | 12345  # INC words tagged with epoch 1, garbage prefixes

    def run(x):
        n = x.numel()
        y = torch.empty(n, dtype=torch.float32, device="cuda")
        words = torch.empty(n // 4, dtype=torch.int64, device="cuda")
        f = D.Flags()
        _lib.call("vt_round_log", D.ptr(x), n, 32, float(tau), _lib.OUT_F32, D.ptr(y), D.ptr(words), words.numel(),
                  0, None, None, None, None, 0, None, f.cnt_ptr, f.err_ptr, D.ptr(ws), ws.numel(), D.stream_ptr())
        err, cnt = f.read()
        assert err == 0
        return words[: cnt[0]].cpu().numpy().view(np.uint64)

    xs = workloads.config0_x(small, 1)
    xb = workloads.config0_x(big, 2)
    want_s = oracle.sparse_from_codes(oracle.direction_array(xs, 32, tau))
    want_b = oracle.sparse_from_codes(oracle.direction_array(xb, 32, tau))
    assert np.array_equal(run(torch.from_numpy(xs).cuda()), want_s)  # epoch = mask: clears, wraps to 0
    assert int(hdr[0]) == 0
    assert np.array_equal(run(torch.from_numpy(xb).cuda()), want_b)  # epoch 1: planted words are gone
    assert int(hdr[0]) == 1


def _torch_words(x, tau, base):
    """Torch FP64 restatement of direction_array's predicate for b_r = 32
    (fpround.py:164-177): p = |x - r| / max(2^E, 2^-126) > tau (exact: the
    divisor is a power of two), UP iff x < r; words (base + i) << 1 | up."""
    import torch
    r = x.float().double()
    _, e = torch.frexp(x)
    scale = torch.clamp(torch.ldexp(torch.ones_like(x), (e - 1).to(torch.int32)), min=2.0 ** -126)
    logged = (x - r).abs() / scale > tau
    idx = torch.nonzero(logged).flatten()
    return ((idx + base) << 1) | (x[idx] < r[idx]).to(torch.int64)


@pytest.mark.slow
@pytest.mark.timeout(900)
def test_max_size_properties():
    """2^32 + 12345 elements (global indices past 32 bits, 524,290 tickets):
    every log word against a torch FP64 restatement of the direction
    predicate, chunk by chunk; FP32 output == x.float(); replay of the same
    input reproduces it with no corrections."""
    import torch
    from paper_2403_09603_b200 import ops, workloads
    n = (1 << 32) + 12345
    tau = workloads.TAU_CONFIG0
    base = 7
    x = workloads.config0_x_torch_bernoulli(n, seed=32)
    y, log = ops.round_and_log(x, 32, tau, global_base=base, log_out=torch.empty(n // 8, dtype=torch.int64,
                                                                                     device="cuda"))
    assert 0.09 * n < log.count < 0.11 * n
    pos = 0
    chunk = 1 << 28
    for lo in range(0, n, chunk):
        xs = x[lo:lo + chunk]
        assert torch.equal(y[lo:lo + chunk].view(torch.int32), xs.float().view(torch.int32))
        want = _torch_words(xs, tau, base + lo)
        got = log.words[pos:pos + want.numel()]
        assert torch.equal(got, want), lo
        pos += want.numel()
    assert pos == log.count
    y2, corr = ops.replay(x, 32, log, global_base=base)
    assert corr == 0 and torch.equal(y2.view(torch.int32), y.view(torch.int32))
