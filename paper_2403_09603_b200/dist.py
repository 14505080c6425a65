"""Contiguous sharding of the hot path across the GPUs of one box.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  The
path shards naturally:

* round-and-log: rank r owns elements [lo_r, hi_r) (boundaries on the
  640-element warp grid) and emits sparse entries with GLOBAL indices;
  the only exchange is an all-gather of the per-rank entry counts, whose
  exclusive prefix places each rank's slice in the global log (concatenation
  in rank order is the reference order).  The log itself stays sharded.
  The exchange is fused into the round-and-log kernel over peer memory
  (``CountExchange``: the last CTA stores the count into every rank's
  symmetric-memory buffer, a wait kernel collects them), or an NCCL
  all-gather.
* replay: each rank consumes its own slice; corrections are all-reduced.
* adaptive threshold: independent tensors go to ranks whole, LPT-balanced
  (``lpt_assign``; no collective beyond gathering the taus).  One tensor
  sharded across ranks (``search_tau_budget_sharded``): one read of each
  shard for the candidates above the global plan's threshold, an all-reduce
  of their digit histogram (16 KiB), an all-gather of the keys in the
  selected digit, the exact order statistic and the FP64 bisection; the
  exact radix select pass by pass (histograms summed over the ranks) as
  the fallback.
* Merkle: leaves are grouped in blocks of 2^K; each rank hashes a
  contiguous run of blocks and builds levels 0..K locally (fewer when the
  whole tree fits one block), all ranks all-gather the block roots and build
  the top levels redundantly.  Every level of ``merkle.build`` over the full
  leaf list is reproduced, and no more (``assemble_levels``; the promotion
  rule only acts at the right edge, which is the last rank's).

The combination logic is pure host arithmetic over tensors (``*_plan`` /
``combine_*``) so it is unit-tested with the gloo backend on CPU; the
device work is the same single-GPU kernels.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

SHARD_ALIGN = 640  # lcm(5 codes per .vtrl byte, 128 elements per warp slot)
BLOCK_LEAVES_LOG2 = 12


def shard_range(n: int, rank: int, world: int, align: int = SHARD_ALIGN) -> tuple[int, int]:
    """Contiguous [lo, hi) of rank; interior boundaries are multiples of align,
    the last rank takes the remainder."""
    units = (n + align - 1) // align
    per, extra = divmod(units, world)
    lo_u = rank * per + min(rank, extra)
    hi_u = lo_u + per + (1 if rank < extra else 0)
    return min(lo_u * align, n), min(hi_u * align, n)


def exclusive_offsets(counts: torch.Tensor) -> torch.Tensor:
    return torch.cumsum(counts, 0) - counts


def _world(group=None) -> int:
    """World size; 1 without an initialised process group (single process)."""
    return dist.get_world_size(group) if dist.is_initialized() else 1


def _all_gather_flat(out: torch.Tensor, mine: torch.Tensor, group=None) -> None:
    """all_gather_into_tensor on NCCL; list form on backends without it (gloo);
    a copy in a single process."""
    if not dist.is_initialized():
        out.copy_(mine.reshape(out.shape))
        return
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, mine, group=group)
    else:
        parts = list(out.chunk(dist.get_world_size(group)))
        tmp = [torch.empty_like(p) for p in parts]
        dist.all_gather(tmp, mine, group=group)
        for p, t in zip(parts, tmp):
            p.copy_(t)


def all_gather_counts(count: int | torch.Tensor, group=None, device=None) -> torch.Tensor:
    """All ranks' int64 counts (one tiny NCCL all-gather over NVLink)."""
    world = _world(group)
    if isinstance(count, torch.Tensor):
        mine = count.reshape(1).to(torch.int64)
    else:
        mine = torch.tensor([int(count)], dtype=torch.int64, device=device)
    out = torch.empty(world, dtype=torch.int64, device=mine.device)
    _all_gather_flat(out, mine, group)
    return out


@dataclass
class ShardedLog:
    """This rank's slice of the global sparse log plus the global layout."""

    local: object          # ops.SparseLog with global indices
    offset: int            # position of local.words[0] in the global log
    total: int             # global entry count
    counts: torch.Tensor   # per-rank counts


class CountExchange:
    """The count exchange of a sharded round-and-log over peer memory: a
    symmetric-memory buffer per rank (``torch.distributed._symmetric_memory``,
    mapped into every peer over NVLink; a plain device buffer in a single
    process) and the two kernels that use it.  ``round_and_log`` runs the
    fused round-and-log whose last CTA stores the call's entry count into
    every rank's buffer (``vt_round_log_exchange``); ``wait`` launches the
    kernel that waits for every rank's count (``vt_counts_wait``).  No NCCL
    call, no host round trip: both are plain kernels on the current stream,
    so a whole step can be graph-captured.  Construction is collective (a
    symmetric-memory rendezvous): every rank of the group constructs its
    exchanges in the same order."""

    def __init__(self, group=None, device=None):
        from . import _device as D
        from . import _lib
        self.D, self.lib = D, _lib
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.world = _world(group)
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        words = int(_lib.lib().vt_exchange_words(self.world))
        if dist.is_initialized():
            import torch.distributed._symmetric_memory as symm
            self.buf = symm.empty(words, dtype=torch.int64, device=dev)
            self.buf.zero_()
            name = (group or dist.group.WORLD).group_name
            self.handle = symm.rendezvous(self.buf, name)
            self.peers = int(self.handle.buffer_ptrs_dev)
            torch.cuda.synchronize(dev)
            dist.barrier(group)  # every buffer is zero before any rank publishes
        else:
            self.buf = torch.zeros(words, dtype=torch.int64, device=dev)
            self._ptrs = torch.tensor([self.buf.data_ptr()], dtype=torch.int64, device=dev)
            self.peers = int(self._ptrs.data_ptr())
        self.counts = torch.zeros(self.world, dtype=torch.int64, device=dev)
        self.flags = torch.zeros(2, dtype=torch.int32, device=dev)

    def round_and_log(self, x_local: torch.Tensor, b_r: int, tau: float, global_base: int, *, out=None,
                      log_out=None, out_dtype=torch.float32, workspace=None):
        """ops.round_and_log(check=False) with the count published to every rank."""
        from . import ops
        from .fpround import _check_b
        _check_b(b_r)
        t = self.D.aligned_f64(x_local.reshape(-1)) if x_local.numel() else x_local.reshape(-1)
        n = t.numel()  # an empty shard still publishes (a count of 0)
        y = out if out is not None else torch.empty(n, dtype=out_dtype, device=t.device)
        self.D.check_out(y, n, out_dtype, t.device, "out")
        words = log_out if log_out is not None else torch.empty(ops.default_log_capacity(n), dtype=torch.int64,
                                                                device=t.device)
        need = int(self.lib.lib().vt_round_log_workspace(max(n, 1)))
        ws = workspace if workspace is not None else self.D.workspace(need, "round_log")
        f = self.D.Flags()
        self.lib.call("vt_round_log_exchange", self.D.ptr(t) if n else None, n, b_r, float(tau),
                      ops._out_kind(out_dtype),
                      self.D.ptr(y), self.D.ptr(words), words.numel(), int(global_base), f.cnt_ptr, f.err_ptr,
                      self.D.ptr(ws), ws.numel(), self.peers, self.world, self.rank, self.D.stream_ptr())
        return ops.PendingRound(y, words, f)

    def wait(self) -> torch.Tensor:
        """Enqueue the wait for every rank's count of the latest exchange;
        returns the device int64[world] they land in (valid in stream order)."""
        self.lib.call("vt_counts_wait", self.peers, self.world, self.rank, self.D.ptr(self.counts),
                      self.flags.data_ptr(), self.D.stream_ptr())
        return self.counts

    def check(self) -> None:
        if int(self.flags[0].item()) & self.lib.ERR_EXCHANGE:
            raise RuntimeError("count exchange: a peer's count did not arrive (10 s)")


def round_and_log_sharded(x_local: torch.Tensor, b_r: int, tau: float, global_base: int,
                          group=None, exchange: CountExchange | None = None, **kw):
    """Sharded round-and-log: this rank's log with global indices plus every
    rank's entry count -- through the peer-memory exchange fused into the
    kernel when ``exchange`` is given, else an NCCL all-gather."""
    from . import ops
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if exchange is not None:
        p = exchange.round_and_log(x_local, b_r, tau, global_base, **kw)
        counts = exchange.wait()
        y, log = p.finish()
        exchange.check()
        counts = counts.clone()
    else:
        y, log = ops.round_and_log(x_local, b_r, tau, global_base=global_base, **kw)
        counts = all_gather_counts(log.count, group, device=x_local.device)
    offs = exclusive_offsets(counts)
    return y, ShardedLog(log, int(offs[rank]), int(counts.sum()), counts)


def replay_sharded(xa_local: torch.Tensor, b_r: int, slog: ShardedLog, global_base: int,
                   group=None, **kw):
    from . import ops
    y, corr = ops.replay(xa_local, b_r, slog.local, global_base=global_base, **kw)
    t = torch.tensor([corr], dtype=torch.int64, device=xa_local.device)
    if dist.is_initialized():
        dist.all_reduce(t, group=group)
    return y, int(t.item())


# ---------------------------------------------------------------------------
# adaptive threshold
# ---------------------------------------------------------------------------

def lpt_assign(sizes: list[int], world: int) -> list[int]:
    """Owner rank of each independent tensor: longest processing time first
    (largest tensor to the least loaded rank; ties to the lower index), so
    the largest per-rank load is within one tensor of the best split."""
    order = sorted(range(len(sizes)), key=lambda i: (-int(sizes[i]), i))
    loads = [0] * world
    owner = [0] * len(sizes)
    for i in order:
        r = min(range(world), key=lambda q: (loads[q], q))
        owner[i] = r
        loads[r] += int(sizes[i])
    return owner


class ShardedKth:
    """One rank's side of the exact order statistic of p over a tensor
    sharded across ranks (vt_tau_kth_begin / hist / select): pass by pass,
    this rank's histogram, summed over the ranks by the caller, then the
    same selection on every rank."""

    PASSES = 5

    def __init__(self, x_local: torch.Tensor, b_r: int, tag: str = "kth_sharded"):
        from . import _device as D
        from . import _lib
        self.D, self.lib = D, _lib
        self.t = D.aligned_f64(x_local.reshape(-1))
        self.b_r = b_r
        self.ws = D.workspace(int(_lib.lib().vt_tau_workspace(self.t.numel())), tag)
        self.key = torch.zeros(1, dtype=torch.int64, device=self.t.device)
        self.flags = D.Flags()

    def begin(self, rank: int) -> None:
        self.lib.call("vt_tau_kth_begin", int(rank), self.D.ptr(self.key), self.D.ptr(self.ws), self.ws.numel(),
                      self.D.stream_ptr())

    def local_hist(self, p: int) -> torch.Tensor:
        """Run this rank's pass-p histogram; returns the (int32 view of the)
        uint32 bins to be summed over the ranks in place."""
        self.lib.call("vt_tau_kth_hist", self.D.ptr(self.t), self.t.numel(), self.b_r, p, self.flags.err_ptr,
                      self.D.ptr(self.ws), self.ws.numel(), self.D.stream_ptr())
        off = int(self.lib.lib().vt_tau_kth_hist_offset(p))
        bins = int(self.lib.lib().vt_tau_kth_hist_bins(p))
        return self.ws[off:off + 4 * bins].view(torch.int32)

    def select(self, p: int) -> None:
        self.lib.call("vt_tau_kth_select", p, self.D.ptr(self.key), self.D.ptr(self.ws), self.ws.numel(),
                      self.D.stream_ptr())

    def value(self) -> float:
        self.D.raise_fpround(self.flags.read()[0])
        return float(self.key.cpu().numpy().view(np.float64)[0])


def kth_largest_distance_sharded(x_local: torch.Tensor, b_r: int, rank: int, group=None) -> float:
    """(rank+1)-th largest p over the union of every rank's shard, exactly
    (rank 0-based from the top); 0.0 when the union has at most rank elements."""
    world = _world(group)
    n = torch.tensor([x_local.numel()], dtype=torch.int64, device=x_local.device)
    if world > 1:
        dist.all_reduce(n, group=group)
    if rank >= int(n.item()):
        return 0.0
    sk = ShardedKth(x_local, b_r)
    sk.begin(rank)
    for p in range(ShardedKth.PASSES):
        h = sk.local_hist(p)
        if world > 1:  # uint32 counts summed as int32: exact modulo 2^32
            dist.all_reduce(h, group=group)
        sk.select(p)
    return sk.value()


SHARD_BINS = 2048  # top-digit bins of the candidate keys (kAdBins)
SHARD_XWORDS = SHARD_BINS + 3  # + keys above tau_hi, candidates, overflow flag


class ShardedBudget:
    """One rank's side of the budget search over a tensor sharded across ranks,
    through the candidate path (vt_tau_shard_*): the caller sums
    ``candidates()`` over the ranks, every rank ``decide``s identically, the
    caller gathers ``digit_keys`` from every rank, and ``finish`` selects the
    exact order statistic.  The plan (candidate threshold L, digit shift)
    depends only on the GLOBAL n and budget, so it is the same on every rank."""

    def __init__(self, x_local: torch.Tensor, b_r: int, n_global: int, budget: int, tag: str = "tau_shard"):
        import ctypes as C

        from . import _device as D
        from . import _lib
        self.D, self.lib = D, _lib
        self.t = D.aligned_f64(x_local.reshape(-1)) if x_local.numel() else x_local.reshape(-1).to(torch.float64)
        self.n = int(self.t.numel())
        self.b_r, self.n_global, self.budget = int(b_r), int(n_global), int(budget)
        dev = self.t.device if self.t.is_cuda else torch.device("cuda", torch.cuda.current_device())
        self.ws = D.workspace(int(_lib.lib().vt_tau_shard_workspace(self.n)), tag)
        self.flags = D.Flags()
        self.dev = dev
        L, s0 = C.c_uint64(0), C.c_int(0)
        _lib.call("vt_tau_shard_plan", self.n_global, self.b_r, self.budget, C.byref(L), C.byref(s0))
        self.L_key, self.s0 = int(L.value), int(s0.value)
        self.digit_count = 0

    def candidates(self) -> torch.Tensor:
        """int64[SHARD_XWORDS]: this rank's digit histogram, keys above tau_hi,
        candidate count, overflow flag -- to be summed over the ranks."""
        xb = torch.empty(SHARD_XWORDS, dtype=torch.int64, device=self.dev)
        self.lib.call("vt_tau_shard_candidates", self.D.ptr(self.t) if self.n else None, self.n, self.b_r,
                      self.n_global, self.budget, self.D.ptr(xb), self.flags.err_ptr, self.D.ptr(self.ws),
                      self.ws.numel(), self.D.stream_ptr())
        return xb

    def decide(self, xsum) -> tuple[str, object, int]:
        """From the summed exchange buffer: ("value", v, -) when the keys above
        tau_hi or the candidates settle v, ("digit", d, rank_in_digit) when the
        digit's keys must be gathered (``self.digit_count`` = their number over
        all ranks), ("exact", None, -) for the exact multi-pass fallback
        (overflow, or fewer candidates than budget + 1 above a threshold
        L > tau_lo)."""
        from .fpround import tau_bounds
        self.D.raise_fpround(self.flags.read()[0])
        xs = np.asarray(xsum, dtype=np.int64)
        hist, above_hi, m, overflow = xs[:SHARD_BINS], int(xs[SHARD_BINS]), int(xs[SHARD_BINS + 1]), \
            int(xs[SHARD_BINS + 2])
        lower, upper = tau_bounds(self.b_r)
        B = self.budget
        if self.n_global <= B:
            return "value", lower, 0
        if overflow:
            return "exact", None, 0
        if above_hi > B:
            return "value", float("inf"), 0
        if m < B + 1:
            lo_key = int(np.array([lower], dtype=np.float64).view(np.uint64)[0])
            return ("value", lower, 0) if self.L_key <= lo_key else ("exact", None, 0)
        rank = B - above_hi  # 0-based from the top among the keys in (L, hi]
        above = 0
        for d in range(SHARD_BINS - 1, -1, -1):
            h = int(hist[d])
            if above + h > rank:
                self.digit_count = h
                return "digit", d, rank - above
            above += h
        return "exact", None, 0  # unreachable when the counts add up

    def digit_keys(self, digit: int) -> torch.Tensor:
        """This rank's candidate keys in ``digit`` (int64 bit patterns of p);
        at most the digit's count over all ranks (``decide``)."""
        out = torch.empty(max(1, int(self.digit_count)), dtype=torch.int64, device=self.dev)
        cnt = torch.zeros(1, dtype=torch.int64, device=self.dev)
        self.lib.call("vt_tau_shard_digit_keys", self.n, self.b_r, self.n_global, self.budget, int(digit),
                      self.D.ptr(out), out.numel(), self.D.ptr(cnt), self.D.ptr(self.ws), self.ws.numel(),
                      self.D.stream_ptr())
        c = int(cnt.item())
        if c > out.numel():
            raise RuntimeError("vt_tau_shard_digit_keys: digit holds more keys than the buffer")
        return out[:c]

    @staticmethod
    def finish(all_keys, rank_in_digit: int) -> float:
        """The rank-th largest of the gathered keys (exact), as the FP64 p."""
        k = np.sort(np.asarray(all_keys, dtype=np.int64).view(np.uint64))[::-1]
        return float(k[rank_in_digit:rank_in_digit + 1].view(np.float64)[0])


class BudgetExchange:
    """The sharded budget search's two exchanges over peer memory
    (``vt_tau_shard_search_x``): a symmetric-memory buffer per rank (a plain
    device buffer in a single process) holding every rank's digit histogram
    and digit keys; the decision, the gather, the exact order statistic and
    the bisection run on the device, so a search is one enqueue and one host
    read.  ``keys_cap`` bounds one rank's keys in the selected digit.
    Construction is collective, like ``CountExchange``'s."""

    def __init__(self, group=None, device=None, keys_cap: int = 1 << 16):
        from . import _device as D
        from . import _lib
        self.D, self.lib = D, _lib
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.world = _world(group)
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.keys_cap = int(keys_cap)
        words = int(_lib.lib().vt_tau_shard_exchange_words(self.world, self.keys_cap))
        if dist.is_initialized():
            import torch.distributed._symmetric_memory as symm
            self.buf = symm.empty(words, dtype=torch.int64, device=dev)
            self.buf.zero_()
            name = (group or dist.group.WORLD).group_name
            self.handle = symm.rendezvous(self.buf, name)
            self.peers = int(self.handle.buffer_ptrs_dev)
            torch.cuda.synchronize(dev)
            dist.barrier(group)  # every buffer is zero before any rank publishes
        else:
            self.buf = torch.zeros(words, dtype=torch.int64, device=dev)
            self._ptrs = torch.tensor([self.buf.data_ptr()], dtype=torch.int64, device=dev)
            self.peers = int(self._ptrs.data_ptr())
        self.out = torch.zeros(3, dtype=torch.int64, device=dev)  # [tau bits, status, error bits]

    def search(self, x_local: torch.Tensor, b_r: int, n_global: int, budget: int, iters: int = 30,
               phases: int = 7) -> None:
        """Enqueue the search (all phases by default); ``result`` reads it."""
        D = self.D
        t = D.aligned_f64(x_local.reshape(-1)) if x_local.numel() else x_local.reshape(-1).to(torch.float64)
        n = int(t.numel())
        ws = D.workspace(int(self.lib.lib().vt_tau_shard_search_x_workspace(n)), "tau_shard_x")
        if phases & 1:
            self.out.zero_()
        o = self.out.data_ptr()
        self.lib.call("vt_tau_shard_search_x", D.ptr(t) if n else None, n, int(b_r), int(n_global), int(budget),
                      int(iters), self.peers, self.buf.data_ptr(), self.world, self.rank, self.keys_cap, o, o + 8,
                      o + 16, D.ptr(ws), ws.numel(), int(phases), D.stream_ptr())

    def result(self) -> tuple[int, float]:
        """(status, tau): status 0 = tau decided on the device, 1 = the exact
        multi-pass path must decide.  One host read."""
        v = self.out.cpu()
        err = int(v[2].item()) & 0xFFFFFFFF
        if err & self.lib.ERR_EXCHANGE:
            raise RuntimeError("budget exchange: a peer's data did not arrive (10 s)")
        self.D.raise_fpround(err)
        return int(v[1].item()), float(v[0:1].view(torch.float64).item())


def _bisect_tau(v: float, b_r: int, iters: int) -> float:
    from .fpround import tau_bounds
    lower, upper = tau_bounds(b_r)
    for _ in range(iters):
        tau = (lower + upper) / 2.0
        if v <= tau:
            upper = tau
        else:
            lower = tau
    return upper


def search_tau_budget_sharded(x_local: torch.Tensor, b_r: int, budget: int, iters: int = 30, group=None,
                              exchange: BudgetExchange | None = None, n_global: int | None = None) -> float:
    """protocol.search_tau_budget over a tensor sharded across ranks: the same
    FP64 bisection on the exact global (budget+1)-th largest p, every rank
    getting the same tau.  Candidate path: one read of each shard, an
    all-reduce of a 2051-word exchange buffer and an all-gather of the keys
    in the selected digit (``ShardedBudget``); the exact 5-pass radix select
    (``kth_largest_distance_sharded``) when the candidates cannot decide.
    With ``exchange`` the two exchanges run over peer memory and every step
    after the shard read on the device (one enqueue, one host read); pass
    ``n_global`` to skip the all-reduce of the shard sizes."""
    world = _world(group)
    if n_global is None:
        n = torch.tensor([x_local.numel()], dtype=torch.int64, device=x_local.device)
        if world > 1:
            dist.all_reduce(n, group=group)
        n_global = int(n.item())
    if n_global == 0 or n_global <= budget:
        from .fpround import tau_bounds
        return _bisect_tau(tau_bounds(b_r)[0], b_r, iters)
    if exchange is not None:
        exchange.search(x_local, b_r, n_global, int(budget), iters)
        status, tau = exchange.result()
        if status == 0:
            return tau
        return _bisect_tau(kth_largest_distance_sharded(x_local, b_r, int(budget), group), b_r, iters)
    sb = ShardedBudget(x_local, b_r, n_global, int(budget))
    xb = sb.candidates()
    if world > 1:
        dist.all_reduce(xb, group=group)
    kind, val, rank = sb.decide(xb.cpu().numpy())
    if kind == "value":
        return _bisect_tau(val, b_r, iters)
    if kind == "exact":
        return _bisect_tau(kth_largest_distance_sharded(x_local, b_r, int(budget), group), b_r, iters)
    keys = sb.digit_keys(val)
    if world > 1:
        cnt = all_gather_counts(keys.numel(), group, device=x_local.device)
        width = max(1, int(cnt.max()))
        pad = torch.zeros(width, dtype=torch.int64, device=x_local.device)
        pad[: keys.numel()] = keys
        allk = torch.empty(world * width, dtype=torch.int64, device=x_local.device)
        _all_gather_flat(allk, pad, group)
        keys = torch.cat([allk[r * width: r * width + int(cnt[r])] for r in range(world)])
    return _bisect_tau(ShardedBudget.finish(keys.cpu().numpy(), rank), b_r, iters)


# ---------------------------------------------------------------------------
# Merkle
# ---------------------------------------------------------------------------

def leaf_block_range(n_leaves: int, rank: int, world: int, k: int = BLOCK_LEAVES_LOG2) -> tuple[int, int]:
    """Leaves [lo, hi) of rank: whole 2^k-leaf blocks, contiguous."""
    blocks = (n_leaves + (1 << k) - 1) >> k
    per, extra = divmod(blocks, world)
    b_lo = rank * per + min(rank, extra)
    b_hi = b_lo + per + (1 if rank < extra else 0)
    return min(b_lo << k, n_leaves), min(b_hi << k, n_leaves)


def local_depth(n_leaves_total: int, k: int = BLOCK_LEAVES_LOG2) -> int:
    """Index of the highest level every rank builds locally: k, or the root's
    level when the whole tree fits in one 2^k block (merkle.build stops at one
    node, merkle.py:63-72)."""
    if n_leaves_total <= 1:
        return 0
    return min(k, (n_leaves_total - 1).bit_length())


def local_levels(leaves: torch.Tensor, depth: int, hash_level) -> list[torch.Tensor]:
    """Levels 0..depth over a run of whole 2^k blocks (depth <= k).  A run
    that shrinks to one node before ``depth`` is the global right edge (the
    last, partial block), where merkle.build promotes the node unchanged, so
    the node repeats up to ``depth``; an empty run gives empty levels."""
    levels = [leaves]
    cur = leaves
    for _ in range(depth):
        if cur.shape[0] > 1:
            cur = hash_level(cur)
        levels.append(cur)
    return levels


def combine_top(block_roots: torch.Tensor, hash_level) -> list[torch.Tensor]:
    """Levels above the block roots (built redundantly on every rank)."""
    levels = [block_roots]
    cur = block_roots
    while cur.shape[0] > 1:
        cur = hash_level(cur)
        levels.append(cur)
    return levels


def assemble_levels(per_rank_local: list[list], top: list) -> list:
    """The full ``merkle.build`` level list from every rank's local levels (in
    rank order) and the top levels: global level L <= depth is the rank-order
    concatenation of local level L; top[0] repeats level depth (the block
    roots), so the levels above are top[1:].  Works on lists of 32-byte
    digests or on [m, 32] uint8 tensors."""
    depth = len(per_rank_local[0]) - 1
    out = []
    for L in range(depth + 1):
        parts = [lv[L] for lv in per_rank_local]
        if isinstance(parts[0], torch.Tensor):
            out.append(torch.cat(parts))
        else:
            out.append([d for p in parts for d in p])
    return out + list(top[1:])


def merkle_sharded(w_local_bytes: torch.Tensor, n_leaves_total: int, leaf_bytes: int = 4096,
                   k: int = BLOCK_LEAVES_LOG2, group=None, hash_leaves=None, hash_level=None,
                   exchange: DigestExchange | None = None, check: bool = True):
    """Per-rank lower levels (0..depth) + all-gathered block roots + top levels.

    Returns (local_levels, top_levels).  Every rank returns depth + 1 local
    levels (``local_depth``: k, or fewer when the tree fits one block; empty
    tensors on a rank that owns no leaves).  Global level L <= depth of the
    full tree is the rank-order concatenation of every rank's local level L
    (ranks own whole blocks); top_levels[0] are the block roots (= global
    level depth) and the levels above it follow (``assemble_levels``).
    With ``exchange`` (a ``DigestExchange`` for this tree's block count) the
    block roots travel over peer memory from the kernel that hashes them,
    instead of an NCCL all-gather; ``check`` reads the exchange's error
    word (a host sync) -- pass False in a timed loop and call
    ``exchange.check()`` after it.
    """
    if hash_leaves is None or hash_level is None:
        from . import merkle as mk
        hash_leaves = hash_leaves or (lambda b: mk.sha256_leaves(b, leaf_bytes))
        hash_level = hash_level or _device_level
    world = _world(group)
    depth = local_depth(n_leaves_total, k)
    leaves = hash_leaves(w_local_bytes) if w_local_bytes.numel() else None
    # each rank contributes its block roots; ranks own whole blocks, so the
    # number of roots per rank is known from the plan
    n_blocks = [(hi - lo + (1 << k) - 1) >> k
                for lo, hi in (leaf_block_range(n_leaves_total, r, world, k) for r in range(world))]
    if exchange is not None:
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        if exchange.n_total != sum(n_blocks):
            raise ValueError(f"DigestExchange sized for {exchange.n_total} block roots, the tree has {sum(n_blocks)}")
        dst = sum(n_blocks[:rank])
        if leaves is None or leaves.shape[0] == 0:
            lv = [torch.zeros((0, 32), dtype=torch.uint8, device=w_local_bytes.device) for _ in range(depth + 1)]
            exchange.publish(lv[-1], dst)
        else:  # local_levels, with the level that yields the block roots publishing them
            lv, cur, published = [leaves], leaves, False
            for L in range(depth):
                if cur.shape[0] > 1:
                    if L == depth - 1:
                        cur, published = exchange.publish_level(cur, dst), True
                    else:
                        cur = hash_level(cur)
                lv.append(cur)
            if not published:
                exchange.publish(lv[-1], dst)
        roots = exchange.wait()
        if check:
            exchange.check()
        return lv, combine_top(roots.clone(), hash_level)
    if leaves is None or leaves.shape[0] == 0:
        dev = w_local_bytes.device
        lv = [torch.zeros((0, 32), dtype=torch.uint8, device=dev) for _ in range(depth + 1)]
    else:
        lv = local_levels(leaves, depth, hash_level)
    mine = lv[-1]
    width = max(n_blocks)
    pad = torch.zeros((width, 32), dtype=torch.uint8, device=mine.device)
    pad[: mine.shape[0]] = mine
    gathered = torch.empty((world * width, 32), dtype=torch.uint8, device=mine.device)
    _all_gather_flat(gathered, pad, group)
    roots = torch.cat([gathered[r * width: r * width + n_blocks[r]] for r in range(world)])
    return lv, combine_top(roots, hash_level)


class DigestExchange:
    """The block-root exchange of ``merkle_sharded`` over peer memory, like
    ``CountExchange``: a symmetric-memory buffer per rank (a plain device
    buffer in a single process) sized for ``n_total`` block roots.  The level
    kernel that produces this rank's block roots also stores each of them
    into every rank's buffer at its global block index
    (``vt_merkle_level_exchange``; ``vt_digests_publish`` when the roots need
    no hashing), and ``wait`` gathers all of them in block order
    (``vt_digests_wait``).  No NCCL call, no host round trip.  Construction
    is collective, like ``CountExchange``'s."""

    def __init__(self, n_total: int, group=None, device=None):
        from . import _device as D
        from . import _lib
        self.D, self.lib = D, _lib
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.world = _world(group)
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.n_total = int(n_total)
        words = int(_lib.lib().vt_digest_exchange_words(self.world, self.n_total))
        if dist.is_initialized():
            import torch.distributed._symmetric_memory as symm
            self.buf = symm.empty(words, dtype=torch.int64, device=dev)
            self.buf.zero_()
            name = (group or dist.group.WORLD).group_name
            self.handle = symm.rendezvous(self.buf, name)
            self.peers = int(self.handle.buffer_ptrs_dev)
            torch.cuda.synchronize(dev)
            dist.barrier(group)  # every buffer is zero before any rank publishes
        else:
            self.buf = torch.zeros(words, dtype=torch.int64, device=dev)
            self._ptrs = torch.tensor([self.buf.data_ptr()], dtype=torch.int64, device=dev)
            self.peers = int(self._ptrs.data_ptr())
        self.roots = torch.empty((self.n_total, 32), dtype=torch.uint8, device=dev)
        self.flags = torch.zeros(2, dtype=torch.int32, device=dev)

    def publish_level(self, cur: torch.Tensor, dst: int) -> torch.Tensor:
        """One Merkle level over ``cur`` ([m, 32] digests) whose outputs are
        this rank's block roots [dst, dst + (m+1)//2): hashed and published."""
        m = int(cur.shape[0])
        out = torch.empty(((m + 1) // 2, 32), dtype=torch.uint8, device=cur.device)
        self.lib.call("vt_merkle_level_exchange", self.D.ptr(cur.contiguous()), m, self.D.ptr(out), self.peers,
                      self.world, self.rank, int(dst), self.n_total, self.D.stream_ptr())
        return out

    def publish(self, roots: torch.Tensor, dst: int) -> None:
        """Publish block roots that need no hashing (possibly none)."""
        n = int(roots.shape[0])
        self.lib.call("vt_digests_publish", self.D.ptr(roots.contiguous()) if n else None, n, self.peers,
                      self.world, self.rank, int(dst), self.n_total, self.D.stream_ptr())

    def wait(self) -> torch.Tensor:
        """Every rank's block roots of the latest exchange, [n_total, 32], in
        block order (valid in stream order)."""
        self.lib.call("vt_digests_wait", self.peers, self.world, self.rank, self.n_total,
                      self.D.ptr(self.roots) if self.n_total else None, self.flags.data_ptr(), self.D.stream_ptr())
        return self.roots

    def check(self) -> None:
        if int(self.flags[0].item()) & self.lib.ERR_EXCHANGE:
            raise RuntimeError("block-root exchange: a peer's roots did not arrive (10 s)")


def _device_level(cur: torch.Tensor) -> torch.Tensor:
    from . import _device as D
    from . import _lib
    m = int(cur.shape[0])
    out = torch.empty(((m + 1) // 2, 32), dtype=torch.uint8, device=cur.device)
    _lib.call("vt_merkle_level", D.ptr(cur.contiguous()), m, D.ptr(out), D.stream_ptr())
    return out
