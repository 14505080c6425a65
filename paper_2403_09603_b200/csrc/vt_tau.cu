// Adaptive-threshold support: the "histogram-of-distances reduction".
//
// The budget search (skeleton of protocol.search_tau,
// pkg/src/vtrain/protocol.py:494-506) needs, per tensor, the predicate
// count(p > tau) <= B for 30 bisection midpoints, where
// p = |x - rnd(x)| / max(scale(x), 2^-126) is exact in FP64
// (fpround.py:171-173).  That predicate equals v <= tau for v the (B+1)-th
// largest p, so the device computes v once by an exact MSD radix select on
// the FP64 bit patterns of p (p >= 0, so bit order is numeric order) and the
// host runs the identical FP64 bisection on v.
//
// Passes: digits [62:49] [48:35] [34:21] [20:7] [6:0] of the key; each pass
// is one streaming read of x with a per-CTA shared-memory histogram
// (match_any-aggregated atomics), then a one-CTA select kernel narrows the
// prefix on the device, so no host round trip happens between passes.
#include <algorithm>
#include <cstring>
#include <vector>

#include <cooperative_groups.h>

#include "vt_common.cuh"

namespace vt {
namespace cg = cooperative_groups;

constexpr int kPasses = 5;
__host__ __device__ constexpr int pass_shift(int p) { return p == 0 ? 49 : p == 1 ? 35 : p == 2 ? 21 : p == 3 ? 7 : 0; }
__host__ __device__ constexpr int pass_bits(int p) { return p == 4 ? 7 : 14; }
constexpr int kMaxBins = 1 << 14;
constexpr int kHistThreads = 512;
constexpr int kSelThreads = 1024;

struct SelectState {
  uint64_t prefix;
  uint64_t mask;
  int64_t rank;  // remaining 0-based rank from the top inside the prefix bucket
  int64_t found;
};

// One isolated FP64 (a candidate's x): no L1 allocation, and the smallest
// L2 prefetch size, so each gather costs its own sector rather than a line.
__device__ __forceinline__ double ldg_sector(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

template <int PASS>
__global__ void __launch_bounds__(kHistThreads) tau_hist_kernel(const double* __restrict__ x, int64_t n,
                                                                Grid g, const SelectState* st,
                                                                uint32_t* __restrict__ hist,
                                                                int32_t* errp) {
  extern __shared__ uint32_t sh[];
  constexpr int nbins = 1 << pass_bits(PASS);
  for (int i = threadIdx.x; i < nbins; i += kHistThreads) sh[i] = 0;
  __syncthreads();
  const uint64_t prefix = st->prefix, mask = st->mask;
  uint32_t err = 0;
  const int64_t stride = (int64_t)gridDim.x * kHistThreads;
  const int64_t n_iter = (n + stride - 1) / stride;
  for (int64_t it = 0; it < n_iter; ++it) {
    const int64_t i = it * stride + (int64_t)blockIdx.x * kHistThreads + threadIdx.x;
    bool take = false;
    uint32_t bin = 0;
    if (i < n) {
      const uint64_t key = dist_key(__ldg(x + i), g, err);
      take = (key & mask) == prefix;
      bin = (uint32_t)(key >> pass_shift(PASS)) & (uint32_t)(nbins - 1);
    }
    // aggregate equal bins inside the warp: one shared atomic per distinct bin
    const uint32_t active = __ballot_sync(0xffffffffu, take);
    if (take) {
      const uint32_t peers = __match_any_sync(active, bin);
      if ((threadIdx.x & 31) == (__ffs(peers) - 1)) atomicAdd(&sh[bin], (uint32_t)__popc(peers));
    }
  }
  report_err(errp, err);
  __syncthreads();
  for (int i = threadIdx.x; i < nbins; i += kHistThreads) {
    const uint32_t c = sh[i];
    if (c) atomicAdd(&hist[i], c);
  }
}

template <int PASS>
__global__ void __launch_bounds__(kSelThreads) tau_select_kernel(const uint32_t* __restrict__ hist,
                                                                 SelectState* st, uint64_t* key_out) {
  constexpr int nbins = 1 << pass_bits(PASS);
  constexpr int per = (nbins + kSelThreads - 1) / kSelThreads;
  __shared__ unsigned long long s_warp[kSelThreads / 32];
  const int t = threadIdx.x;
  const int64_t rank = st->rank;
  // thread t owns bins [hi - per, hi) counting from the TOP of the key range
  const int hi = nbins - t * per;
  unsigned long long mine = 0;
  for (int k = 0; k < per; ++k) {
    const int b = hi - 1 - k;
    if (b >= 0) mine += hist[b];
  }
  // exclusive scan over threads (descending bins)
  unsigned long long incl = mine;
  const int lane = t & 31, warp = t >> 5;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long v = s_warp[lane];
    unsigned long long w = v;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long u = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += u;
    }
    s_warp[lane] = w - v;
  }
  __syncthreads();
  const unsigned long long above = s_warp[warp] + incl - mine;
  if ((long long)above <= rank && rank < (long long)(above + mine)) {
    unsigned long long acc = above;
    for (int k = 0; k < per; ++k) {
      const int b = hi - 1 - k;
      if (b < 0) break;
      const unsigned long long c = hist[b];
      if (rank < (long long)(acc + c)) {
        const uint64_t p = st->prefix | ((uint64_t)b << pass_shift(PASS));
        st->prefix = p;
        st->mask |= ((uint64_t)(nbins - 1)) << pass_shift(PASS);
        st->rank = rank - (long long)acc;
        if (PASS == kPasses - 1) {
          *key_out = p;
          st->found = 1;
        }
        break;
      }
      acc += c;
    }
  }
}

__global__ void init_state_kernel(SelectState* st, int64_t rank, uint64_t* key_out) {
  st->prefix = 0;
  st->mask = 0;
  st->rank = rank;
  st->found = 0;
  *key_out = 0;
}

__device__ __forceinline__ unsigned long long order_key(double v) {
  const unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void min_init_kernel(double* out) {
  *reinterpret_cast<unsigned long long*>(out) = order_key(__longlong_as_double(0x7ff0000000000000ll));
}

__global__ void min_kernel(const double* __restrict__ s, int64_t n, double* out, int32_t* nanp) {
  unsigned long long best = ~0ull;
  bool nan = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = s[i];
    if (v != v) nan = true;
    else best = min(best, order_key(v));
  }
  for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best != ~0ull)
    atomicMin(reinterpret_cast<unsigned long long*>(out), best);
  if (__syncthreads_or(nan) && threadIdx.x == 0) atomicOr(reinterpret_cast<int*>(nanp), 1);
}

__global__ void min_final_kernel(double* out) {
  const unsigned long long k = *reinterpret_cast<unsigned long long*>(out);
  const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  *out = __longlong_as_double((long long)b);
}

// ---------------------------------------------------------------------------
// Budget selection (the fast path of the budget search).
//
// The bisection only ever compares v with midpoints strictly inside
// (tau_lo, tau_hi), so v may be clamped: v <= tau_lo -> tau_lo, v > tau_hi ->
// +inf.  Keys inside (tau_lo, tau_hi] are offsets o = key - lo_key - 1 in
// [0, W); they are resolved from the top in 13-bit digits.  Each full
// streaming pass over x histograms the next digit inside the selected
// prefix (spread-out bins: plain shared atomics) and, as soon as the
// selected digit holds at most kCandCap keys, compacts them instead; a
// one-CTA kernel then finishes the selection on the candidates.  Typical
// data needs two passes; a distribution with a hot digit (e.g. many exact
// midpoints) takes one more.  Level selection runs on the device, so no
// host round trip happens until the final key.
// ---------------------------------------------------------------------------

constexpr int kBudBits = 13;
constexpr int kBudBins = 1 << kBudBits;
constexpr int kBudMaxLevels = 5;
constexpr int64_t kCandCap = 1 << 16;

struct BudState {
  uint64_t lo_key, hi_key;
  uint64_t cnt_above;  // keys > hi_key
  uint64_t cand;       // candidates appended
  uint64_t prefix;     // fixed offset bits (under pmask)
  uint64_t pmask;
  int64_t rank;        // remaining 0-based rank from the top inside the prefix
  uint64_t bin_count;  // keys inside the prefix
  int level;           // next digit level to histogram
  int compacting;      // the current pass compacts instead of histogramming
  int status;          // 0 running, 1 done (key written)
  int nlevels;
  int shift[kBudMaxLevels];
  int bits[kBudMaxLevels];
};

// One streaming pass of the budget selection by the calling CTA (256
// threads); `sh` = kBudBins words of shared memory.
__device__ void bud_pass_body(const double* __restrict__ x, int64_t n, const Grid& g, BudState* st,
                              uint32_t* __restrict__ hist, uint64_t* __restrict__ cand, int32_t* errp,
                              uint32_t* sh, int64_t blk, int64_t nblk) {
  __shared__ unsigned long long s_above;
  const int level = st->level;
  const bool compact = st->compacting != 0;
  const bool first = level == 0 && !compact;
  const uint64_t lo = st->lo_key, hi = st->hi_key, prefix = st->prefix, pmask = st->pmask;
  const int sh_lv = compact ? 0 : st->shift[level];
  const uint32_t dmask = compact ? 0u : ((1u << st->bits[level]) - 1u);
  if (!compact) {
    for (int i = threadIdx.x; i < kBudBins; i += 256) sh[i] = 0;
  }
  if (threadIdx.x == 0) s_above = 0;
  __syncthreads();
  uint32_t err = 0, above = 0;
  const int lane = threadIdx.x & 31;
  const bool vec = (reinterpret_cast<uintptr_t>(x) & 31) == 0;
  // fast path valid for b_r = 32 over the default bisection range (2^-25, 2^-24]
  const bool fast32 = g.drop == 29 && lo == 0x3E60000000000000ull && hi == 0x3E70000000000000ull;
  // four consecutive elements per thread per step (one 256-bit load)
  for (int64_t base = blk * 1024; base < n; base += nblk * 1024) {
    const int64_t i0 = base + 4 * threadIdx.x;
    D4 xv;
    if (vec && i0 + 3 < n) {
      xv = ldg_stream4(x + i0);
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v) xv.v[v] = (i0 + v < n) ? x[i0 + v] : 0.0;
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      bool in = false;
      uint64_t k = 0;
      if (i0 + v < n) {
        const double xe = xv.v[v];
        const int hi32 = __double2hiint(xe);
        if (fast32 && !outside_normal32((uint32_t)hi32 & 0x7fffffffu)) {
          // b_r = 32, 2^-126 <= |x| < FLT_MAX: p = d * 2^-52 with d the distance
          // in dropped-bit units (d <= 2^28, so never above tau_hi = 2^-24);
          // inside (2^-25, 2^-24] iff d > 2^27, at key offset (d - 2^27) * 2^25 - 1
          const uint32_t lo32 = (uint32_t)__double2loint(xe);
          const uint32_t low = lo32 & 0x1fffffffu;
          const bool up = (low + ((lo32 >> 29) & 1u)) > 0x10000000u;
          const uint32_t d = up ? (0x20000000u - low) : low;
          const uint64_t o = ((uint64_t)(d - 0x08000000u) << 25) - 1ull;
          in = d > 0x08000000u && (o & pmask) == prefix;
          k = lo + 1ull + o;
        } else {
          k = dist_key(xe, g, err);
          if (k > hi) above += first ? 1u : 0u;
          else in = k > lo && ((k - lo - 1) & pmask) == prefix;
        }
      }
      if (compact) {
        const uint32_t m = __ballot_sync(0xffffffffu, in);
        if (m) {
          const int leader = __ffs(m) - 1;
          unsigned long long pos = 0;
          if (lane == leader)
            pos = atomicAdd(reinterpret_cast<unsigned long long*>(&st->cand), (unsigned long long)__popc(m));
          pos = __shfl_sync(0xffffffffu, pos, leader);
          if (in) {
            const uint64_t slot = pos + __popc(m & ((1u << lane) - 1u));
            if ((int64_t)slot < kCandCap) cand[slot] = k;
          }
        }
      } else if (in) {
        atomicAdd(&sh[(uint32_t)((k - lo - 1) >> sh_lv) & dmask], 1u);
      }
    }
  }
  report_err(errp, err);
  if (first) {
    for (int o = 16; o > 0; o >>= 1) above += __shfl_xor_sync(0xffffffffu, above, o);
    if (lane == 0 && above) atomicAdd(&s_above, (unsigned long long)above);
  }
  __syncthreads();
  if (!compact) {
    for (int i = threadIdx.x; i < kBudBins; i += 256)
      if (sh[i]) atomicAdd(&hist[(size_t)level * kBudBins + i], sh[i]);
  }
  if (first && threadIdx.x == 0 && s_above)
    atomicAdd(reinterpret_cast<unsigned long long*>(&st->cnt_above), s_above);
}

__global__ void __launch_bounds__(256) bud_pass_kernel(const double* __restrict__ x, int64_t n, Grid g,
                                                       BudState* st, uint32_t* __restrict__ hist,
                                                       uint64_t* __restrict__ cand, int32_t* errp) {
  __shared__ uint32_t sh[kBudBins];
  if (st->status != 0) return;
  bud_pass_body(x, n, g, st, hist, cand, errp, sh, blockIdx.x, gridDim.x);
}

// Copy a global histogram into shared memory with batches of independent
// loads (the scan below would otherwise pay one memory round trip per bin).
__device__ void stage_hist(const uint32_t* __restrict__ g, uint32_t* sh, int nbins) {
  const int nthr = blockDim.x;
  for (int i0 = threadIdx.x; i0 < nbins; i0 += 8 * nthr) {
    uint32_t v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = (i0 + k * nthr < nbins) ? g[i0 + k * nthr] : 0u;
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (i0 + k * nthr < nbins) sh[i0 + k * nthr] = v[k];
  }
  __syncthreads();
}

// Pick the digit of the rank-th largest key (descending scan by one CTA of
// up to kSelThreads threads) from a histogram in shared memory.
__device__ void select_digit(const uint32_t* hist, int nbins, int64_t rank, int& bin, int64_t& above_out) {
  __shared__ unsigned long long s_warp[kSelThreads / 32];
  __shared__ int s_bin;
  __shared__ long long s_above;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int nthr = blockDim.x, nwarps = nthr >> 5;
  const int per = (nbins + nthr - 1) / nthr;
  const int hi = nbins - t * per;
  unsigned long long mine = 0;
  for (int k = 0; k < per; ++k) {
    const int b = hi - 1 - k;
    if (b >= 0) mine += hist[b];
  }
  unsigned long long incl = mine;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) s_warp[warp] = incl;
  if (t == 0) s_bin = -1;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long a = lane < nwarps ? s_warp[lane] : 0ull;
    unsigned long long w = a;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long u = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += u;
    }
    if (lane < nwarps) s_warp[lane] = w - a;
  }
  __syncthreads();
  const unsigned long long above = s_warp[warp] + incl - mine;
  if ((long long)above <= rank && rank < (long long)(above + mine)) {
    unsigned long long acc = above;
    for (int k = 0; k < per; ++k) {
      const int b = hi - 1 - k;
      if (b < 0) break;
      const unsigned long long c = hist[b];
      if (rank < (long long)(acc + c)) {
        s_bin = b;
        s_above = (long long)acc;
        break;
      }
      acc += c;
    }
  }
  __syncthreads();
  bin = s_bin;
  above_out = s_above;
}

// After a pass: either finish from the candidates, or select the digit of
// this level and decide whether the next pass compacts or histograms.
__device__ void bud_step_body(BudState* st, const uint32_t* __restrict__ hist, const uint64_t* __restrict__ cand,
                              int64_t budget, uint64_t* key_out, uint32_t* sh) {
  const uint64_t lo1 = st->lo_key + 1;
  if (st->compacting) {  // exact select among the compacted candidates
    const int64_t m = (int64_t)st->cand;
    uint64_t prefix = st->prefix, pmask = st->pmask;
    int64_t rank = st->rank;
    for (int lv = st->level; lv < st->nlevels; ++lv) {
      const int sh_lv = st->shift[lv], bits = st->bits[lv];
      for (int i = threadIdx.x; i < kBudBins; i += blockDim.x) sh[i] = 0;
      __syncthreads();
      for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
        const uint64_t o = cand[i] - lo1;
        if ((o & pmask) == prefix) atomicAdd(&sh[(o >> sh_lv) & ((1u << bits) - 1u)], 1u);
      }
      __syncthreads();
      int bin;
      int64_t above;
      select_digit(sh, 1 << bits, rank, bin, above);
      prefix |= (uint64_t)bin << sh_lv;
      pmask |= ((1ull << bits) - 1ull) << sh_lv;
      rank -= above;
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      *key_out = lo1 + prefix;
      st->status = 1;
    }
    return;
  }
  const int level = st->level;
  int64_t rank = st->rank;
  if (level == 0) {
    const uint64_t above_hi = st->cnt_above;
    if ((int64_t)above_hi > budget) {  // more than budget keys above tau_hi: v > tau_hi
      if (threadIdx.x == 0) {
        *key_out = 0x7ff0000000000000ull;
        st->status = 1;
      }
      return;
    }
    rank = budget - (int64_t)above_hi;
  }
  int bin;
  int64_t above;
  stage_hist(hist + (size_t)level * kBudBins, sh, 1 << st->bits[level]);
  select_digit(sh, 1 << st->bits[level], rank, bin, above);
  if (threadIdx.x == 0) {
    if (bin < 0) {  // fewer than budget+1 keys above tau_lo: v <= tau_lo
      *key_out = st->lo_key;
      st->status = 1;
      return;
    }
    const int sh_lv = st->shift[level];
    st->prefix |= (uint64_t)bin << sh_lv;
    st->pmask |= ((1ull << st->bits[level]) - 1ull) << sh_lv;
    st->rank = rank - above;
    st->bin_count = hist[(size_t)level * kBudBins + bin];
    st->level = level + 1;
    if (level + 1 >= st->nlevels) {  // every offset bit fixed
      *key_out = lo1 + st->prefix;
      st->status = 1;
    } else if ((int64_t)st->bin_count <= kCandCap) {
      st->compacting = 1;
    }
  }
}

__global__ void __launch_bounds__(kSelThreads) bud_step_kernel(BudState* st, const uint32_t* __restrict__ hist,
                                                               const uint64_t* __restrict__ cand, int64_t budget,
                                                               uint64_t* key_out) {
  __shared__ uint32_t sh[kBudBins];
  if (st->status != 0) return;
  bud_step_body(st, hist, cand, budget, key_out, sh);
}

// one thread: fresh selection state for keys in (lo_key, hi_key]
__device__ void bud_init_body(BudState* st, uint64_t lo_key, uint64_t hi_key, uint64_t* key_out) {
  st->lo_key = lo_key;
  st->hi_key = hi_key;
  st->cnt_above = 0;
  st->cand = 0;
  st->prefix = 0;
  st->pmask = 0;
  st->rank = 0;
  st->bin_count = 0;
  st->level = 0;
  st->compacting = 0;
  st->status = 0;
  const uint64_t width = hi_key - lo_key;  // offsets 0 .. width-1
  int top = 64 - __clzll((long long)(width - 1));
  if (width <= 1) top = 1;
  int nl = 0;
  while (top > 0 && nl < kBudMaxLevels) {
    const int b = top < kBudBits ? top : kBudBits;
    top -= b;
    st->shift[nl] = top;
    st->bits[nl] = b;
    ++nl;
  }
  st->nlevels = nl;
  *key_out = 0;
}

__global__ void bud_init_kernel(BudState* st, uint64_t lo_key, uint64_t hi_key, uint64_t* key_out,
                                uint32_t* hist) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kBudMaxLevels * kBudBins; i += gridDim.x * blockDim.x)
    hist[i] = 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) bud_init_body(st, lo_key, hi_key, key_out);
}

}  // namespace vt

using namespace vt;

namespace vt {
__host__ __device__ constexpr size_t tau_ws_bytes() {
  return ((size_t)kPasses * kMaxBins * sizeof(uint32_t) + 256) > (512 + (size_t)kBudMaxLevels * kBudBins * 4 +
                                                                  (size_t)kCandCap * 8)
             ? ((size_t)kPasses * kMaxBins * sizeof(uint32_t) + 256)
             : (512 + (size_t)kBudMaxLevels * kBudBins * 4 + (size_t)kCandCap * 8);
}
}  // namespace vt

extern "C" size_t vt_tau_workspace(int64_t n) {
  (void)n;
  return tau_ws_bytes();
}

extern "C" int vt_tau_budget_key(const double* x, int64_t n, int b_r, int64_t budget, double tau_lo,
                                 double tau_hi, uint64_t* key_out, int32_t* status_out, int32_t* err, void* ws,
                                 size_t ws_bytes, vt_stream_t stream) {
  if (n < 0 || b_r < 10 || b_r > 32 || budget < 0 || !key_out || !status_out || !err || !ws ||
      ws_bytes < vt_tau_workspace(n) || !(tau_lo > 0.0) || !(tau_hi > tau_lo)) {
    vt_set_error("vt_tau_budget_key: bad argument");
    return VT_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* w = static_cast<uint8_t*>(ws);
  BudState* st = reinterpret_cast<BudState*>(w);
  uint32_t* hist = reinterpret_cast<uint32_t*>(w + 512);
  uint64_t* cand = reinterpret_cast<uint64_t*>(w + 512 + (size_t)kBudMaxLevels * kBudBins * 4);
  uint64_t lo_key, hi_key;
  memcpy(&lo_key, &tau_lo, 8);
  memcpy(&hi_key, &tau_hi, 8);
  bud_init_kernel<<<(kBudMaxLevels * kBudBins + 255) / 256, 256, 0, s>>>(st, lo_key, hi_key, key_out, hist);
  int rc = vt_check_launch("bud_init_kernel");
  if (rc) return rc;
  const Grid g = make_grid(b_r, 0.0);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 2047) / 2048, 148 * 8));
  // level passes: at most nlevels histogram passes plus one compaction pass;
  // kernels return at once when the state says done
  for (int p = 0; p <= kBudMaxLevels; ++p) {
    if (n > 0) {
      bud_pass_kernel<<<blocks, 256, 0, s>>>(x, n, g, st, hist, cand, err);
      if ((rc = vt_check_launch("bud_pass_kernel"))) return rc;
    }
    bud_step_kernel<<<1, kSelThreads, 0, s>>>(st, hist, cand, budget, key_out);
    if ((rc = vt_check_launch("bud_step_kernel"))) return rc;
  }
  if (cudaMemcpyAsync(status_out, &st->status, 4, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return vt_check_launch("status copy");
  return VT_OK;
}

namespace vt {
// Straddle samples of protocol.collect_divergence_samples (protocol.py:483-490)
// reduced on the fly: for every element where the two profiles' outputs
// round to different grid points from opposite sides, both normalized
// distances are samples; search_tau only needs their minimum (and whether
// any is NaN), so nothing is materialised.
__global__ void straddle_min_kernel(const double* __restrict__ y1, const double* __restrict__ y2, int64_t n,
                                    Grid g, double* out_min, unsigned long long* count, int32_t* nanp,
                                    int32_t* errp) {
  unsigned long long best = ~0ull;
  uint32_t cnt = 0, err = 0;
  bool nan = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double a = __ldg(y1 + i), b = __ldg(y2 + i);
    const double r1 = __longlong_as_double((long long)round_only(a, g, err));
    const double r2 = __longlong_as_double((long long)round_only(b, g, err));
    const bool straddle = (r1 != r2) && (((a > r1) && (b < r2)) || ((a < r1) && (b > r2)));
    if (straddle) {
      cnt += 2;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const double y = s ? b : a, r = s ? r2 : r1;
        int e = 0;
        (void)frexp(y, &e);
        double scale = (y == 0.0) ? 0x1p-126 : ldexp(1.0, e - 1);
        scale = scale < 0x1p-126 ? 0x1p-126 : scale;
        const double p = __ddiv_rn(fabs(__dsub_rn(y, r)), scale);
        if (p != p) nan = true;
        else best = min(best, (unsigned long long)__double_as_longlong(p) | 0x8000000000000000ull);
      }
    }
  }
  report_err(errp, err);
  for (int o = 16; o > 0; o >>= 1) {
    best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (best != ~0ull) atomicMin(reinterpret_cast<unsigned long long*>(out_min), best);
    if (cnt) atomicAdd(count, (unsigned long long)cnt);
  }
  if (__syncthreads_or(nan) && threadIdx.x == 0) atomicOr(reinterpret_cast<int*>(nanp), 1);
}

// p >= 0 always, so the order key is the bit pattern with the sign bit set
__global__ void straddle_final_kernel(double* out_min) {
  const unsigned long long k = *reinterpret_cast<unsigned long long*>(out_min);
  *out_min = (k == ~0ull) ? __longlong_as_double(0x7ff0000000000000ll)
                          : __longlong_as_double((long long)(k & 0x7fffffffffffffffull));
}

__global__ void straddle_init_kernel(double* out_min, unsigned long long* count) {
  *reinterpret_cast<unsigned long long*>(out_min) = ~0ull;
  *count = 0;
}

// The search_tau skeleton (protocol.py:494-506) in budget form, on one
// thread: identical IEEE FP64 operations to the host loop, so the same tau.
__global__ void budget_bisect_kernel(const uint64_t* key, double lower, double upper, int iters, DevThr* out,
                                     double* tau_out) {
  const double v = __longlong_as_double((long long)*key);
  for (int i = 0; i < iters; ++i) {
    const double tau = __dmul_rn(__dadd_rn(lower, upper), 0.5);
    if (v <= tau) upper = tau;
    else lower = tau;
  }
  *out = thresholds_for(upper);
  *tau_out = upper;
}
}  // namespace vt

extern "C" int vt_straddle_min(const double* y1, const double* y2, int64_t n, int b_r, double* out_min,
                               int64_t* count, int32_t* nan_flag, int32_t* err, vt_stream_t stream) {
  if (n < 0 || b_r < 10 || b_r > 32 || !out_min || !count || !nan_flag || !err || (n && (!y1 || !y2))) {
    vt_set_error("vt_straddle_min: bad argument");
    return VT_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  unsigned long long* c = reinterpret_cast<unsigned long long*>(count);
  straddle_init_kernel<<<1, 1, 0, s>>>(out_min, c);
  if (n) {
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8));
    straddle_min_kernel<<<blocks, 256, 0, s>>>(y1, y2, n, make_grid(b_r, 0.0), out_min, c, nan_flag, err);
  }
  straddle_final_kernel<<<1, 1, 0, s>>>(out_min);
  return vt_check_launch("straddle_min_kernel");
}

namespace vt {
// ---------------------------------------------------------------------------
// One-pass adaptive round-and-log (the budget search of SURVEY.md A.4 without
// extra streaming passes over x in the common case).
//
//   1. rl_fused at a candidate threshold L below the expected tau (about
//      kCandFactor x budget elements have p > L when the dropped mantissa
//      bits are uniform): y (final: rnd does not depend on tau) plus the
//      ascending candidate words (local index << 1 | up);
//   2. the candidates' keys (FP64 bits of p, gathered from x) and the
//      histogram of their top digit above L -> the digit of the
//      (budget+1)-th largest key;
//   3. the keys of that digit, their exact selection and the FP64 bisection
//      (protocol.py:494-506 skeleton) -> tau;
//   4. the log is exactly the candidates with p > tau, in order.
// A single call runs 2-4 as one cooperative launch (adapt_tail_kernel); a
// batch (adapt_*_batch_kernel) gives each tensor a share of three grids.
// If fewer than budget+1 candidates exist (v <= L) or they overflow the
// buffer, the exact selection over x (the multi-pass radix select above,
// fb_selection) and a second rounding pass at the device tau run instead.
// ---------------------------------------------------------------------------

constexpr int kCandFactor = 3;
constexpr int kAdBits = 11;  // digit width of the candidate selection
constexpr int kAdBins = 1 << kAdBits;
constexpr int kAdThreads = 256;
constexpr int kFChunk = 8192;  // candidates per filter ticket
constexpr int kSmallSel = 2048;  // digit keys selected by direct counting (in 16 KB of shared memory)

struct AdaptHdr {
  int32_t fallback;    // 1: the exact path runs (written by the tail / hist kernels every call)
  uint32_t arrived;    // CTAs done (hist, select kernels; reset by the last one)
  int64_t ccount;      // candidates (cursor_out of the rounding pass)
  int64_t scratch;     // the rounding pass's counters[0] (unused)
  uint64_t above;      // keys > hi_key
  int64_t rank;        // remaining rank inside the selected digit
  uint64_t digit;      // selected top digit of (key - L_key - 1)
  uint64_t bin_count;  // keys in that digit
  int32_t done;        // 1: decided at the top digit (v > tau_hi)
  int32_t pad;
  uint64_t cand2;      // keys of the selected digit (compacted)
  uint32_t f_epoch, f_ticket, f_done, f_pad;
  uint64_t above_lo;   // in-place calls: keys > lo_key (decides v <= tau_lo without a fallback)
};

// keys are FP64 bit patterns of p >= 0, so integer order is numeric order
__device__ __forceinline__ bool last_cta(uint32_t* arrived, uint32_t count) {
  __shared__ unsigned s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(arrived, 1u) == count - 1;
  __syncthreads();
  if (s_last) __threadfence();
  return s_last != 0;
}

// A candidate's digit code: 0xfffe below L (never, for keys the rounding
// pass logged), the top digit of key - L - 1 for keys in (L, hi], 0xffff
// above hi.  ad_ord maps codes to the key order: -1, digit, kAdBins.
__device__ __forceinline__ uint16_t ad_code(uint64_t key, uint64_t L_key, uint64_t hi_key, int s0) {
  return key > hi_key ? (uint16_t)0xffffu : key > L_key ? (uint16_t)((key - L_key - 1) >> s0) : (uint16_t)0xfffeu;
}
__device__ __forceinline__ int ad_ord(uint32_t c) { return c == 0xfffeu ? -1 : c == 0xffffu ? kAdBins : (int)c; }

// blk / nblk: this CTA's index among the CTAs working on the tensor (the
// whole grid for a single call, the tensor's share of a batched grid)
__device__ __forceinline__ void adapt_hist_body(const double* __restrict__ x, const Grid& g,
                                                const uint64_t* __restrict__ cw, uint64_t* __restrict__ ck,
                                                uint16_t* __restrict__ cd, int64_t cap, int64_t budget, uint64_t L_key, uint64_t hi_key, int s0,
                                                AdaptHdr* h, uint32_t* __restrict__ hist,
                                                uint64_t* __restrict__ fstatus, int64_t blk,
                                                int64_t nblk) {
  __shared__ uint32_t sh[kAdBins];
  __shared__ unsigned long long s_above;
  const int64_t M = h->ccount;
  if (M > cap || M < budget + 1) {  // v <= L, or too many candidates: the exact path decides
    if (blk == 0 && threadIdx.x == 0) {
      h->fallback = 1;
      h->done = 0;
    }
    return;
  }
  if (blk == 0 && threadIdx.x == 0) h->fallback = 0;
  for (int64_t i = blk * kAdThreads + threadIdx.x; i < (M + kFChunk - 1) / kFChunk;
       i += nblk * kAdThreads)
    fstatus[i] = 0ull;  // the filter's look-back words for this call's chunks
  for (int i = threadIdx.x; i < kAdBins; i += kAdThreads) sh[i] = 0;
  if (threadIdx.x == 0) s_above = 0;
  __syncthreads();
  uint32_t err = 0, above = 0;
  constexpr int kGU = 8;  // independent loads in flight per thread
  const int64_t stride = nblk * kAdThreads;
  for (int64_t i0 = blk * kAdThreads + threadIdx.x; i0 < M; i0 += kGU * stride) {
    uint64_t key[kGU];
    uint64_t w[kGU];
    // the rounding pass staged the candidates' x bits in ck; gather only the
    // rows it could not stage.  The selection and the filter read the 2-byte
    // digit codes and compute a key only where the code cannot decide.
#pragma unroll
    for (int u = 0; u < kGU; ++u) w[u] = (i0 + u * stride < M) ? ck[i0 + u * stride] : 0ull;
#pragma unroll
    for (int u = 0; u < kGU; ++u) {
      // a NaN x equal to the marker is gathered again: the same value
      const double xu = w[u] == kKeyMissing ? ldg_sector(x + (cw[i0 + u * stride] >> 1))
                                             : __longlong_as_double((long long)w[u]);
      key[u] = dist_key(xu, g, err);
      if (i0 + u * stride < M) {
        if (w[u] == kKeyMissing) ck[i0 + u * stride] = (uint64_t)__double_as_longlong(xu);
        cd[i0 + u * stride] = ad_code(key[u], L_key, hi_key, s0);
      }
    }
#pragma unroll
    for (int u = 0; u < kGU; ++u) {
      if (i0 + u * stride >= M) break;
      if (key[u] > hi_key) ++above;
      else if (key[u] > L_key) atomicAdd(&sh[(uint32_t)((key[u] - L_key - 1) >> s0)], 1u);
    }
  }
  for (int o = 16; o > 0; o >>= 1) above += __shfl_xor_sync(0xffffffffu, above, o);
  if ((threadIdx.x & 31) == 0 && above) atomicAdd(&s_above, (unsigned long long)above);
  __syncthreads();
  for (int i = threadIdx.x; i < kAdBins; i += kAdThreads)
    if (sh[i]) atomicAdd(&hist[i], sh[i]);
  if (threadIdx.x == 0 && s_above) atomicAdd(reinterpret_cast<unsigned long long*>(&h->above), s_above);
  if (!last_cta(&h->arrived, (uint32_t)nblk)) return;
  // last CTA: the digit of the (budget+1)-th largest key
  const int64_t above_hi = (int64_t)h->above;
  if (above_hi > budget) {
    if (threadIdx.x == 0) h->done = 1;
  } else {
    int bin;
    int64_t above_bin;
    stage_hist(hist, sh, kAdBins);
    select_digit(sh, kAdBins, budget - above_hi, bin, above_bin);
    if (threadIdx.x == 0) {
      h->done = 0;
      h->digit = (uint64_t)bin;
      h->rank = budget - above_hi - above_bin;
      h->bin_count = hist[bin];
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kAdBins; i += kAdThreads) hist[i] = 0u;  // clean for the next call
  if (threadIdx.x == 0) {
    h->above = 0;
    h->arrived = 0;
  }
}

// One FP64 bisection thread: the search_tau skeleton on the selected key.
__device__ void bisect_to(uint64_t key, double lower, double upper, int iters, DevThr* out, double* tau_out) {
  const double v = __longlong_as_double((long long)key);
  for (int i = 0; i < iters; ++i) {
    const double tau = __dmul_rn(__dadd_rn(lower, upper), 0.5);
    if (v <= tau) upper = tau;
    else lower = tau;
  }
  *out = thresholds_for(upper);
  *tau_out = upper;
}

// The rank-th largest (0-based from the top) of m offsets by direct counting
// in shared memory (sk: m uint64 slots), one CTA: for few keys this beats the
// digit-by-digit histogram selection.  Equal keys give the same answer.
__device__ uint64_t select_by_count(const uint64_t* __restrict__ src, int m, int64_t rank, uint64_t* sk) {
  __shared__ unsigned long long s_pick;
  for (int i = threadIdx.x; i < m; i += blockDim.x) sk[i] = src[i];
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    const uint64_t ki = sk[i];
    int gt = 0, eq = 0;
    for (int j = 0; j < m; ++j) {
      const uint64_t kj = sk[j];
      gt += kj > ki ? 1 : 0;
      eq += kj == ki ? 1 : 0;
    }
    if (gt <= rank && rank < gt + eq) s_pick = ki;
  }
  __syncthreads();
  const uint64_t v = s_pick;
  __syncthreads();
  return v;
}

__device__ __forceinline__ void adapt_select_body(const uint64_t* __restrict__ ck, const uint16_t* __restrict__ cd,
                                                  const Grid& g, uint64_t L_key, uint64_t hi_key,
                                                  int s0, AdaptHdr* h, uint64_t* __restrict__ cand2, double lower,
                                                  double upper, int iters, DevThr* dthr, double* tau_out,
                                                  uint64_t* key_out, int64_t blk, int64_t nblk) {
  __shared__ __align__(16) uint32_t sh[kAdBins];
  if (h->fallback) return;
  if (h->done) {  // 1: more than budget keys above tau_hi (v > tau_hi); 2: v <= tau_lo
    if (blk == 0 && threadIdx.x == 0) {
      const uint64_t v = h->done == 1 ? 0x7ff0000000000000ull : (uint64_t)__double_as_longlong(lower);
      *key_out = v;
      bisect_to(v, lower, upper, iters, dthr, tau_out);
      h->done = 0;
      h->above_lo = 0;
    }
    return;
  }
  const int64_t M = h->ccount;
  const uint64_t digit = h->digit;
  const uint64_t lo1 = L_key + 1;
  const int lane = threadIdx.x & 31;
  constexpr int kSU = 8;  // independent code loads in flight per thread
  const int64_t stride = nblk * kAdThreads;
  for (int64_t i0 = blk * kAdThreads; i0 < M; i0 += kSU * stride) {
    uint32_t code[kSU];
#pragma unroll
    for (int u = 0; u < kSU; ++u) {
      const int64_t i = i0 + u * stride + threadIdx.x;
      code[u] = i < M ? cd[i] : 0xfffeu;
    }
#pragma unroll
    for (int u = 0; u < kSU; ++u) {
      const int64_t i = i0 + u * stride + threadIdx.x;
      const bool in = code[u] == (uint32_t)digit;
      const uint32_t m = __ballot_sync(0xffffffffu, in);
      if (m) {
        uint64_t key = 0;
        if (in) {
          uint32_t e = 0;  // reported by the histogram pass
          key = dist_key(__longlong_as_double((long long)ck[i]), g, e);
        }
        const int leader = __ffs(m) - 1;
        unsigned long long pos = 0;
        if (lane == leader)
          pos = atomicAdd(reinterpret_cast<unsigned long long*>(&h->cand2), (unsigned long long)__popc(m));
        pos = __shfl_sync(0xffffffffu, pos, leader);
        if (in) cand2[pos + __popc(m & ((1u << lane) - 1u))] = key - lo1;
      }
    }
  }
  if (!last_cta(&h->arrived, (uint32_t)nblk)) return;
  // last CTA: exact selection of the rank-th largest among the digit's keys
  const int64_t m = (int64_t)h->cand2;
  int64_t rank = h->rank;
  if (m <= kAdBins / 2) {  // the digit's offsets fit the histogram's shared memory
    const uint64_t off = select_by_count(cand2, (int)m, rank, reinterpret_cast<uint64_t*>(sh));
    if (threadIdx.x == 0) {
      const uint64_t key = lo1 + off;
      *key_out = key;
      bisect_to(key, lower, upper, iters, dthr, tau_out);
      h->cand2 = 0;
      h->arrived = 0;
      h->above_lo = 0;
    }
    return;
  }
  uint64_t low = 0, lmask = 0;
  for (int top = s0; top > 0;) {
    const int bits = top < kAdBits ? top : kAdBits;
    top -= bits;
    for (int i = threadIdx.x; i < kAdBins; i += kAdThreads) sh[i] = 0;
    __syncthreads();
    for (int64_t i = threadIdx.x; i < m; i += kAdThreads) {
      const uint64_t o = cand2[i];
      if ((o & lmask) == low) atomicAdd(&sh[(uint32_t)(o >> top) & ((1u << bits) - 1u)], 1u);
    }
    __syncthreads();
    int bin;
    int64_t above;
    select_digit(sh, 1 << bits, rank, bin, above);
    low |= (uint64_t)bin << top;
    lmask |= ((1ull << bits) - 1ull) << top;
    rank -= above;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const uint64_t key = lo1 + ((digit << s0) | low);
    *key_out = key;
    bisect_to(key, lower, upper, iters, dthr, tau_out);
    h->cand2 = 0;
    h->arrived = 0;
    h->above_lo = 0;
  }
}

// The log: candidates with p > tau, in order.  Persistent CTAs draw chunk
// tickets; each chunk's kept count goes through an epoch-tagged decoupled
// look-back over the chunk status words (the status word format of the
// round-and-log kernel).
constexpr int kLBShift = 44;
constexpr uint64_t kLBEpoch = (1ull << 20) - 1;
constexpr uint64_t kLBA = 1ull << 42, kLBI = 2ull << 42, kLBV = (1ull << 42) - 1;
__device__ __forceinline__ uint64_t lbw(uint32_t e, uint64_t f, uint64_t v) {
  return ((uint64_t)e << kLBShift) | f | (v & kLBV);
}

__device__ __forceinline__ void adapt_filter_body(const uint64_t* __restrict__ cw, const uint64_t* __restrict__ ck,
                                                  const uint16_t* __restrict__ cd, const Grid& g, uint64_t L_key,
                                                  uint64_t hi_key, int s0,
                                                  AdaptHdr* h, const DevThr* dthr, uint64_t* sparse, int64_t cap,
                                                  int64_t global_base, const int64_t* cursor_in, int64_t* cursor_out,
                                                  int64_t* counters, uint64_t* status, int64_t nblk) {
  constexpr int kPer = kFChunk / kAdThreads;  // 32 candidates per thread
  constexpr int kAdWarps = kAdThreads / 32;
  static_assert(kPer == 32, "one keep bit per candidate in a 32-bit mask");
  __shared__ uint32_t s_warp[kAdWarps];
  __shared__ int64_t s_t, s_base;
  __shared__ uint32_t s_epoch;
  if (h->fallback) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t M = h->ccount;
  const int64_t nchunks = (M + kFChunk - 1) / kFChunk;
  const uint64_t tau_key = (uint64_t)__double_as_longlong(dthr->tau);
  const int tau_ord = ad_ord(ad_code(tau_key, L_key, hi_key, s0));
  // keep <=> key > tau: decided by the codes except in tau's own digit
  auto keep_bit = [&](uint32_t c, int64_t i) -> uint32_t {
    const int o = ad_ord(c);
    if (o != tau_ord) return o > tau_ord ? 1u : 0u;
    uint32_t e = 0;
    return dist_key(__longlong_as_double((long long)ck[i]), g, e) > tau_key ? 1u : 0u;
  };
  const int64_t cur = cursor_in ? *cursor_in : 0;
  if (tid == 0) s_epoch = ((*(volatile uint32_t*)&h->f_epoch) + 1u) & (uint32_t)kLBEpoch;
  __syncthreads();
  const uint32_t epoch = s_epoch;
  while (true) {
    if (tid == 0) s_t = (int64_t)atomicAdd(&h->f_ticket, 1u);
    __syncthreads();
    const int64_t t = s_t;
    __syncthreads();
    if (t >= nchunks) break;
    // kPer consecutive candidates per thread (16-byte loads); one look-back
    // per kFChunk candidates
    const int64_t c0 = t * kFChunk + (int64_t)tid * kPer;
    uint32_t keep = 0;
    if (c0 + kPer <= M) {
      uint4 cc[kPer / 8];  // 32 codes, 64 bytes
#pragma unroll
      for (int v = 0; v < kPer / 8; ++v) cc[v] = *reinterpret_cast<const uint4*>(cd + c0 + 8 * v);
#pragma unroll
      for (int v = 0; v < kPer / 2; ++v) {
        const uint4& q = cc[v >> 2];
        const uint32_t pr = (v & 3) == 0 ? q.x : (v & 3) == 1 ? q.y : (v & 3) == 2 ? q.z : q.w;
        keep |= keep_bit(pr & 0xffffu, c0 + 2 * v) << (2 * v);
        keep |= keep_bit(pr >> 16, c0 + 2 * v + 1) << (2 * v + 1);
      }
    } else {
      for (int k = 0; k < kPer && c0 + k < M; ++k) keep |= keep_bit(cd[c0 + k], c0 + k) << k;
    }
    const uint32_t cnt = __popc(keep);
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    if (lane == 31) s_warp[warp] = inc;
    __syncthreads();
    uint32_t wpre = 0, agg = 0;
#pragma unroll
    for (int w = 0; w < kAdWarps; ++w) {
      wpre += (w < warp) ? s_warp[w] : 0u;
      agg += s_warp[w];
    }
    if (warp == 0) {  // publish + look-back (32 predecessors per round trip)
      int64_t excl = 0;
      if (t == 0) {
        if (lane == 0) st_relaxed_u64(status, lbw(epoch, kLBI, agg));
      } else {
        if (lane == 0) st_relaxed_u64(status + t, lbw(epoch, kLBA, agg));
        int64_t pred = t - 1;
        while (true) {
          const int64_t idx = pred - lane;
          uint64_t w = lbw(epoch, kLBI, 0);
          if (idx >= 0) w = ld_relaxed_u64(status + idx);
          const bool valid = ((w >> kLBShift) & kLBEpoch) == epoch;
          const uint64_t flag = valid ? ((w >> 42) & 3ull) : 0ull;
          const uint32_t incm = __ballot_sync(0xffffffffu, flag == 2);
          const uint32_t inv = __ballot_sync(0xffffffffu, flag == 0);
          const int first = incm ? (__ffs(incm) - 1) : 31;
          if (inv & ((2u << first) - 1u)) {
            __nanosleep(32);
            continue;
          }
          uint64_t v = (lane <= first) ? (w & kLBV) : 0ull;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          excl += (int64_t)v;
          if (incm) break;
          pred -= 32;
        }
        if (lane == 0) st_relaxed_u64(status + t, lbw(epoch, kLBI, (uint64_t)excl + agg));
      }
      if (lane == 0) {
        s_base = cur + excl;
        if (t == nchunks - 1) {
          atomicAdd(reinterpret_cast<unsigned long long*>(counters), (unsigned long long)(excl + (int64_t)agg));
          if (cursor_out) *cursor_out = cur + excl + (int64_t)agg;
        }
      }
    }
    __syncthreads();
    int64_t pos = s_base + wpre + (inc - cnt);
    // the kept words: each half's needed 16-byte pairs of cw are requested
    // before its first store (two memory round trips, not one per kept word)
    const bool whole = c0 + kPer <= M;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      ulonglong2 wv[kPer / 4];
#pragma unroll
      for (int v = 0; v < kPer / 4; ++v) {
        const int k = half * (kPer / 2) + 2 * v;
        if ((keep >> k) & 3u)
          wv[v] = whole ? *reinterpret_cast<const ulonglong2*>(cw + c0 + k)
                        : make_ulonglong2(cw[c0 + k], (keep >> (k + 1)) & 1u ? cw[c0 + k + 1] : 0ull);
      }
#pragma unroll
      for (int v = 0; v < kPer / 2; ++v) {
        const int k = half * (kPer / 2) + v;
        if ((keep >> k) & 1u) {
          const uint64_t w = (v & 1) ? wv[v >> 1].y : wv[v >> 1].x;
          if (pos < cap) sparse[pos] = ((uint64_t)(global_base + (int64_t)(w >> 1)) << 1) | (w & 1ull);
          ++pos;
        }
      }
    }
  }
  if (last_cta(&h->f_done, (uint32_t)nblk)) {
    if (tid == 0) {
      h->f_ticket = 0u;
      h->f_done = 0u;
      h->f_epoch = epoch;
      __threadfence();
    }
  }
}

// In-place calls: one streaming read of x appends the keys above L
// (unordered, warp-aggregated); the rounding pass then runs at the selected
// tau and writes the ordered log itself.
__global__ void __launch_bounds__(kAdThreads) adapt_keys_kernel(const double* __restrict__ x, int64_t n, Grid g,
                                                                uint64_t L_key, int64_t thr_L,
                                                                uint64_t* __restrict__ ck, int64_t cap, AdaptHdr* h,
                                                                int32_t* errp) {
  // keys are staged per CTA and appended with one global atomic per flush:
  // a global atomic per warp ballot serialises on the counter's L2 slice
  constexpr int kSteps = 4;                 // x 1024 elements per CTA iteration, loads issued up front
  constexpr int kIter = 1024 * kSteps;
  constexpr int kBuf = kIter + 1024;        // one iteration adds at most kIter
  __shared__ uint64_t sbuf[kBuf];
  __shared__ uint32_t scount;
  __shared__ unsigned long long sbase;
  uint32_t err = 0;
  const int lane = threadIdx.x & 31;
  const bool vec = (reinterpret_cast<uintptr_t>(x) & 31) == 0;
  if (threadIdx.x == 0) scount = 0;
  __syncthreads();
  auto flush = [&]() {
    const uint32_t c = scount;
    if (threadIdx.x == 0) sbase = atomicAdd(reinterpret_cast<unsigned long long*>(&h->ccount), (unsigned long long)c);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < c; i += kAdThreads)
      if ((int64_t)(sbase + i) < cap) ck[sbase + i] = sbuf[i];
    __syncthreads();
    if (threadIdx.x == 0) scount = 0;
    __syncthreads();
  };
  // whole iterations take unguarded 256-bit loads; the ragged tail (or an
  // unaligned x) loads element by element, zero past n
  const int64_t nfull = vec ? (n / kIter) * kIter : 0;
  for (int64_t base = (int64_t)blockIdx.x * kIter; base < n; base += (int64_t)gridDim.x * kIter) {
    D4 xv[kSteps];
    if (base < nfull) {
#pragma unroll
      for (int st = 0; st < kSteps; ++st) xv[st] = ldg_stream4(x + base + st * 1024 + 4 * threadIdx.x);
    } else {
#pragma unroll
      for (int st = 0; st < kSteps; ++st) {
        const int64_t i0 = base + st * 1024 + 4 * threadIdx.x;
#pragma unroll
        for (int v = 0; v < 4; ++v) xv[st].v[v] = (i0 + v < n) ? x[i0 + v] : 0.0;
      }
    }
    constexpr int kE = kSteps * 4;
    {  // general b_r: the test on the 64-bit distance of round_dir (b_r = 32: adapt_keys32_kernel)
      uint32_t cm = 0, slowm = 0;
#pragma unroll
      for (int e = 0; e < kE; ++e) {
        const uint64_t bits = (uint64_t)__double_as_longlong(xv[e >> 2].v[e & 3]);
        const uint64_t mag = bits & kMag;
        const uint64_t low = mag & g.low_mask;
        const uint64_t hb = mag >> g.drop;
        const bool up = (low > g.half) || ((low == g.half) && (hb & 1ull));
        const uint64_t rmag = (hb + (up ? 1ull : 0ull)) << g.drop;
        err |= (mag >= kExpAllOnes) ? (uint32_t)VT_ERR_NONFINITE
                                    : ((rmag > g.gmax_bits) ? (uint32_t)VT_ERR_RANGE : 0u);
        const int64_t d = (int64_t)(up ? (g.one - low) : low);
        cm |= (d > thr_L ? 1u : 0u) << e;
        slowm |= (mag < kNormalMin ? 1u : 0u) << e;
      }
      if (slowm) {
#pragma unroll
        for (int e = 0; e < kE; ++e) {
          if ((slowm >> e) & 1u) {
            const uint64_t key = dist_key(xv[e >> 2].v[e & 3], g, err);
            cm = (cm & ~(1u << e)) | ((key > L_key ? 1u : 0u) << e);
          }
        }
      }
      if (base + kIter > n) {  // the ragged last iteration: drop elements >= n
        uint32_t vm = 0;
#pragma unroll
        for (int e = 0; e < kE; ++e) vm |= (base + (e >> 2) * 1024 + 4 * threadIdx.x + (e & 3) < n ? 1u : 0u) << e;
        cm &= vm;
      }
      // warp-aggregated append of the candidates' x values
      const uint32_t c = __popc(cm);
      uint32_t inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
      if (tot) {
        uint32_t wb = 0;
        if (lane == 31) wb = atomicAdd(&scount, tot);
        uint32_t pos = __shfl_sync(0xffffffffu, wb, 31) + inc - c;
        // the candidate's x itself: the tail kernel turns it into its key
#pragma unroll
        for (int e = 0; e < kE; ++e)
          if ((cm >> e) & 1u) sbuf[pos++] = (uint64_t)__double_as_longlong(xv[e >> 2].v[e & 3]);
      }
    }
    __syncthreads();
    if (scount > (uint32_t)(kBuf - kIter)) flush();
  }
  if (scount) flush();
  report_err(errp, err);
}

// b_r = 32 form of adapt_keys_kernel: per element one shifted unsigned
// compare on the low word (the rl kernel's test, thr < low29 < 2^29 - thr);
// each warp appends its candidates' x values to its own shared-memory run
// (ballot rank, no atomics, no block barriers) and flushes the run with one
// global atomic when it fills.  +-0 (and the zeros loaded past n) have
// low29 = 0 and are never counted; only nonzero values outside the FP32
// normal range take the FP64 key of dist_key (rare path).
__global__ void __launch_bounds__(kAdThreads) adapt_keys32_kernel(const double* __restrict__ x, int64_t n, Grid g,
                                                                  uint64_t L_key, uint32_t c8L, uint32_t w8L,
                                                                  uint64_t* __restrict__ ck, int64_t cap,
                                                                  AdaptHdr* h, int32_t* errp) {
  constexpr int kSteps = 4;  // x 1024 elements per CTA iteration, loads issued up front
  constexpr int kIter = 1024 * kSteps;
  constexpr int kE = kSteps * 4;
  constexpr int kRun = 640;  // entries per warp run; one iteration adds at most 32 * kE = 512
  __shared__ uint64_t sbuf[kAdThreads / 32][kRun];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t* run = sbuf[warp];
  const uint32_t lt = lanemask_lt();
  uint32_t err = 0, cnt = 0;
  auto flush = [&]() {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(reinterpret_cast<unsigned long long*>(&h->ccount), (unsigned long long)cnt);
    base = __shfl_sync(0xffffffffu, base, 0);
    __syncwarp();
    for (uint32_t i = lane; i < cnt; i += 32)
      if ((int64_t)(base + i) < cap) ck[base + i] = run[i];
    __syncwarp();
    cnt = 0;
  };
  const bool vec = (reinterpret_cast<uintptr_t>(x) & 31) == 0;
  const int64_t nfull = vec ? (n / kIter) * kIter : 0;
  // back to front: the in-place rounding pass that follows streams x front to
  // back, so the part of x this pass read last is the part it reads first,
  // while it is still in L2
  const int64_t nit = (n + kIter - 1) / kIter;
  for (int64_t it = nit - 1 - (int64_t)blockIdx.x; it >= 0; it -= (int64_t)gridDim.x) {
    const int64_t base = it * kIter;
    D4 xv[kSteps];
    if (base < nfull) {
#pragma unroll
      for (int st = 0; st < kSteps; ++st) xv[st] = ldg_stream4(x + base + st * 1024 + 4 * threadIdx.x);
    } else {
#pragma unroll
      for (int st = 0; st < kSteps; ++st) {
        const int64_t i0 = base + st * 1024 + 4 * threadIdx.x;
#pragma unroll
        for (int v = 0; v < 4; ++v) xv[st].v[v] = (i0 + v < n) ? x[i0 + v] : 0.0;
      }
    }
    bool badw = false;
#pragma unroll
    for (int e = 0; e < kE; ++e) {
      const uint64_t bits = (uint64_t)__double_as_longlong(xv[e >> 2].v[e & 3]);
      const uint32_t lo32 = (uint32_t)bits, ahi = (uint32_t)(bits >> 32) & 0x7fffffffu;
      // outside the FP32 normal range: never a fast candidate; the FP64 key
      // path decides it unless ahi == 0 (+-0 and FP64 subnormals: p ~ 0)
      const bool o = outside_normal32(ahi);
      const bool in = ((lo32 << 3) - c8L) < w8L && !o;
      badw |= o && ahi != 0u;
      const uint32_t m = __ballot_sync(0xffffffffu, in);
      if (m) {
        if (in) run[cnt + __popc(m & lt)] = bits;
        cnt += __popc(m);
      }
    }
    if (__any_sync(0xffffffffu, badw)) {
#pragma unroll
      for (int e = 0; e < kE; ++e) {
        const double xe = xv[e >> 2].v[e & 3];
        const uint64_t bits = (uint64_t)__double_as_longlong(xe);
        const uint32_t ahi = (uint32_t)(bits >> 32) & 0x7fffffffu;
        bool in = false;
        if (outside_normal32(ahi) && ahi != 0u) in = dist_key(xe, g, err) > L_key;
        const uint32_t m = __ballot_sync(0xffffffffu, in);
        if (m) {
          if (in) run[cnt + __popc(m & lt)] = bits;
          cnt += __popc(m);
        }
      }
    }
    if (cnt > (uint32_t)(kRun - 32 * kE)) flush();
  }
  if (cnt) flush();
  report_err(errp, err);
}

// Exact fallback, gated on h->fallback: the multi-pass budget selection over
// x as ONE cooperative launch (grid-wide syncs between a pass and the
// selection step after it; the final step runs the FP64 bisection).  In the
// common case the whole grid returns at once: one near-empty launch per call
// instead of seven.
__device__ void fb_selection(const double* __restrict__ x, int64_t n, const Grid& g, AdaptHdr* h, BudState* st,
                             uint32_t* hist, uint64_t* cand, int64_t budget, uint64_t lo_key, uint64_t hi_key,
                             double lower, double upper, int iters, uint64_t* key_out, DevThr* dthr,
                             double* tau_out, int32_t* errp, uint32_t* sh) {
  cg::grid_group grid = cg::this_grid();
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = gtid; i < (int64_t)kBudMaxLevels * kBudBins; i += (int64_t)gridDim.x * blockDim.x) hist[i] = 0u;
  if (gtid == 0) {
    bud_init_body(st, lo_key, hi_key, key_out);
    h->above_lo = 0;
  }
  grid.sync();
  for (int p = 0; p <= kBudMaxLevels; ++p) {
    if (*(volatile int*)&st->status != 0) break;  // grid-uniform: read after a grid sync
    bud_pass_body(x, n, g, st, hist, cand, errp, sh, blockIdx.x, gridDim.x);
    grid.sync();
    if (blockIdx.x == 0) {
      bud_step_body(st, hist, cand, budget, key_out, sh);
      __syncthreads();
      if (threadIdx.x == 0 && st->status != 0) bisect_to(*key_out, lower, upper, iters, dthr, tau_out);
    }
    grid.sync();
  }
}

// ---------------------------------------------------------------------------
// The single-call tail as ONE cooperative launch (grid-wide syncs between
// phases instead of kernel boundaries and last-CTA hand-offs):
//   0. can the candidates decide?  (else: in-place "v <= tau_lo", or the
//      exact multi-pass fallback, fb_selection, in this same launch)
//   1. every candidate's key (gathered from x, or from the x value the
//      in-place key pass staged) and the top-digit histogram above L
//   2. every CTA selects the digit of the (budget+1)-th largest key from the
//      global histogram; the keys of that digit are compacted
//   3. CTA 0: exact selection among them and the FP64 bisection -> tau
//   4. out of place: the log = candidates with key > tau, in order (per-CTA
//      contiguous ranges, counts exchanged through a grid sync)
// ---------------------------------------------------------------------------
struct TailArgs {
  const double* x;
  Grid g0;
  const uint64_t* cw;
  uint64_t* ck;
  uint64_t* c2;
  uint32_t* ahist;
  AdaptHdr* h;
  int64_t cap, budget, n;
  uint64_t L_key, lo_key, hi_key;
  int s0, iters;
  double lower, upper;
  DevThr* dthr;
  double* tau_out;
  uint64_t* key;
  BudState* st;
  uint32_t* bhist;
  uint64_t* bcand;
  int32_t* err;
  // out of place: the ordered filter into the log (sparse == nullptr: in place)
  uint64_t* sparse;
  int64_t sparse_cap, global_base;
  const int64_t* cursor_in;
  int64_t* cursor_out;
  int64_t* counters;
};

__device__ __forceinline__ unsigned long long block_sum(unsigned long long v, unsigned long long* s_acc) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (threadIdx.x == 0) *s_acc = 0;
  __syncthreads();
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(s_acc, v);
  __syncthreads();
  return *s_acc;
}

// Phases of the tail for one tensor, run by its nblk CTAs (blk = this CTA's
// index among them): the whole grid for a single call, the tensor's share of
// the grid in a batch.  Grid-wide syncs separate the phases.
struct TailSel {
  int bin;
  int64_t rank;
  bool past_hi;  // more than budget keys above tau_hi: v > tau_hi
};

// 1. every candidate's key (gathered from x, or the x value the in-place key
// pass staged) and the histogram of its top digit above L
__device__ void tail_hist(const TailArgs& a, int64_t M, int64_t blk, int64_t nblk, uint32_t* sh,
                          unsigned long long* s_acc, uint32_t& err) {
  const int tid = threadIdx.x;
  const bool gather = a.sparse != nullptr;
  for (int i = tid; i < kAdBins; i += kAdThreads) sh[i] = 0;
  __syncthreads();
  unsigned long long above = 0;
  constexpr int kGU = 8;
  const int64_t stride = nblk * kAdThreads;
  for (int64_t i0 = blk * kAdThreads + tid; i0 < M; i0 += kGU * stride) {
    // ck holds each candidate's x: from the key pass (in place) or staged by
    // the rounding pass (out of place), which marks the rows it could not
    // stage -- those are gathered from x (a NaN equal to the marker too: the
    // same value)
    double xv[kGU];
#pragma unroll
    for (int u = 0; u < kGU; ++u)
      xv[u] = (i0 + u * stride < M) ? __longlong_as_double((long long)a.ck[i0 + u * stride]) : 0.0;
    if (gather) {
#pragma unroll
      for (int u = 0; u < kGU; ++u)
        if (i0 + u * stride < M && __double_as_longlong(xv[u]) == (long long)kKeyMissing)
          xv[u] = ldg_sector(a.x + (a.cw[i0 + u * stride] >> 1));
    }
#pragma unroll
    for (int u = 0; u < kGU; ++u) {
      if (i0 + u * stride >= M) break;
      const uint64_t key = dist_key(xv[u], a.g0, err);
      a.ck[i0 + u * stride] = key;
      if (key > a.hi_key) ++above;
      else if (key > a.L_key) atomicAdd(&sh[(uint32_t)((key - a.L_key - 1) >> a.s0)], 1u);
    }
  }
  above = block_sum(above, s_acc);
  for (int i = tid; i < kAdBins; i += kAdThreads)
    if (sh[i]) atomicAdd(&a.ahist[i], sh[i]);
  if (tid == 0 && above) atomicAdd(reinterpret_cast<unsigned long long*>(&a.h->above), above);
}

// 2. the digit of the (budget+1)-th largest key (every CTA of the tensor
// computes the same one from the global histogram), then its keys compacted
__device__ TailSel tail_digit(const TailArgs& a, int64_t M, int64_t blk, int64_t nblk, uint32_t* sh) {
  TailSel t{0, 0, false};
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t above_hi = (int64_t)a.h->above;
  t.past_hi = above_hi > a.budget;
  if (t.past_hi) return t;
  int64_t above_bin;
  stage_hist(a.ahist, sh, kAdBins);
  select_digit(sh, kAdBins, a.budget - above_hi, t.bin, above_bin);
  t.rank = a.budget - above_hi - above_bin;
  const uint64_t digit = (uint64_t)t.bin, lo1 = a.L_key + 1;
  const int64_t stride = nblk * kAdThreads;
  constexpr int kDU = 8;  // keys in flight per thread (each round of the loop is one memory latency)
  for (int64_t i0 = blk * kAdThreads; i0 < M; i0 += kDU * stride) {  // warp-uniform bounds: ballots follow
    uint64_t key[kDU];
#pragma unroll
    for (int u = 0; u < kDU; ++u) {
      const int64_t i = i0 + u * stride + tid;
      key[u] = i < M ? a.ck[i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kDU; ++u) {
      const int64_t i = i0 + u * stride + tid;
      const bool in = i < M && key[u] <= a.hi_key && key[u] >= lo1 && ((key[u] - lo1) >> a.s0) == digit;
      const uint32_t m = __ballot_sync(0xffffffffu, in);
      if (m) {
        const int leader = __ffs(m) - 1;
        unsigned long long pos = 0;
        if (lane == leader)
          pos = atomicAdd(reinterpret_cast<unsigned long long*>(&a.h->cand2), (unsigned long long)__popc(m));
        pos = __shfl_sync(0xffffffffu, pos, leader);
        if (in) a.c2[pos + __popc(m & lanemask_lt())] = key[u] - lo1;
      }
    }
  }
  return t;
}

// 3. one CTA: exact selection among the digit's keys and the FP64 bisection;
// the tensor's state is left clean for its next call
__device__ void tail_exact(const TailArgs& a, const TailSel& t, uint32_t* sh) {
  const int tid = threadIdx.x;
  AdaptHdr* h = a.h;
  const uint64_t lo1 = a.L_key + 1;
  uint64_t key = 0x7ff0000000000000ull;
  if (!t.past_hi && (int64_t)h->cand2 <= kSmallSel) {
    // few keys in the digit: direct counting (the offsets carry the digit bits)
    key = lo1 + select_by_count(a.c2, (int)h->cand2, t.rank, reinterpret_cast<uint64_t*>(sh));
  } else if (!t.past_hi) {
    const int64_t m = (int64_t)h->cand2;
    int64_t rank = t.rank;
    uint64_t low = 0, lmask = 0;
    for (int top = a.s0; top > 0;) {
      const int bits = top < kAdBits ? top : kAdBits;
      top -= bits;
      for (int i = tid; i < kAdBins; i += kAdThreads) sh[i] = 0;
      __syncthreads();
      for (int64_t i = tid; i < m; i += kAdThreads) {
        const uint64_t o = a.c2[i];
        if ((o & lmask) == low) atomicAdd(&sh[(uint32_t)(o >> top) & ((1u << bits) - 1u)], 1u);
      }
      __syncthreads();
      int b2;
      int64_t ab2;
      select_digit(sh, 1 << bits, rank, b2, ab2);
      low |= (uint64_t)b2 << top;
      lmask |= ((1ull << bits) - 1ull) << top;
      rank -= ab2;
      __syncthreads();
    }
    key = lo1 + (((uint64_t)t.bin << a.s0) | low);
  }
  if (tid == 0) {
    *a.key = key;
    bisect_to(key, a.lower, a.upper, a.iters, a.dthr, a.tau_out);
    h->above = 0;
    h->cand2 = 0;
    h->above_lo = 0;
    h->fallback = 0;
  }
}

#ifndef VT_TAIL_GRID_EXACT
#define VT_TAIL_GRID_EXACT 1
#endif
#ifndef VT_GRID_SEL_MIN  // digit keys up to this many: block 0 alone (select_by_count), no grid-wide hand-off
#define VT_GRID_SEL_MIN 192
#endif
// 3'. the same selection over the whole grid when the digit holds few keys
// (the common case): one warp per key counts, across its lanes, how many of
// the m keys are larger / equal; the warp holding the (rank)-th largest
// writes it and runs the bisection (equal keys write the same values).  One
// CTA doing the m^2 / 256 comparisons alone took 22 us for m = 516 (2^26
// N(0,1)); the last CTA out resets the tensor's state.
__device__ void tail_exact_grid(const TailArgs& a, const TailSel& t, uint32_t* sh, int64_t blk, int64_t nblk) {
  AdaptHdr* h = a.h;
  const int64_t m = (int64_t)h->cand2;
  if (t.past_hi || m > kSmallSel || m <= VT_GRID_SEL_MIN) {  // few keys: one CTA counts them faster
    if (blk == 0) tail_exact(a, t, sh);
    return;
  }
  const uint64_t lo1 = a.L_key + 1;
  const int lane = threadIdx.x & 31;
  const int64_t warps = nblk * (kAdThreads / 32);
  for (int64_t i = (blk * kAdThreads + threadIdx.x) >> 5; i < m; i += warps) {
    const uint64_t ki = a.c2[i];
    uint32_t gt = 0, eq = 0;
#pragma unroll 4
    for (int64_t j = lane; j < m; j += 32) {
      const uint64_t kj = a.c2[j];
      gt += kj > ki ? 1u : 0u;
      eq += kj == ki ? 1u : 0u;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      gt += __shfl_xor_sync(0xffffffffu, gt, o);
      eq += __shfl_xor_sync(0xffffffffu, eq, o);
    }
    if (lane == 0 && (int64_t)gt <= t.rank && t.rank < (int64_t)(gt + eq)) {
      *a.key = lo1 + ki;
      bisect_to(lo1 + ki, a.lower, a.upper, a.iters, a.dthr, a.tau_out);
    }
  }
  if (last_cta(&h->arrived, (uint32_t)nblk) && threadIdx.x == 0) {  // every CTA has read cand2
    h->arrived = 0;
    h->above = 0;
    h->cand2 = 0;
    h->above_lo = 0;
    h->fallback = 0;
  }
}

// 4a. per-CTA count of the candidates with key > tau in its contiguous range
__device__ void tail_filter_count(const TailArgs& a, int64_t M, int64_t blk, int64_t nblk,
                                  unsigned long long* s_acc) {
  const uint64_t tau_key = (uint64_t)__double_as_longlong(a.dthr->tau);
  const int64_t per = ((M + nblk - 1) / nblk + kAdThreads - 1) / kAdThreads * kAdThreads;
  const int64_t r0 = blk * per, r1 = r0 + per < M ? r0 + per : M;
  unsigned long long cnt = 0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kAdThreads) cnt += a.ck[i] > tau_key ? 1u : 0u;
  cnt = block_sum(cnt, s_acc);
  if (threadIdx.x == 0) a.c2[blk] = cnt;  // the digit keys are done with: per-CTA counts
}

// 4b. the log words of that range at the prefix of the earlier CTAs' counts
#ifndef VT_FILTER_RUNS  // A/B: 8 contiguous candidates per thread per round (else one per thread)
#define VT_FILTER_RUNS 1
#endif

__device__ void tail_filter_write(const TailArgs& a, int64_t M, int64_t blk, int64_t nblk,
                                  unsigned long long* s_acc, uint32_t* s_warp) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t tau_key = (uint64_t)__double_as_longlong(a.dthr->tau);
  const int64_t per = ((M + nblk - 1) / nblk + kAdThreads - 1) / kAdThreads * kAdThreads;
  const int64_t r0 = blk * per, r1 = r0 + per < M ? r0 + per : M;
  unsigned long long pre = 0;
  for (int64_t b = tid; b < blk; b += kAdThreads) pre += a.c2[b];
  pre = block_sum(pre, s_acc);
  const int64_t cur = a.cursor_in ? *a.cursor_in : 0;
  int64_t pos = cur + (int64_t)pre;
  if (VT_FILTER_RUNS) {
    // each thread a run of 8 consecutive candidates per round (all loads of a
    // round in flight at once), one CTA-wide exclusive scan of the run counts
    constexpr int kRun = 8;
    for (int64_t c0 = r0; c0 < r1; c0 += (int64_t)kRun * kAdThreads) {
      const int64_t i0 = c0 + (int64_t)tid * kRun;
      uint64_t k[kRun];
#pragma unroll
      for (int u = 0; u < kRun; ++u) k[u] = (i0 + u < r1) ? a.ck[i0 + u] : 0ull;
      uint32_t keep = 0;
#pragma unroll
      for (int u = 0; u < kRun; ++u) keep |= (i0 + u < r1 && k[u] > tau_key) ? (1u << u) : 0u;
      const uint32_t cnt = __popc(keep);
      uint32_t inc = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += v;
      }
      if (lane == 31) s_warp[warp] = inc;
      __syncthreads();
      uint32_t wpre = 0, tot = 0;
#pragma unroll
      for (int w = 0; w < kAdThreads / 32; ++w) {
        wpre += w < warp ? s_warp[w] : 0u;
        tot += s_warp[w];
      }
      int64_t p = pos + wpre + (inc - cnt);
#pragma unroll
      for (int u = 0; u < kRun; ++u) {
        if (keep & (1u << u)) {
          const uint64_t w = a.cw[i0 + u];
          if (p < a.sparse_cap) a.sparse[p] = ((uint64_t)(a.global_base + (int64_t)(w >> 1)) << 1) | (w & 1ull);
          ++p;
        }
      }
      pos += tot;
      __syncthreads();
    }
  } else {
    for (int64_t c0 = r0; c0 < r1; c0 += kAdThreads) {
      const int64_t i = c0 + tid;
      const bool keep = i < r1 && a.ck[i] > tau_key;
      const uint32_t m = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) s_warp[warp] = __popc(m);
      __syncthreads();
      uint32_t wpre = 0, tot = 0;
#pragma unroll
      for (int w = 0; w < kAdThreads / 32; ++w) {
        wpre += w < warp ? s_warp[w] : 0u;
        tot += s_warp[w];
      }
      if (keep) {
        const int64_t p = pos + wpre + __popc(m & lanemask_lt());
        const uint64_t w = a.cw[i];
        if (p < a.sparse_cap) a.sparse[p] = ((uint64_t)(a.global_base + (int64_t)(w >> 1)) << 1) | (w & 1ull);
      }
      pos += tot;
      __syncthreads();
    }
  }
  if (blk == nblk - 1 && tid == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(a.counters), (unsigned long long)(pos - cur));
    if (a.cursor_out) *a.cursor_out = pos;
  }
}

#ifdef VT_TIMELINE  // development builds only: per-CTA phase stamps of adapt_tail_kernel
__device__ uint64_t g_tl_tail[1024][8];
__device__ __forceinline__ void tail_mark(int i) {
  if (threadIdx.x == 0 && blockIdx.x < 1024) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tl_tail[blockIdx.x][i] = t;
  }
}
extern "C" int vt_debug_timeline_tail(uint64_t* host) {
  return (int)cudaMemcpyFromSymbol(host, g_tl_tail, sizeof(g_tl_tail));
}
#define TTL(i) tail_mark(i)
__device__ __forceinline__ void g_tl_tail_cand2(uint64_t v) { g_tl_tail[1023][0] = v; }
#else
#define TTL(i)
#define g_tl_tail_cand2(v)
#endif

__global__ void __launch_bounds__(kAdThreads) adapt_tail_kernel(const TailArgs a) {
  __shared__ __align__(16) uint32_t sh[kBudBins];
  __shared__ unsigned long long s_acc;
  __shared__ uint32_t s_warp[kAdThreads / 32];
  cg::grid_group grid = cg::this_grid();
  AdaptHdr* h = a.h;
  const int tid = threadIdx.x;
  const int64_t blk = blockIdx.x, nblk = gridDim.x;
  const bool gather = a.sparse != nullptr;
  const int64_t M = h->ccount;
  const int64_t budget = a.budget;
  // 0. grid-uniform decision (every CTA reads the same words)
  if (M > a.cap || M < budget + 1) {
    if (!gather && M <= a.cap) {
      // in place, too few candidates: count the keys above tau_lo (one pass
      // over x, which the rounding pass has not overwritten yet)
      uint32_t e2 = 0;
      unsigned long long c = 0;
      const int64_t n4 = a.n / 4 * 4;
      for (int64_t i = (blk * kAdThreads + tid) * 4; i < a.n; i += nblk * kAdThreads * 4) {
        if (i < n4) {
          const D4 xv = ldg_stream4(a.x + i);
#pragma unroll
          for (int v = 0; v < 4; ++v) c += dist_key(xv.v[v], a.g0, e2) > a.lo_key ? 1u : 0u;
        } else {
          for (int64_t j = i; j < a.n; ++j) c += dist_key(a.x[j], a.g0, e2) > a.lo_key ? 1u : 0u;
        }
      }
      c = block_sum(c, &s_acc);
      if (tid == 0 && c) atomicAdd(reinterpret_cast<unsigned long long*>(&h->above_lo), c);
      grid.sync();
    }
    const bool low = !gather && M <= a.cap && (int64_t)h->above_lo <= budget;
    grid.sync();  // every CTA has read above_lo (and the candidate count)
    if (blk == 0 && tid == 0) h->ccount = 0;  // the next in-place key pass appends from 0
    if (low) {  // at most budget keys above tau_lo: v <= tau_lo fixes the bisection
      if (blk == 0 && tid == 0) {
        h->fallback = 0;
        h->above_lo = 0;
        *a.key = a.lo_key;
        bisect_to(a.lo_key, a.lower, a.upper, a.iters, a.dthr, a.tau_out);
      }
      return;
    }
    if (blk == 0 && tid == 0) h->fallback = 1;
    fb_selection(a.x, a.n, a.g0, h, a.st, a.bhist, a.bcand, budget, a.lo_key, a.hi_key, a.lower, a.upper, a.iters,
                 a.key, a.dthr, a.tau_out, a.err, sh);
    return;
  }
  uint32_t err = 0;
  TTL(0);
  tail_hist(a, M, blk, nblk, sh, &s_acc, err);
  TTL(1);
  grid.sync();
  TTL(2);
  if (blk == 0 && tid == 0) h->ccount = 0;  // read by every CTA at entry; the next in-place key pass appends from 0
  const TailSel t = tail_digit(a, M, blk, nblk, sh);
  TTL(3);
  grid.sync();
  TTL(4);
  // every CTA clears its share of the histogram (all read it before the sync)
  for (int64_t i = blk * kAdThreads + tid; i < kAdBins; i += nblk * kAdThreads) a.ahist[i] = 0u;
  if (blk == 0 && tid == 0) g_tl_tail_cand2(a.h->cand2);
#if VT_TAIL_GRID_EXACT
  tail_exact_grid(a, t, sh, blk, nblk);
#else
  if (blk == 0) tail_exact(a, t, sh);
#endif
  TTL(5);
  report_err(a.err, err);
  if (!gather) return;
  grid.sync();
  tail_filter_count(a, M, blk, nblk, &s_acc);
  grid.sync();
  tail_filter_write(a, M, blk, nblk, &s_acc, s_warp);
}

// Cooperative grid for the fallback kernels: every CTA co-resident.
template <typename K>
int coop_grid(K kernel) {
  static int grid = 0;
  if (!grid) {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, kAdThreads, 0);
    grid = std::max(1, std::min(per, 2) * sms);
  }
  return grid;
}
}  // namespace vt

namespace vt {
// Adaptive workspace: [header 256 B: DevThr, key, status, AdaptHdr]
// [candidate digit histogram] [tau workspace (exact fallback)] [round-and-log
// workspace] [filter status] [candidate words | keys | digit keys: cap each].
// Everything that outlives a call (the headers, the self-cleaning histogram,
// the round-and-log epoch header) sits at offsets independent of n, because
// one workspace serves calls of any size; the filter status words are
// cleared by the batched histogram kernel for the chunks a call uses.
struct AdaptLayout {
  size_t tau, rl, hist, cw, ck, c2, cd, fst, total;
  int64_t cap;
};
__host__ __device__ inline size_t al256(size_t v) { return (v + 255) & ~(size_t)255; }
// rl_bytes: the tensor's own round-and-log workspace (0 in a batch, whose
// rounding passes share one)
__host__ __device__ inline AdaptLayout adapt_layout_rl(int64_t n, size_t rl_bytes) {
  AdaptLayout L;
  L.cap = (n + 15) / 16 > 8192 ? (n + 15) / 16 : 8192;
  size_t o = 256;
  L.hist = o;
  o += al256((size_t)kAdBins * 4);
  L.tau = o;
  o += al256(tau_ws_bytes());
  L.rl = o;
  o += al256(rl_bytes);
  L.fst = o;
  o += al256((size_t)((L.cap + kFChunk - 1) / kFChunk) * 8);
  L.cw = o;
  o += al256((size_t)L.cap * 8);
  L.ck = o;
  o += al256((size_t)L.cap * 8);
  L.c2 = o;
  o += al256((size_t)L.cap * 8);
  L.cd = o;
  o += al256((size_t)L.cap * 2);
  L.total = o;
  return L;
}

struct AdPtrs {
  DevThr* dthr;
  uint64_t* key;
  AdaptHdr* h;
  BudState* st;
  uint32_t *bhist, *ahist;
  uint64_t *bcand, *cw, *ck, *c2, *fst;
  uint16_t* cd;  // batched calls: each candidate's digit code (ad_code)
  int64_t cap;
};

__host__ __device__ inline AdPtrs adapt_ptrs(uint8_t* w, const AdaptLayout& lay) {
  AdPtrs p;
  p.dthr = reinterpret_cast<DevThr*>(w);
  p.key = reinterpret_cast<uint64_t*>(w + 64);
  p.h = reinterpret_cast<AdaptHdr*>(w + 128);
  uint8_t* tws = w + lay.tau;
  p.st = reinterpret_cast<BudState*>(tws);
  p.bhist = reinterpret_cast<uint32_t*>(tws + 512);
  p.bcand = reinterpret_cast<uint64_t*>(tws + 512 + (size_t)kBudMaxLevels * kBudBins * 4);
  p.ahist = reinterpret_cast<uint32_t*>(w + lay.hist);
  p.cw = reinterpret_cast<uint64_t*>(w + lay.cw);
  p.ck = reinterpret_cast<uint64_t*>(w + lay.ck);
  p.c2 = reinterpret_cast<uint64_t*>(w + lay.c2);
  p.cd = reinterpret_cast<uint16_t*>(w + lay.cd);
  p.fst = reinterpret_cast<uint64_t*>(w + lay.fst);
  p.cap = lay.cap;
  return p;
}

}  // namespace vt

namespace {
AdaptLayout adapt_layout(int64_t n) { return adapt_layout_rl(n, vt_round_log_workspace(n)); }
}  // namespace

extern "C" size_t vt_round_log_adaptive_workspace(int64_t n) { return adapt_layout(n).total; }

namespace vt {
// The candidate plan of one adaptive call: threshold L below the expected
// tau (about kCandFactor x (budget + 1) elements above it when p is uniform
// on [0, hi], as the dropped bits of real data are) and the top-digit shift
// of the key offsets above L.
struct AdPlan {
  double lo, hi, L, want;
  uint64_t lo_key, hi_key, L_key;
  int s0, thrL;
  Grid gL, g0;
};

AdPlan adapt_plan(int64_t n, int b_r, int64_t budget) {
  AdPlan P;
  P.lo = 0x1p-25;
  P.hi = ldexp(1.0, 8 - b_r);
  memcpy(&P.lo_key, &P.lo, 8);
  memcpy(&P.hi_key, &P.hi, 8);
  P.want = (double)kCandFactor * (double)(budget + 1) + 1024.0;
  P.L = P.hi * (1.0 - P.want / (double)n);
  if (!(P.L > P.lo)) P.L = P.lo;
  memcpy(&P.L_key, &P.L, 8);
  const uint64_t W = P.hi_key - P.L_key;  // key offsets 0 .. W - 1 above L
  const int wbits = W > 1 ? 64 - __builtin_clzll(W - 1) : 1;
  P.s0 = std::max(0, wbits - kAdBits);
  P.gL = make_grid(b_r, P.L);
  P.thrL = (int)std::min<int64_t>(std::max<int64_t>(P.gL.thr, 0), INT32_MAX);
  P.g0 = make_grid(b_r, 0.0);
  return P;
}

// One streaming read of x: the x values of every candidate (p > L), unordered,
// appended to ck (h->ccount is 0 on entry: zero-filled workspace, reset by
// every tail).
int adapt_key_pass(const double* x, int64_t n, int b_r, const AdPlan& P, uint64_t* ck, int64_t cap, AdaptHdr* h,
                   int32_t* err, cudaStream_t s) {
  // one wave (4 CTAs per SM, the register-limited residency) up to 2^25
  // elements: GPT-2-sized in-place calls 47.6 vs 50.9 us at 6.3 M elements;
  // two waves above (2^26 standalone search 0.1155 vs 0.1168 ms)
  const int64_t per_sm = n <= (int64_t(1) << 25) ? 4 : 8;
  const unsigned kb = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 4095) / 4096, 148 * per_sm));
  if (b_r == 32) {
    // candidate <=> (low32 << 3) - c8 < w8 (thresholds in [2^27, 2^28] here)
    const uint32_t t = (uint32_t)(P.gL.thr < 0 ? 0 : (P.gL.thr > (1 << 28) ? (1 << 28) : P.gL.thr));
    const uint32_t c8L = (t + 1u) << 3;
    const uint32_t w8L = (t >= (1u << 28)) ? 0u : ((0x20000000u - 2u * t - 1u) << 3);
    adapt_keys32_kernel<<<kb, kAdThreads, 0, s>>>(x, n, P.g0, P.L_key, c8L, w8L, ck, cap, h, err);
  } else {
    adapt_keys_kernel<<<kb, kAdThreads, 0, s>>>(x, n, P.g0, P.L_key, P.gL.thr, ck, cap, h, err);
  }
  return vt_check_launch("adapt_keys_kernel");
}

TailArgs tail_args(const double* x, int64_t n, int64_t budget, int iters, const AdPlan& P, const AdPtrs& A,
                   double* tau_out, int32_t* err) {
  TailArgs ta{};
  ta.x = x;
  ta.g0 = P.g0;
  ta.cw = A.cw;
  ta.ck = A.ck;
  ta.c2 = A.c2;
  ta.ahist = A.ahist;
  ta.h = A.h;
  ta.cap = A.cap;
  ta.budget = budget;
  ta.n = n;
  ta.L_key = P.L_key;
  ta.lo_key = P.lo_key;
  ta.hi_key = P.hi_key;
  ta.s0 = P.s0;
  ta.iters = iters;
  ta.lower = P.lo;
  ta.upper = P.hi;
  ta.dthr = A.dthr;
  ta.tau_out = tau_out;
  ta.key = A.key;
  ta.st = A.st;
  ta.bhist = A.bhist;
  ta.bcand = A.bcand;
  ta.err = err;
  return ta;
}

int launch_tail(TailArgs& ta, double want, cudaStream_t s) {
  const int gmax = coop_grid(adapt_tail_kernel);
  const int grid = (int)std::min<int64_t>(gmax, std::max<int64_t>(64, (int64_t)(want / 2048)));
  void* args[] = {&ta};
  cudaLaunchCooperativeKernel((const void*)adapt_tail_kernel, dim3(grid), dim3(kAdThreads), args, 0, s);
  return vt_check_launch("adapt_tail_kernel");
}

__global__ void copy_key_kernel(const uint64_t* key, uint64_t* out) { *out = *key; }
}  // namespace vt

extern "C" int vt_round_log_adaptive(const double* x, int64_t n, int b_r, int64_t budget, int iters, int out_kind,
                                     void* out, uint64_t* sparse, int64_t sparse_cap, int64_t global_base,
                                     const int64_t* cursor_in, int64_t* cursor_out, double* tau_out,
                                     int64_t* counters, int32_t* err, void* ws, size_t ws_bytes, vt_stream_t stream) {
  if (n <= 0 || b_r < 10 || b_r > 32 || budget < 0 || iters < 0 || !tau_out || !sparse || !ws ||
      ws_bytes < vt_round_log_adaptive_workspace(n) || reinterpret_cast<uintptr_t>(ws) % 256) {
    vt_set_error("vt_round_log_adaptive: bad argument (n > 0, 256-byte aligned workspace)");
    return VT_EINVAL;
  }
  if ((out_kind == VT_OUT_F32 && (reinterpret_cast<uintptr_t>(out) & 15)) ||
      (reinterpret_cast<uintptr_t>(x) & 31) || (out_kind == VT_OUT_F64 && (reinterpret_cast<uintptr_t>(out) & 31))) {
    vt_set_error("vt_round_log_adaptive: misaligned x / output");
    return VT_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* w = static_cast<uint8_t*>(ws);
  const AdaptLayout lay = adapt_layout(n);
  const AdPtrs A = adapt_ptrs(w, lay);
  void* rws = w + lay.rl;
  const bool fast = b_r == 32;
  const AdPlan P = adapt_plan(n, b_r, budget);

  // In place (y overwrites x) the candidates' keys could not be gathered
  // after the rounding pass: their keys come from a read of x first.
  const size_t ybytes = out_kind == VT_OUT_F64 ? 8 : out_kind == VT_OUT_F32 ? 4 : 0;
  const uintptr_t xa = reinterpret_cast<uintptr_t>(x), ya = reinterpret_cast<uintptr_t>(out);
  const bool aliased = ybytes && ya < xa + (uintptr_t)n * 8 && xa < ya + (uintptr_t)n * ybytes;
  int rc = 0;
  if (aliased) {
    // 1'. the candidates' x values (unordered) from one read of x
    if ((rc = adapt_key_pass(x, n, b_r, P, A.ck, lay.cap, A.h, err, s))) return rc;
  } else {
    // 1. rounding pass: y + candidate words (local index << 1 | up) with p > L
    // (and each candidate's x at its position in ck: the tail reads it there)
    rc = rl_stream(x, n, P.gL, P.thrL, fast, out_kind, out, A.cw, lay.cap, 0, nullptr, &A.h->ccount, &A.h->scratch,
                   err, rws, s, nullptr, nullptr, A.ck);
    if (rc) return rc;
  }
  // 2-4. one cooperative launch: selection of the (budget+1)-th largest p
  // among the candidates, bisection, and (out of place) the ordered log; or
  // the exact fallback when the candidates cannot decide
  {
    TailArgs ta = tail_args(x, n, budget, iters, P, A, tau_out, err);
    if (!aliased) {
      ta.sparse = sparse;
      ta.sparse_cap = sparse_cap;
      ta.global_base = global_base;
      ta.cursor_in = cursor_in;
      ta.cursor_out = cursor_out;
      ta.counters = counters;
    }
    if ((rc = launch_tail(ta, P.want, s))) return rc;
  }
  // the rounding pass at the device tau: always for in-place calls, else only after a fallback
  return rl_stream(x, n, make_grid(b_r, P.lo), 0, fast, out_kind, out, sparse, sparse_cap, global_base, cursor_in,
                   cursor_out, counters, err, rws, s, A.dthr, aliased ? nullptr : &A.h->fallback);
}

// The standalone budget search (protocol.search_tau_budget): the in-place
// path's single read of x for the candidates' values, then the tail's
// selection + FP64 bisection (the exact multi-pass fallback inside the same
// cooperative launch when the candidates cannot decide).  No rounding pass.
extern "C" size_t vt_tau_budget_workspace(int64_t n) { return adapt_layout_rl(n > 0 ? n : 1, 0).total; }

extern "C" int vt_tau_budget(const double* x, int64_t n, int b_r, int64_t budget, int iters, double* tau_out,
                             uint64_t* key_out, int32_t* err, void* ws, size_t ws_bytes, vt_stream_t stream) {
  if (n <= 0 || b_r < 10 || b_r > 32 || budget < 0 || iters < 0 || !tau_out || !ws ||
      ws_bytes < vt_tau_budget_workspace(n) || reinterpret_cast<uintptr_t>(ws) % 256 ||
      (reinterpret_cast<uintptr_t>(x) & 31)) {
    vt_set_error("vt_tau_budget: bad argument (n > 0, 32-byte aligned x, 256-byte aligned workspace)");
    return VT_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const AdaptLayout lay = adapt_layout_rl(n, 0);
  const AdPtrs A = adapt_ptrs(static_cast<uint8_t*>(ws), lay);
  const AdPlan P = adapt_plan(n, b_r, budget);
  int rc = adapt_key_pass(x, n, b_r, P, A.ck, lay.cap, A.h, err, s);
  if (rc) return rc;
  TailArgs ta = tail_args(x, n, budget, iters, P, A, tau_out, err);  // sparse == nullptr: select only
  if ((rc = launch_tail(ta, P.want, s))) return rc;
  if (key_out) {
    copy_key_kernel<<<1, 1, 0, s>>>(A.key, key_out);
    return vt_check_launch("copy_key_kernel");
  }
  return 0;
}


// ---------------------------------------------------------------------------
// One tensor sharded over ranks: the budget search through the
// candidate path, with the two exchanges as collectives between the steps.
//   1. every rank: one read of its shard for the candidates above the GLOBAL
//      plan's L (the plan depends only on the global n and budget, so every
//      rank uses the same L), their keys, and a histogram of their top digit
//      plus the count above tau_hi, the candidate count and an overflow flag
//      (vt_tau_shard_candidates) -> summed over the ranks (all-reduce);
//   2. every rank: the same digit from the summed histogram, then its keys in
//      that digit (vt_tau_shard_digit_keys) -> gathered from every rank;
//   3. the exact order statistic among the gathered keys and the FP64
//      bisection (host).  One read of x per rank instead of the 5-pass exact
//      select, which remains the fallback (too few candidates / overflow).
// Exchange buffer (int64): [0, 2048) digit counts, [2048] keys > tau_hi,
// [2049] candidates, [2050] 1 if this rank's candidates overflowed.
// ---------------------------------------------------------------------------
namespace vt {
constexpr int kShardX = kAdBins + 3;

__global__ void __launch_bounds__(kAdThreads) shard_hist_kernel(uint64_t* __restrict__ ck, const AdaptHdr* h,
                                                                int64_t cap, Grid g0, uint64_t L_key,
                                                                uint64_t hi_key, int s0,
                                                                unsigned long long* __restrict__ xbuf,
                                                                int32_t* errp) {
  __shared__ uint32_t sh[kAdBins];
  __shared__ unsigned long long s_above;
  const int64_t Mraw = h->ccount;
  const int64_t M = Mraw < cap ? Mraw : cap;
  for (int i = threadIdx.x; i < kAdBins; i += kAdThreads) sh[i] = 0u;
  if (threadIdx.x == 0) s_above = 0ull;
  __syncthreads();
  uint32_t err = 0;
  unsigned long long above = 0;
  constexpr int kU = 8;  // loads in flight per thread
  const int64_t stride = (int64_t)gridDim.x * kAdThreads;
  for (int64_t i0 = (int64_t)blockIdx.x * kAdThreads + threadIdx.x; i0 < M; i0 += kU * stride) {
    uint64_t v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) v[u] = (i0 + u * stride < M) ? ck[i0 + u * stride] : 0ull;
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= M) break;
      const uint64_t key = dist_key(__longlong_as_double((long long)v[u]), g0, err);
      ck[i] = key;  // the keys, in place of the x values, for the digit step
      if (key > hi_key) ++above;
      else if (key > L_key) atomicAdd(&sh[(uint32_t)((key - L_key - 1) >> s0)], 1u);
    }
  }
  for (int o = 16; o > 0; o >>= 1) above += __shfl_xor_sync(0xffffffffu, above, o);
  if ((threadIdx.x & 31) == 0 && above) atomicAdd(&s_above, above);
  __syncthreads();
  for (int i = threadIdx.x; i < kAdBins; i += kAdThreads)
    if (sh[i]) atomicAdd(xbuf + i, (unsigned long long)sh[i]);
  if (threadIdx.x == 0) {
    if (s_above) atomicAdd(xbuf + kAdBins, s_above);
    if (blockIdx.x == 0) {
      xbuf[kAdBins + 1] = (unsigned long long)Mraw;
      xbuf[kAdBins + 2] = Mraw > cap ? 1ull : 0ull;
    }
  }
  report_err(errp, err);
}

__global__ void __launch_bounds__(kAdThreads) shard_digit_kernel(const uint64_t* __restrict__ ck, AdaptHdr* h,
                                                                 int64_t cap, uint64_t L_key, uint64_t hi_key,
                                                                 int s0, uint64_t digit,
                                                                 uint64_t* __restrict__ out, int64_t out_cap,
                                                                 unsigned long long* count) {
  const int64_t Mraw = h->ccount;
  const int64_t M = Mraw < cap ? Mraw : cap;
  const uint64_t lo1 = L_key + 1;
  const int lane = threadIdx.x & 31;
  constexpr int kU = 8;  // loads in flight per thread
  const int64_t stride = (int64_t)gridDim.x * kAdThreads;
  for (int64_t i0 = (int64_t)blockIdx.x * kAdThreads; i0 < M; i0 += kU * stride) {  // warp-uniform bounds
    uint64_t kv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + u * stride + threadIdx.x;
      kv[u] = i < M ? ck[i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t i = i0 + u * stride + threadIdx.x;
      const uint64_t key = kv[u];
      const bool in = i < M && key <= hi_key && key >= lo1 && ((key - lo1) >> s0) == digit;
      const uint32_t m = __ballot_sync(0xffffffffu, in);
      if (m) {
        const int leader = __ffs(m) - 1;
        unsigned long long pos = 0;
        if (lane == leader) pos = atomicAdd(count, (unsigned long long)__popc(m));
        pos = __shfl_sync(0xffffffffu, pos, leader);
        const unsigned long long p = pos + __popc(m & lanemask_lt());
        if (in && (int64_t)p < out_cap) out[p] = key;
      }
    }
  }
}

__global__ void shard_reset_kernel(AdaptHdr* h) { h->ccount = 0; }
}  // namespace vt

extern "C" size_t vt_tau_shard_workspace(int64_t n) { return adapt_layout_rl(n > 0 ? n : 1, 0).total; }

extern "C" int vt_tau_shard_candidates(const double* x, int64_t n, int b_r, int64_t n_global, int64_t budget,
                                       int64_t* xbuf, int32_t* err, void* ws, size_t ws_bytes, vt_stream_t stream) {
  if (n < 0 || n_global < n || n_global <= 0 || b_r < 10 || b_r > 32 || budget < 0 || !xbuf || !err || !ws ||
      ws_bytes < vt_tau_shard_workspace(n) || reinterpret_cast<uintptr_t>(ws) % 256 ||
      (n && (!x || (reinterpret_cast<uintptr_t>(x) & 31)))) {
    vt_set_error("vt_tau_shard_candidates: bad argument (0 <= n <= n_global, 32-byte aligned x, workspace)");
    return VT_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const AdaptLayout lay = adapt_layout_rl(n > 0 ? n : 1, 0);
  const AdPtrs A = adapt_ptrs(static_cast<uint8_t*>(ws), lay);
  const AdPlan P = adapt_plan(n_global, b_r, budget);  // the GLOBAL plan: the same L on every rank
  cudaMemsetAsync(xbuf, 0, sizeof(int64_t) * kShardX, s);
  shard_reset_kernel<<<1, 1, 0, s>>>(A.h);
  int rc = vt_check_launch("shard_reset_kernel");
  if (rc) return rc;
  if (n > 0 && (rc = adapt_key_pass(x, n, b_r, P, A.ck, lay.cap, A.h, err, s))) return rc;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((lay.cap + 4095) / 4096, 148 * 4));
  shard_hist_kernel<<<grid, kAdThreads, 0, s>>>(A.ck, A.h, lay.cap, P.g0, P.L_key, P.hi_key, P.s0,
                                                reinterpret_cast<unsigned long long*>(xbuf), err);
  return vt_check_launch("shard_hist_kernel");
}

extern "C" int vt_tau_shard_plan(int64_t n_global, int b_r, int64_t budget, uint64_t* L_key, int* s0) {
  if (n_global <= 0 || b_r < 10 || b_r > 32 || budget < 0 || !L_key || !s0) {
    vt_set_error("vt_tau_shard_plan: bad argument");
    return VT_EINVAL;
  }
  const AdPlan P = adapt_plan(n_global, b_r, budget);
  *L_key = P.L_key;
  *s0 = P.s0;
  return VT_OK;
}

extern "C" int vt_tau_shard_digit_keys(int64_t n, int b_r, int64_t n_global, int64_t budget, int64_t digit,
                                       uint64_t* keys_out, int64_t keys_cap, int64_t* count, void* ws,
                                       size_t ws_bytes, vt_stream_t stream) {
  if (n < 0 || n_global <= 0 || b_r < 10 || b_r > 32 || budget < 0 || digit < 0 || digit >= kAdBins || !count ||
      (keys_cap > 0 && !keys_out) || !ws || ws_bytes < vt_tau_shard_workspace(n)) {
    vt_set_error("vt_tau_shard_digit_keys: bad argument");
    return VT_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const AdaptLayout lay = adapt_layout_rl(n > 0 ? n : 1, 0);
  const AdPtrs A = adapt_ptrs(static_cast<uint8_t*>(ws), lay);
  const AdPlan P = adapt_plan(n_global, b_r, budget);
  cudaMemsetAsync(count, 0, sizeof(int64_t), s);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((lay.cap + 4095) / 4096, 148 * 4));
  shard_digit_kernel<<<grid, kAdThreads, 0, s>>>(A.ck, A.h, lay.cap, P.L_key, P.hi_key, P.s0, (uint64_t)digit,
                                                 keys_out, keys_cap, reinterpret_cast<unsigned long long*>(count));
  int rc = vt_check_launch("shard_digit_kernel");
  if (rc) return rc;
  shard_reset_kernel<<<1, 1, 0, s>>>(A.h);  // the workspace's candidate count starts at 0 for the next call
  return vt_check_launch("shard_reset_kernel");
}


// ---------------------------------------------------------------------------
// The same search with both exchanges over peer memory and no host step in
// the common path (vt_tau_shard_search_x): the rank's summed-histogram
// decision, its digit keys and the exact selection + bisection all run on
// the device, so one call enqueues the whole search and the host reads
// (status, tau) once.  Exchange buffer per rank (uint64 words, symmetric
// memory; zero-filled once):
//   [0] sequence number, [1] key counter, [2] CTA done counter,
//   [3 + par*W + r] rank r's phase-A (histogram) tag, [3 + 2W + par*W + r]
//   its phase-B (keys) tag, then the histogram buffers [par][r][kShardX],
//   the key counts [par][r], the keys [par][r][keys_cap] and a local
//   decision block {mode, digit, rank in digit, value bits}.
// Parities alternate per call as in the count exchange (vt_stream.cu).
// ---------------------------------------------------------------------------
namespace vt {
struct SXLayout {
  int world;
  int64_t kcap, hist, counts, keys, dec, total;
};
__host__ __device__ inline SXLayout sx_layout(int world, int64_t kcap) {
  SXLayout l;
  l.world = world;
  l.kcap = kcap;
  l.hist = 3 + 4 * (int64_t)world;
  l.counts = l.hist + 2 * (int64_t)world * kShardX;
  l.keys = l.counts + 2 * (int64_t)world;
  l.dec = l.keys + 2 * (int64_t)world * kcap;
  l.total = l.dec + 8;
  return l;
}
struct SXArgs {
  uint64_t* const* peers;
  uint64_t* own;
  int world, rank;
  SXLayout L;
  int64_t budget, n_global;
  uint64_t L_key, hi_key, lo_key;
  int s0, iters;
  double lower, upper;
};
enum { kSXValue = 0, kSXDigit = 1, kSXExact = 2 };

// 1 CTA: this rank's histogram buffer to every rank (phase A)
__global__ void __launch_bounds__(256) sx_publish_hist_kernel(const SXArgs a, const unsigned long long* xbuf) {
  const uint64_t seq = a.own[0] + 1ull;
  const int par = (int)(seq & 1ull);
  for (int p = 0; p < a.world; ++p) {
    uint64_t* dst = a.peers[p] + a.L.hist + ((int64_t)par * a.world + a.rank) * kShardX;
    for (int i = threadIdx.x; i < kShardX; i += blockDim.x) dst[i] = xbuf[i];
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    a.own[0] = seq;
    for (int p = 0; p < a.world; ++p) st_release_sys_u64(a.peers[p] + 3 + par * a.world + a.rank, seq);
  }
}

__device__ bool sx_wait(const SXArgs& a, int64_t tag0, uint64_t seq, int par, int32_t* err) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  for (int q = threadIdx.x; q < a.world; q += blockDim.x) {
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (ld_acquire_sys_u64(a.own + tag0 + par * a.world + q) != seq) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 10ull * 1000 * 1000 * 1000) {
        atomicOr(err, VT_ERR_EXCHANGE);
        s_ok = 0;
        break;
      }
      __nanosleep(100);
    }
  }
  __syncthreads();
  return s_ok != 0;
}

// 1 CTA: sum every rank's histogram buffer, decide as ShardedBudget.decide
__global__ void __launch_bounds__(256) sx_decide_kernel(const SXArgs a, int32_t* err) {
  __shared__ unsigned long long sum[kShardX];
  const uint64_t seq = a.own[0];
  const int par = (int)(seq & 1ull);
  uint64_t* dec = a.own + a.L.dec;
  if (!sx_wait(a, 3, seq, par, err)) {
    if (threadIdx.x == 0) {
      dec[0] = kSXExact;
      a.own[1] = 0ull;
      a.own[2] = 0ull;
    }
    return;
  }
  for (int i = threadIdx.x; i < kShardX; i += blockDim.x) {
    unsigned long long v = 0;
    for (int r = 0; r < a.world; ++r) v += __ldcg(a.own + a.L.hist + ((int64_t)par * a.world + r) * kShardX + i);
    sum[i] = v;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  a.own[1] = 0ull;  // the digit-key pass counts from 0
  a.own[2] = 0ull;
  const int64_t B = a.budget;
  const int64_t above_hi = (int64_t)sum[kAdBins], m = (int64_t)sum[kAdBins + 1];
  const bool overflow = sum[kAdBins + 2] != 0ull;
  uint64_t mode = kSXExact, digit = 0, rank = 0, val = 0;
  if (a.n_global <= B) {
    mode = kSXValue;
    val = a.lo_key;
  } else if (overflow) {
    mode = kSXExact;
  } else if (above_hi > B) {
    mode = kSXValue;
    val = 0x7ff0000000000000ull;  // v > tau_hi: the bisection ends at upper
  } else if (m < B + 1) {
    if (a.L_key <= a.lo_key) {
      mode = kSXValue;
      val = a.lo_key;
    }
  } else {
    const int64_t rk = B - above_hi;  // 0-based from the top among the keys in (L, hi]
    int64_t above = 0;
    for (int d = kAdBins - 1; d >= 0; --d) {
      const int64_t h = (int64_t)sum[d];
      if (above + h > rk) {
        mode = kSXDigit;
        digit = (uint64_t)d;
        rank = (uint64_t)(rk - above);
        break;
      }
      above += h;
    }
  }
  dec[0] = mode;
  dec[1] = digit;
  dec[2] = rank;
  dec[3] = val;
}

// grid: this rank's keys in the decided digit into every rank's key area (phase B)
__global__ void __launch_bounds__(kAdThreads) sx_digit_keys_kernel(const SXArgs a, const uint64_t* __restrict__ ck,
                                                                   const AdaptHdr* h, int64_t cap) {
  __shared__ unsigned s_last;
  const uint64_t seq = a.own[0];
  const int par = (int)(seq & 1ull);
  const uint64_t* dec = a.own + a.L.dec;
  const int lane = threadIdx.x & 31;
  if (dec[0] == kSXDigit) {
    const uint64_t digit = dec[1], lo1 = a.L_key + 1;
    const int64_t Mraw = h->ccount;
    const int64_t M = Mraw < cap ? Mraw : cap;
    constexpr int kU = 8;  // loads in flight per thread
    const int64_t stride = (int64_t)gridDim.x * kAdThreads;
    for (int64_t i0 = (int64_t)blockIdx.x * kAdThreads; i0 < M; i0 += kU * stride) {  // warp-uniform bounds
      uint64_t kv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = i0 + u * stride + threadIdx.x;
        kv[u] = i < M ? ck[i] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = i0 + u * stride + threadIdx.x;
        const uint64_t key = kv[u];
        const bool in = i < M && key <= a.hi_key && key >= lo1 && ((key - lo1) >> a.s0) == digit;
        const uint32_t m = __ballot_sync(0xffffffffu, in);
        if (m) {
          const int leader = __ffs(m) - 1;
          unsigned long long pos = 0;
          if (lane == leader)
            pos = atomicAdd(reinterpret_cast<unsigned long long*>(a.own + 1), (unsigned long long)__popc(m));
          pos = __shfl_sync(0xffffffffu, pos, leader);
          const int64_t q = (int64_t)(pos + __popc(m & lanemask_lt()));
          if (in && q < a.L.kcap)
            for (int p = 0; p < a.world; ++p)
              a.peers[p][a.L.keys + ((int64_t)par * a.world + a.rank) * a.L.kcap + q] = key;
        }
      }
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0)
    s_last = atomicAdd(reinterpret_cast<unsigned long long*>(a.own + 2), 1ull) == (unsigned long long)gridDim.x - 1;
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence_system();
  const uint64_t cnt = dec[0] == kSXDigit ? *(volatile uint64_t*)(a.own + 1) : 0ull;
  for (int p = 0; p < a.world; ++p) a.peers[p][a.L.counts + (int64_t)par * a.world + a.rank] = cnt;
  __threadfence_system();
  for (int p = 0; p < a.world; ++p) st_release_sys_u64(a.peers[p] + 3 + 2 * a.world + par * a.world + a.rank, seq);
}

// 1 CTA: gather every rank's digit keys, the exact order statistic, the bisection
__global__ void __launch_bounds__(kAdThreads) sx_finish_kernel(const SXArgs a, AdaptHdr* h, double* tau_out,
                                                               int32_t* status, int32_t* err) {
  __shared__ __align__(16) uint32_t sh[kBudBins];
  __shared__ int64_t s_tot;
  __shared__ int s_bad;
  const uint64_t seq = a.own[0];
  const int par = (int)(seq & 1ull);
  const uint64_t* dec = a.own + a.L.dec;
  const uint64_t mode = dec[0];
  const bool ok = sx_wait(a, 3 + 2 * (int64_t)a.world, seq, par, err);
  if (threadIdx.x == 0) {
    h->ccount = 0;  // the shard workspace's candidate count starts at 0 for the next call
    int64_t tot = 0;
    int bad = !ok || mode == kSXExact;
    if (ok && mode == kSXDigit)
      for (int r = 0; r < a.world; ++r) {
        const int64_t c = (int64_t)__ldcg(a.own + a.L.counts + (int64_t)par * a.world + r);
        if (c > a.L.kcap) bad = 1;
        tot += c;
      }
    s_tot = tot;
    s_bad = bad;
  }
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) *status = 1;  // the exact multi-pass path decides (host)
    return;
  }
  uint64_t key;
  if (mode == kSXValue) {
    key = dec[3];
  } else {
    // the rank-th largest among the gathered digit offsets o = key - L - 1 (the
    // digit's bits included), digit by digit over the low s0 bits
    const uint64_t lo1 = a.L_key + 1;
    const int64_t m = s_tot;
    int64_t rank = (int64_t)dec[2];
    uint64_t low = 0, lmask = 0;
    const uint64_t* base = a.own + a.L.keys + (int64_t)par * a.world * a.L.kcap;
    for (int top = a.s0; top > 0;) {
      const int bits = top < kAdBits ? top : kAdBits;
      top -= bits;
      for (int i = threadIdx.x; i < kAdBins; i += kAdThreads) sh[i] = 0;
      __syncthreads();
      for (int r = 0; r < a.world; ++r) {
        const int64_t c = (int64_t)__ldcg(a.own + a.L.counts + (int64_t)par * a.world + r);
        for (int64_t i = threadIdx.x; i < c; i += kAdThreads) {
          const uint64_t o = __ldcg(base + (int64_t)r * a.L.kcap + i) - lo1;
          if ((o & lmask) == low) atomicAdd(&sh[(uint32_t)(o >> top) & ((1u << bits) - 1u)], 1u);
        }
      }
      __syncthreads();
      int b2;
      int64_t ab2;
      select_digit(sh, 1 << bits, rank, b2, ab2);
      low |= (uint64_t)b2 << top;
      lmask |= ((1ull << bits) - 1ull) << top;
      rank -= ab2;
      __syncthreads();
    }
    (void)m;
    key = lo1 + ((dec[1] << a.s0) | low);
  }
  if (threadIdx.x == 0) {
    DevThr d;
    bisect_to(key, a.lower, a.upper, a.iters, &d, tau_out);
    *status = 0;
  }
}
}  // namespace vt

extern "C" size_t vt_tau_shard_exchange_words(int world, int64_t keys_cap) {
  return (world > 0 && keys_cap > 0) ? (size_t)vt::sx_layout(world, keys_cap).total : 0;
}

extern "C" int vt_tau_shard_search_x(const double* x, int64_t n, int b_r, int64_t n_global, int64_t budget,
                                     int iters, uint64_t* const* xpeers, uint64_t* own, int world, int rank,
                                     int64_t keys_cap, double* tau_out, int32_t* status, int32_t* err, void* ws,
                                     size_t ws_bytes, int phases, vt_stream_t stream) {
  using namespace vt;
  if (phases <= 0 || phases > 7 ||
      n < 0 || n_global < n || n_global <= 0 || b_r < 10 || b_r > 32 || budget < 0 || iters < 0 || !xpeers ||
      !own || world <= 0 || rank < 0 || rank >= world || keys_cap <= 0 || !tau_out || !status || !err || !ws ||
      ws_bytes < vt_tau_shard_workspace(n) + sizeof(int64_t) * kShardX ||
      reinterpret_cast<uintptr_t>(ws) % 256 || (n && (!x || (reinterpret_cast<uintptr_t>(x) & 31)))) {
    vt_set_error("vt_tau_shard_search_x: bad argument");
    return VT_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const AdaptLayout lay = adapt_layout_rl(n > 0 ? n : 1, 0);
  const AdPtrs A = adapt_ptrs(static_cast<uint8_t*>(ws), lay);
  const AdPlan P = adapt_plan(n_global, b_r, budget);
  // this rank's histogram buffer: after the shard workspace
  unsigned long long* xbuf =
      reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(ws) + vt_tau_shard_workspace(n));
  SXArgs a;
  a.peers = xpeers;
  a.own = own;
  a.world = world;
  a.rank = rank;
  a.L = sx_layout(world, keys_cap);
  a.budget = budget;
  a.n_global = n_global;
  a.L_key = P.L_key;
  a.hi_key = P.hi_key;
  a.lo_key = P.lo_key;
  a.s0 = P.s0;
  a.iters = iters;
  a.lower = P.lo;
  a.upper = P.hi;
  int rc;
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((lay.cap + 4095) / 4096, 148 * 4));
  if (phases & 1) {  // A: candidates, their digit histogram, to every rank
    cudaMemsetAsync(xbuf, 0, sizeof(int64_t) * kShardX, s);
    shard_reset_kernel<<<1, 1, 0, s>>>(A.h);
    if ((rc = vt_check_launch("shard_reset_kernel"))) return rc;
    if (n > 0 && (rc = adapt_key_pass(x, n, b_r, P, A.ck, lay.cap, A.h, err, s))) return rc;
    shard_hist_kernel<<<grid, kAdThreads, 0, s>>>(A.ck, A.h, lay.cap, P.g0, P.L_key, P.hi_key, P.s0, xbuf, err);
    if ((rc = vt_check_launch("shard_hist_kernel"))) return rc;
    sx_publish_hist_kernel<<<1, 256, 0, s>>>(a, xbuf);
    if ((rc = vt_check_launch("sx_publish_hist_kernel"))) return rc;
  }
  if (phases & 2) {  // B: the decision from every rank's histogram, this rank's digit keys to every rank
    sx_decide_kernel<<<1, 256, 0, s>>>(a, err);
    if ((rc = vt_check_launch("sx_decide_kernel"))) return rc;
    sx_digit_keys_kernel<<<grid, kAdThreads, 0, s>>>(a, A.ck, A.h, lay.cap);
    if ((rc = vt_check_launch("sx_digit_keys_kernel"))) return rc;
  }
  if (phases & 4) {  // C: every rank's digit keys, the exact order statistic, the bisection
    sx_finish_kernel<<<1, kAdThreads, 0, s>>>(a, A.h, tau_out, status, err);
    if ((rc = vt_check_launch("sx_finish_kernel"))) return rc;
  }
  return VT_OK;
}

extern "C" size_t vt_tau_shard_search_x_workspace(int64_t n) {
  return vt_tau_shard_workspace(n) + sizeof(int64_t) * vt::kShardX;
}


// ---------------------------------------------------------------------------
// Batched adaptive round-and-log: many independent tensors (configs[2]: the
// 161 ResNet-50 intermediates), each with its own budget, tau and log, in a
// fixed number of launches instead of ~12 per tensor:
//
//   rl_batch_kernel (candidate pass) -> adapt_hist_batch -> adapt_select_batch
//   -> adapt_filter_batch -> [exact fallback: adapt_fb_roster, one
//   cooperative adapt_fb_batch, rl_batch_kernel gated per tensor]
//
// Same per-tensor algorithm and state as vt_round_log_adaptive (the kernel
// bodies are shared); each tensor gets a share of the tail grids in
// proportion to its expected candidate count, and the per-tensor "last CTA"
// steps count that share.  The tables travel as __grid_constant__ kernel
// parameters, so a batch is graph-capturable with no descriptor upload.
// ---------------------------------------------------------------------------
namespace vt {

struct AdSeg {
  const double* x;
  uint8_t* ws;        // the tensor's adaptive state (adapt_layout_rl(n, 0))
  uint64_t* log;
  int64_t* flags;     // int32 error bits at flags[0], log entries at flags[2]
  double* tau_out;
  int64_t n, budget, log_cap, global_base;
  uint64_t L_key;
  int32_t s0, blk0;   // top-digit shift; first CTA of the tensor in the tail grids
};

// the batch's fallback roster: which tensors run the exact selection
struct FbRoster {
  int32_t count;
  int32_t pad[63];
  int32_t list[kMaxBatch];
};

struct AdBatch {
  Grid g0;
  double lo, hi;
  uint64_t lo_key, hi_key;
  FbRoster* fb;
  int32_t nseg, nblk, iters, pad;
  AdSeg seg[kMaxBatch];
};

__device__ __forceinline__ int ad_find(const AdBatch& b, int64_t blk) {
  int lo = 0, hi = b.nseg - 1;  // last tensor with blk0 <= blk
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (b.seg[mid].blk0 <= blk) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ int64_t ad_nblk(const AdBatch& b, int j) {
  return (j + 1 < b.nseg ? b.seg[j + 1].blk0 : b.nblk) - b.seg[j].blk0;
}

__global__ void __launch_bounds__(kAdThreads) adapt_hist_batch_kernel(const __grid_constant__ AdBatch b) {
  const int j = ad_find(b, blockIdx.x);
  const AdSeg& sg = b.seg[j];
  const AdPtrs p = adapt_ptrs(sg.ws, adapt_layout_rl(sg.n, 0));
  if (blockIdx.x == 0 && threadIdx.x == 0) b.fb->count = 0;  // the previous batch's fallback kernels are done
  adapt_hist_body(sg.x, b.g0, p.cw, p.ck, p.cd, p.cap, sg.budget, sg.L_key, b.hi_key, sg.s0, p.h, p.ahist, p.fst,
                  (int64_t)blockIdx.x - sg.blk0, ad_nblk(b, j));
}

__global__ void __launch_bounds__(kAdThreads) adapt_select_batch_kernel(const __grid_constant__ AdBatch b) {
  const int j = ad_find(b, blockIdx.x);
  const AdSeg& sg = b.seg[j];
  const AdPtrs p = adapt_ptrs(sg.ws, adapt_layout_rl(sg.n, 0));
  adapt_select_body(p.ck, p.cd, b.g0, sg.L_key, b.hi_key, sg.s0, p.h, p.c2, b.lo, b.hi, b.iters, p.dthr, sg.tau_out, p.key,
                    (int64_t)blockIdx.x - sg.blk0, ad_nblk(b, j));
}

#ifndef VT_FILTER_MINB  // resident CTAs per SM the batch filter is compiled for (64 registers; 1: 68 registers, 3 CTAs/SM, configs[2] 2.15-2.17 vs 2.14 ms)
#define VT_FILTER_MINB 4
#endif
__global__ void __launch_bounds__(kAdThreads, VT_FILTER_MINB) adapt_filter_batch_kernel(const __grid_constant__ AdBatch b) {
  const int j = ad_find(b, blockIdx.x);
  const AdSeg& sg = b.seg[j];
  const AdPtrs p = adapt_ptrs(sg.ws, adapt_layout_rl(sg.n, 0));
  adapt_filter_body(p.cw, p.ck, p.cd, b.g0, sg.L_key, b.hi_key, sg.s0, p.h, p.dthr, sg.log, sg.log_cap, sg.global_base, nullptr, nullptr, sg.flags + 2,
                    p.fst, ad_nblk(b, j));
}

// exact fallback: one CTA per tensor adds the tensors that need it to a
// roster; one cooperative launch then runs the exact selection of every
// rostered tensor in turn (returning at once when the roster is empty)
__global__ void adapt_fb_roster_kernel(const __grid_constant__ AdBatch b) {
  const AdSeg& sg = b.seg[blockIdx.x];
  const AdPtrs p = adapt_ptrs(sg.ws, adapt_layout_rl(sg.n, 0));
  if (threadIdx.x == 0 && p.h->fallback) b.fb->list[atomicAdd(&b.fb->count, 1)] = (int32_t)blockIdx.x;
}

__global__ void __launch_bounds__(kAdThreads) adapt_fb_batch_kernel(const __grid_constant__ AdBatch b) {
  __shared__ uint32_t sh[kBudBins];
  const int nfb = *(volatile int32_t*)&b.fb->count;
  for (int k = 0; k < nfb; ++k) {
    const AdSeg& sg = b.seg[b.fb->list[k]];
    const AdPtrs p = adapt_ptrs(sg.ws, adapt_layout_rl(sg.n, 0));
    fb_selection(sg.x, sg.n, b.g0, p.h, p.st, p.bhist, p.bcand, sg.budget, b.lo_key, b.hi_key, b.lo, b.hi, b.iters,
                 p.key, p.dthr, sg.tau_out, reinterpret_cast<int32_t*>(sg.flags), sh);
  }
}
}  // namespace vt

namespace {
size_t batch_rl_bytes(const int64_t* n, int nseg) {
  int64_t worst = 0;  // the largest chunk's tickets: chunks run one after another on one stream
  for (int c = 0; c < nseg; c += kMaxBatch) {
    int64_t t = 0;
    for (int j = c; j < std::min(nseg, c + kMaxBatch); ++j) t += rl_batch_tickets(n[j]);
    worst = std::max(worst, t);
  }
  return al256(sizeof(FbRoster)) + al256(rl_batch_workspace(worst));
}
}  // namespace

extern "C" size_t vt_round_log_adaptive_batch_workspace(const int64_t* n, int nseg) {
  if (!n || nseg <= 0) return 0;
  size_t total = batch_rl_bytes(n, nseg);
  for (int j = 0; j < nseg; ++j) total += adapt_layout_rl(std::max<int64_t>(n[j], 0), 0).total;
  return total;
}

extern "C" int vt_round_log_adaptive_batch(const vt_adaptive_segment* segs, int nseg, int b_r, int iters,
                                           int out_kind, void* ws, size_t ws_bytes, vt_stream_t stream) {
  if (!segs || nseg <= 0 || b_r < 10 || b_r > 32 || iters < 0 || !ws || reinterpret_cast<uintptr_t>(ws) % 256 ||
      (out_kind != VT_OUT_F32 && out_kind != VT_OUT_F64)) {
    vt_set_error("vt_round_log_adaptive_batch: bad argument");
    return VT_EINVAL;
  }
  std::vector<int64_t> ns((size_t)nseg);
  const size_t ybytes = out_kind == VT_OUT_F64 ? 8 : 4;
  for (int j = 0; j < nseg; ++j) {
    const vt_adaptive_segment& sg = segs[j];
    ns[(size_t)j] = sg.n;
    const uintptr_t xa = reinterpret_cast<uintptr_t>(sg.x), ya = reinterpret_cast<uintptr_t>(sg.out);
    if (sg.n <= 0 || !sg.x || !sg.out || !sg.log || !sg.tau_out || !sg.flags || sg.budget < 0 ||
        sg.log_cap < 0 || (xa & 31) || (ya & (out_kind == VT_OUT_F64 ? 31 : 15))) {
      vt_set_error("vt_round_log_adaptive_batch: bad segment (n > 0, x 32-byte aligned, output aligned)");
      return VT_EINVAL;
    }
    if (ya < xa + (uintptr_t)sg.n * 8 && xa < ya + (uintptr_t)sg.n * ybytes) {
      vt_set_error("vt_round_log_adaptive_batch: in-place segments are not batched (use vt_round_log_adaptive)");
      return VT_EINVAL;
    }
  }
  if (ws_bytes < vt_round_log_adaptive_batch_workspace(ns.data(), nseg)) {
    vt_set_error("vt_round_log_adaptive_batch: workspace too small");
    return VT_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* w = static_cast<uint8_t*>(ws);
  FbRoster* roster = reinterpret_cast<FbRoster*>(w);
  void* rl_hdr = w + al256(sizeof(FbRoster));
  uint8_t* seg_ws = w + batch_rl_bytes(ns.data(), nseg);
  const bool fast = b_r == 32;
  const double lo = 0x1p-25, hi = ldexp(1.0, 8 - b_r);
  uint64_t lo_key, hi_key;
  memcpy(&lo_key, &lo, 8);
  memcpy(&hi_key, &hi, 8);
  const Grid g0 = make_grid(b_r, 0.0);
  int rc = 0;
  for (int c0 = 0; c0 < nseg; c0 += kMaxBatch) {
    const int m = std::min(nseg - c0, kMaxBatch);
    RLBatch cand{}, fb{};
    AdBatch ab{};
    cand.g = fb.g = g0;
    cand.hdr = fb.hdr = rl_hdr;
    cand.nseg = fb.nseg = ab.nseg = m;
    ab.g0 = g0;
    ab.lo = lo;
    ab.hi = hi;
    ab.lo_key = lo_key;
    ab.hi_key = hi_key;
    ab.iters = iters;
    ab.fb = roster;
    fb.any = &roster->count;
    int64_t tick = 0, blk = 0;
    for (int i = 0; i < m; ++i) {
      const vt_adaptive_segment& sg = segs[c0 + i];
      const int64_t n = sg.n, budget = sg.budget;
      const AdaptLayout lay = adapt_layout_rl(n, 0);
      const AdPtrs p = adapt_ptrs(seg_ws, lay);
      // candidate threshold and top-digit width: as vt_round_log_adaptive
      const double want = (double)kCandFactor * (double)(budget + 1) + 1024.0;
      double L = hi * (1.0 - want / (double)n);
      if (!(L > lo)) L = lo;
      uint64_t L_key;
      memcpy(&L_key, &L, 8);
      const uint64_t W = hi_key - L_key;
      const int wbits = W > 1 ? 64 - __builtin_clzll(W - 1) : 1;
      const Grid gL = make_grid(b_r, L);
      int32_t* err = reinterpret_cast<int32_t*>(sg.flags);
      RLSeg& rc_ = cand.seg[i];
      rc_.x = sg.x;
      rc_.out = sg.out;
      rc_.sparse = p.cw;
      rc_.keys = p.ck;  // the rounding pass stages each candidate's key
      rc_.cursor_out = &p.h->ccount;
      rc_.counters = &p.h->scratch;
      rc_.err = err;
      rc_.n = n;
      rc_.cap = p.cap;
      rc_.global_base = 0;
      rc_.tick0 = tick;
      rc_.thr = gL.thr;
      rc_.thr_sub = gL.thr_sub;
      rc_.thr32 = (int32_t)std::min<int64_t>(std::max<int64_t>(gL.thr, 0), INT32_MAX);
      RLSeg& rf = fb.seg[i];
      rf = rc_;
      rf.sparse = sg.log;
      rf.cursor_out = nullptr;
      rf.counters = sg.flags + 2;
      rf.cap = sg.log_cap;
      rf.global_base = sg.global_base;
      rf.dthr = p.dthr;
      rf.gate = &p.h->fallback;
      rf.keys = nullptr;
      tick += rl_batch_tickets(n);
      AdSeg& a = ab.seg[i];
      a.x = sg.x;
      a.ws = seg_ws;
      a.log = sg.log;
      a.flags = sg.flags;
      a.tau_out = sg.tau_out;
      a.n = n;
      a.budget = budget;
      a.log_cap = sg.log_cap;
      a.global_base = sg.global_base;
      a.L_key = L_key;
      a.s0 = std::max(0, wbits - kAdBits);
      a.blk0 = (int32_t)blk;
      // a tail CTA per 8192 expected candidates: each has several gathers /
      // filter tickets in flight, so the chain of dependent steps per CTA
      // (ticket, load, look-back, store, arrival) is paid ~2 waves deep
      blk += std::max<int64_t>(1, std::min<int64_t>((int64_t)(want + 8191) / 8192, 148 * 4));
      seg_ws += lay.total;
    }
    cand.total = fb.total = tick;
    ab.nblk = (int32_t)blk;
    // 1. rounding pass over every tensor: y + ordered candidate words
    if ((rc = rl_stream_batch(cand, fast, out_kind, s, /*keys=*/true))) return rc;
    // 2-4. per tensor: digit histogram, exact selection + bisection, ordered filter
    adapt_hist_batch_kernel<<<(unsigned)blk, kAdThreads, 0, s>>>(ab);
    if ((rc = vt_check_launch("adapt_hist_batch_kernel"))) return rc;
    adapt_select_batch_kernel<<<(unsigned)blk, kAdThreads, 0, s>>>(ab);
    if ((rc = vt_check_launch("adapt_select_batch_kernel"))) return rc;
    adapt_filter_batch_kernel<<<(unsigned)blk, kAdThreads, 0, s>>>(ab);
    if ((rc = vt_check_launch("adapt_filter_batch_kernel"))) return rc;
    // exact fallback for the tensors whose candidates could not decide (no-ops otherwise)
    adapt_fb_roster_kernel<<<(unsigned)m, 32, 0, s>>>(ab);
    if ((rc = vt_check_launch("adapt_fb_roster_kernel"))) return rc;
    {
      void* args[] = {&ab};
      cudaLaunchCooperativeKernel((const void*)adapt_fb_batch_kernel, dim3(coop_grid(adapt_fb_batch_kernel)),
                                  dim3(kAdThreads), args, 0, s);
      if ((rc = vt_check_launch("adapt_fb_batch_kernel"))) return rc;
    }
    if ((rc = rl_stream_batch(fb, fast, out_kind, s))) return rc;
  }
  return 0;
}

namespace {
template <int P>
int hist_pass(const double* x, int64_t n, const Grid& g, SelectState* st, uint32_t* hist, int32_t* err,
              cudaStream_t s) {
  constexpr size_t smem = sizeof(uint32_t) << pass_bits(P);
  auto hk = tau_hist_kernel<P>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t want = (n + kHistThreads * 8 - 1) / (kHistThreads * 8);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, 148 * 2));
  hk<<<blocks, kHistThreads, smem, s>>>(x, n, g, st, hist + (size_t)P * kMaxBins, err);
  return vt_check_launch("tau_hist_kernel");
}

template <int P>
int select_pass(SelectState* st, uint32_t* hist, uint64_t* key_out, cudaStream_t s) {
  tau_select_kernel<P><<<1, kSelThreads, 0, s>>>(hist + (size_t)P * kMaxBins, st, key_out);
  return vt_check_launch("tau_select_kernel");
}

template <int P>
int run_pass(const double* x, int64_t n, const Grid& g, SelectState* st, uint32_t* hist,
             uint64_t* key_out, int32_t* err, cudaStream_t s) {
  int rc = hist_pass<P>(x, n, g, st, hist, err, s);
  return rc ? rc : select_pass<P>(st, hist, key_out, s);
}
}  // namespace

extern "C" int vt_tau_kth_key(const double* x, int64_t n, int b_r, int64_t rank, uint64_t* key_out,
                              int32_t* err, void* ws, size_t ws_bytes, vt_stream_t stream) {
  if (n < 0 || b_r < 10 || b_r > 32 || rank < 0 || !key_out || !err || !ws ||
      ws_bytes < vt_tau_workspace(n)) {
    vt_set_error("vt_tau_kth_key: bad argument");
    return VT_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* hist = static_cast<uint32_t*>(ws);
  SelectState* st = reinterpret_cast<SelectState*>(static_cast<uint8_t*>(ws) + (size_t)kPasses * kMaxBins * 4);
  if (cudaMemsetAsync(hist, 0, (size_t)kPasses * kMaxBins * 4, s) != cudaSuccess) return vt_check_launch("memset");
  init_state_kernel<<<1, 1, 0, s>>>(st, rank, key_out);
  int rc = vt_check_launch("init_state_kernel");
  if (rc || n == 0 || rank >= n) return rc;
  const Grid g = make_grid(b_r, 0.0);
  if ((rc = run_pass<0>(x, n, g, st, hist, key_out, err, s))) return rc;
  if ((rc = run_pass<1>(x, n, g, st, hist, key_out, err, s))) return rc;
  if ((rc = run_pass<2>(x, n, g, st, hist, key_out, err, s))) return rc;
  if ((rc = run_pass<3>(x, n, g, st, hist, key_out, err, s))) return rc;
  return run_pass<4>(x, n, g, st, hist, key_out, err, s);
}

// Sharded exact order statistic (one tensor split across ranks): the passes
// of vt_tau_kth_key one at a time, so the ranks can sum each pass's
// histogram (ncclAllReduce) before every rank makes the same selection.
extern "C" size_t vt_tau_kth_hist_offset(int pass) { return (size_t)pass * kMaxBins * sizeof(uint32_t); }
extern "C" int vt_tau_kth_hist_bins(int pass) { return pass == 4 ? (1 << pass_bits(4)) : (1 << pass_bits(0)); }

extern "C" int vt_tau_kth_begin(int64_t rank, uint64_t* key_out, void* ws, size_t ws_bytes, vt_stream_t stream) {
  if (rank < 0 || !key_out || !ws || ws_bytes < vt_tau_workspace(0)) {
    vt_set_error("vt_tau_kth_begin: bad argument");
    return VT_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* hist = static_cast<uint32_t*>(ws);
  SelectState* st = reinterpret_cast<SelectState*>(static_cast<uint8_t*>(ws) + (size_t)kPasses * kMaxBins * 4);
  if (cudaMemsetAsync(hist, 0, (size_t)kPasses * kMaxBins * 4, s) != cudaSuccess) return vt_check_launch("memset");
  init_state_kernel<<<1, 1, 0, s>>>(st, rank, key_out);
  return vt_check_launch("init_state_kernel");
}

extern "C" int vt_tau_kth_hist(const double* x, int64_t n, int b_r, int pass, int32_t* err, void* ws,
                               size_t ws_bytes, vt_stream_t stream) {
  if (n < 0 || b_r < 10 || b_r > 32 || pass < 0 || pass >= kPasses || !err || !ws || (n > 0 && !x) ||
      ws_bytes < vt_tau_workspace(n)) {
    vt_set_error("vt_tau_kth_hist: bad argument");
    return VT_EINVAL;
  }
  if (n == 0) return VT_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* hist = static_cast<uint32_t*>(ws);
  SelectState* st = reinterpret_cast<SelectState*>(static_cast<uint8_t*>(ws) + (size_t)kPasses * kMaxBins * 4);
  const Grid g = make_grid(b_r, 0.0);
  switch (pass) {
    case 0: return hist_pass<0>(x, n, g, st, hist, err, s);
    case 1: return hist_pass<1>(x, n, g, st, hist, err, s);
    case 2: return hist_pass<2>(x, n, g, st, hist, err, s);
    case 3: return hist_pass<3>(x, n, g, st, hist, err, s);
    default: return hist_pass<4>(x, n, g, st, hist, err, s);
  }
}

extern "C" int vt_tau_kth_select(int pass, uint64_t* key_out, void* ws, size_t ws_bytes, vt_stream_t stream) {
  if (pass < 0 || pass >= kPasses || !key_out || !ws || ws_bytes < vt_tau_workspace(0)) {
    vt_set_error("vt_tau_kth_select: bad argument");
    return VT_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t* hist = static_cast<uint32_t*>(ws);
  SelectState* st = reinterpret_cast<SelectState*>(static_cast<uint8_t*>(ws) + (size_t)kPasses * kMaxBins * 4);
  switch (pass) {
    case 0: return select_pass<0>(st, hist, key_out, s);
    case 1: return select_pass<1>(st, hist, key_out, s);
    case 2: return select_pass<2>(st, hist, key_out, s);
    case 3: return select_pass<3>(st, hist, key_out, s);
    default: return select_pass<4>(st, hist, key_out, s);
  }
}

extern "C" int vt_min_f64(const double* s, int64_t n, double* out, int32_t* nan_flag, vt_stream_t stream) {
  if (n < 0 || !out || !nan_flag || (n && !s)) {
    vt_set_error("vt_min_f64: bad argument");
    return VT_EINVAL;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  min_init_kernel<<<1, 1, 0, st>>>(out);
  if (n) {
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 4));
    min_kernel<<<blocks, 256, 0, st>>>(s, n, out, nan_flag);
  }
  min_final_kernel<<<1, 1, 0, st>>>(out);
  return vt_check_launch("min_kernel");
}
