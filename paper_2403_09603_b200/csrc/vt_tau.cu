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

#include "vt_common.cuh"

namespace vt {

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

// FP64 bit pattern of p for one element; err gets rnd's error bits.
__device__ __forceinline__ uint64_t dist_key(double x, const Grid& g, uint32_t& err) {
  const uint64_t bits = (uint64_t)__double_as_longlong(x);
  const uint64_t mag = bits & kMag;
  if (mag >= kNormalMin) {
    const uint64_t low = mag & g.low_mask;
    const uint64_t base = mag >> g.drop;
    const bool up = (low > g.half) || ((low == g.half) && (base & 1ull));
    const uint64_t rmag = (base + (up ? 1ull : 0ull)) << g.drop;
    err |= (mag >= kExpAllOnes) ? (uint32_t)VT_ERR_NONFINITE
                                : ((rmag > g.gmax_bits) ? (uint32_t)VT_ERR_RANGE : 0u);
    const uint64_t d = up ? (g.one - low) : low;  // |x - r| = d * 2^(E-52), scale = 2^E
    return (uint64_t)__double_as_longlong(__dmul_rn(__ull2double_rn(d), 0x1p-52));
  }
  const double r = __dmul_rn(rint(__dmul_rn(x, g.sub_up)), g.sub_dn);
  return (uint64_t)__double_as_longlong(__dmul_rn(fabs(__dsub_rn(x, r)), 0x1p126));
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

__global__ void __launch_bounds__(256) bud_pass_kernel(const double* __restrict__ x, int64_t n, Grid g,
                                                       BudState* st, uint32_t* __restrict__ hist,
                                                       uint64_t* __restrict__ cand, int32_t* errp) {
  __shared__ uint32_t sh[kBudBins];
  __shared__ unsigned long long s_above;
  if (st->status != 0) return;
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
  for (int64_t base = (int64_t)blockIdx.x * 1024; base < n; base += (int64_t)gridDim.x * 1024) {
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

// Pick the digit of the rank-th largest key (descending scan by one CTA).
__device__ void select_digit(const uint32_t* hist, int nbins, int64_t rank, int& bin, int64_t& above_out) {
  __shared__ unsigned long long s_warp[kSelThreads / 32];
  __shared__ int s_bin;
  __shared__ long long s_above;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int per = (nbins + kSelThreads - 1) / kSelThreads;
  const int hi = nbins - t * per;
  unsigned long long mine = 0;
  for (int k = 0; k < per; ++k) {
    const int b = hi - 1 - k;
    if (b >= 0) mine += hist[b];
  }
  unsigned long long incl = mine;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[warp] = incl;
  if (t == 0) s_bin = -1;
  __syncthreads();
  if (warp == 0) {
    const unsigned long long v = s_warp[lane];
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
__global__ void __launch_bounds__(kSelThreads) bud_step_kernel(BudState* st, const uint32_t* __restrict__ hist,
                                                               const uint64_t* __restrict__ cand, int64_t budget,
                                                               uint64_t* key_out) {
  __shared__ uint32_t sh[kBudBins];
  if (st->status != 0) return;
  const uint64_t lo1 = st->lo_key + 1;
  if (st->compacting) {  // exact select among the compacted candidates
    const int64_t m = (int64_t)st->cand;
    uint64_t prefix = st->prefix, pmask = st->pmask;
    int64_t rank = st->rank;
    for (int lv = st->level; lv < st->nlevels; ++lv) {
      const int sh_lv = st->shift[lv], bits = st->bits[lv];
      for (int i = threadIdx.x; i < kBudBins; i += kSelThreads) sh[i] = 0;
      __syncthreads();
      for (int64_t i = threadIdx.x; i < m; i += kSelThreads) {
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
  select_digit(hist + (size_t)level * kBudBins, 1 << st->bits[level], rank, bin, above);
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

__global__ void bud_init_kernel(BudState* st, uint64_t lo_key, uint64_t hi_key, uint64_t* key_out,
                                uint32_t* hist) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kBudMaxLevels * kBudBins; i += gridDim.x * blockDim.x)
    hist[i] = 0u;
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
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

}  // namespace vt

using namespace vt;

extern "C" size_t vt_tau_workspace(int64_t n) {
  (void)n;
  const size_t radix = (size_t)kPasses * kMaxBins * sizeof(uint32_t) + 256;
  const size_t budget = 512 + (size_t)kBudMaxLevels * kBudBins * 4 + (size_t)kCandCap * 8;
  return std::max(radix, budget);
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

extern "C" size_t vt_round_log_adaptive_workspace(int64_t n) {
  return 256 + vt_tau_workspace(n) + vt_round_log_workspace(n);
}

extern "C" int vt_round_log_adaptive(const double* x, int64_t n, int b_r, int64_t budget, int iters, int out_kind,
                                     void* out, uint64_t* sparse, int64_t sparse_cap, int64_t global_base,
                                     const int64_t* cursor_in, int64_t* cursor_out, double* tau_out,
                                     int64_t* counters, int32_t* err, void* ws, size_t ws_bytes, vt_stream_t stream) {
  if (n <= 0 || b_r < 10 || b_r > 32 || budget < 0 || iters < 0 || !tau_out || !sparse || !ws ||
      ws_bytes < vt_round_log_adaptive_workspace(n) || reinterpret_cast<uintptr_t>(ws) % 256) {
    vt_set_error("vt_round_log_adaptive: bad argument (n > 0, 256-byte aligned workspace)");
    return VT_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint8_t* w = static_cast<uint8_t*>(ws);
  DevThr* dthr = reinterpret_cast<DevThr*>(w);
  uint64_t* key = reinterpret_cast<uint64_t*>(w + 64);
  int32_t* status = reinterpret_cast<int32_t*>(w + 72);
  void* tws = w + 256;
  const size_t tws_bytes = vt_tau_workspace(n);
  void* rws = w + 256 + ((tws_bytes + 255) & ~(size_t)255);
  // the round-and-log workspace keeps an epoch header at its start: keep it
  // at a fixed place (it must stay zero-filled until first use)
  const double lo = 0x1p-25, hi = ldexp(1.0, 8 - b_r);
  int rc = vt_tau_budget_key(x, n, b_r, budget, lo, hi, key, status, err, tws, tws_bytes, stream);
  if (rc) return rc;
  budget_bisect_kernel<<<1, 1, 0, s>>>(key, lo, hi, iters, dthr, tau_out);
  if ((rc = vt_check_launch("budget_bisect_kernel"))) return rc;
  const Grid g = make_grid(b_r, lo);  // thresholds come from dthr
  const size_t rws_bytes = ws_bytes - (static_cast<uint8_t*>(rws) - w);
  if (rws_bytes < vt_round_log_workspace(n)) {
    vt_set_error("vt_round_log_adaptive: workspace too small");
    return VT_EINVAL;
  }
  if (out_kind == VT_OUT_F32 && (reinterpret_cast<uintptr_t>(out) & 15)) {
    vt_set_error("vt_round_log_adaptive: misaligned output");
    return VT_EINVAL;
  }
  if ((reinterpret_cast<uintptr_t>(x) & 31) || (out_kind == VT_OUT_F64 && (reinterpret_cast<uintptr_t>(out) & 31))) {
    vt_set_error("vt_round_log_adaptive: misaligned x / output");
    return VT_EINVAL;
  }
  return rl_stream(x, n, g, 0, b_r == 32, out_kind, out, sparse, sparse_cap, global_base, cursor_in, cursor_out,
                   counters, err, rws, s, dthr);
}

namespace {
template <int P>
int run_pass(const double* x, int64_t n, const Grid& g, SelectState* st, uint32_t* hist,
             uint64_t* key_out, int32_t* err, cudaStream_t s) {
  constexpr size_t smem = sizeof(uint32_t) << pass_bits(P);
  auto hk = tau_hist_kernel<P>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t want = (n + kHistThreads * 8 - 1) / (kHistThreads * 8);
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, 148 * 2));
  hk<<<blocks, kHistThreads, smem, s>>>(x, n, g, st, hist + (size_t)P * kMaxBins, err);
  int rc = vt_check_launch("tau_hist_kernel");
  if (rc) return rc;
  tau_select_kernel<P><<<1, kSelThreads, 0, s>>>(hist + (size_t)P * kMaxBins, st, key_out);
  return vt_check_launch("tau_select_kernel");
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
