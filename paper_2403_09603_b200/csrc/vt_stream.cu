// Persistent, TMA-pipelined streaming kernels for the north-star path
// (sparse log, FP32 / FP64 output):
//
//   rl_stream_kernel   trainer round-and-log (protocol._TrainerChannel.process,
//                      pkg/src/vtrain/protocol.py:198-202) -- rounds every element,
//                      and stages each tile's logged elements as 16-bit local
//                      entries (11-bit offset | up << 15) + a per-tile count;
//   rl_expand_kernel   block-level decoupled look-back prefix sum over the tile
//                      counts, then expands the staged entries into the global
//                      ascending uint64 log (global_index << 1 | up);
//   rp_stream_kernel   auditor replay (protocol._AuditorChannel.process,
//                      protocol.py:212-216) -- scatters the tile's log slice into a
//                      shared-memory code map and replays every element.
//
// Each CTA is persistent (grid = resident CTAs) and walks tiles
// blockIdx.x, blockIdx.x + gridDim.x, ...; the FP64 input of the next
// kStages tiles is in flight at all times through cp.async.bulk (TMA bulk
// copies, L2 evict-first) into a shared-memory ring guarded by mbarriers, so
// HBM streams continuously while the SM computes.  No CTA ever waits on
// another CTA in the streaming pass; the only cross-CTA wait is the
// look-back of the small expand pass.
#include <algorithm>

#include "vt_common.cuh"

namespace vt {

constexpr int kSThreads = 256;
constexpr int kSTile = 2048;  // elements per tile (16 KiB of FP64)
constexpr int kStages = 4;
constexpr int kSWarpElems = kSTile / kWarps;  // 256
constexpr int kSSlots = kSWarpElems / 64;     // 4 slots x 32 lanes x 2 elements
constexpr int kGroupTiles = 64;               // tiles per expand CTA
constexpr int kStageRow = kSWarpElems + 8;    // per-warp staging row + trash slot
constexpr size_t kRingBytes = (size_t)kStages * kSTile * sizeof(double);

// ---------------------------------------------------------------------------
// TMA bulk copy + mbarrier helpers
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// One thread: expect `bytes` on `bar` and start the bulk copy global -> shared.
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t pol) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// Stage the tile's FP64 input in ring slot `s`: full tiles by TMA (issued
// ahead of time), the partial last tile by plain loads here.
struct Ring {
  double* xs;
  uint64_t* bars;
};

__device__ __forceinline__ const double* acquire_tile(const Ring& r, const double* x, int64_t n, int64_t t,
                                                      int64_t full_tiles, int s, uint32_t phase) {
  double* dst = r.xs + (size_t)s * kSTile;
  if (t < full_tiles) {
    mbar_wait(r.bars + s, phase);
  } else {
    const int64_t base = t * kSTile;
    for (int e = threadIdx.x; e < kSTile; e += kSThreads) dst[e] = (base + e < n) ? x[base + e] : 0.0;
    __syncthreads();
  }
  return dst;
}

__device__ __forceinline__ void issue_tile(const Ring& r, const double* x, int64_t t, int64_t full_tiles, int s,
                                           uint64_t pol) {
  if (t < full_tiles) tma_load(r.xs + (size_t)s * kSTile, x + t * kSTile, kSTile * sizeof(double), r.bars + s, pol);
}

// Output stores relative to the tile: `o` points at the tile's first output
// element, `lim` = valid elements in the tile (checked only when !FULL).
template <int OUT, bool FULL>
__device__ __forceinline__ void store2(void* o, int e0, int lim, float a, float b) {
  if (OUT == VT_OUT_F32) {
    float* p = static_cast<float*>(o) + e0;
    if (FULL || e0 + 1 < lim) {
      *reinterpret_cast<float2*>(p) = make_float2(a, b);
    } else if (e0 < lim) {
      p[0] = a;
    }
  } else if (OUT == VT_OUT_F64) {
    double* p = static_cast<double*>(o) + e0;
    if (FULL || e0 + 1 < lim) {
      *reinterpret_cast<double2*>(p) = make_double2((double)a, (double)b);
    } else if (e0 < lim) {
      p[0] = (double)a;
    }
  }
}

template <int OUT, bool FULL>
__device__ __forceinline__ void store2(void* o, int e0, int lim, uint64_t a, uint64_t b) {
  const double da = __longlong_as_double((long long)a), db = __longlong_as_double((long long)b);
  if (OUT == VT_OUT_F32) {
    store2<OUT, FULL>(o, e0, lim, __double2float_rn(da), __double2float_rn(db));
  } else if (OUT == VT_OUT_F64) {
    double* p = static_cast<double*>(o) + e0;
    if (FULL || e0 + 1 < lim) {
      *reinterpret_cast<double2*>(p) = make_double2(da, db);
    } else if (e0 < lim) {
      p[0] = da;
    }
  }
}

template <int OUT>
__device__ __forceinline__ void* tile_out(void* out, int64_t tbase) {
  if (OUT == VT_OUT_F32) return static_cast<float*>(out) + tbase;
  if (OUT == VT_OUT_F64) return static_cast<double*>(out) + tbase;
  return out;
}

// ---------------------------------------------------------------------------
// trainer: streaming pass
// ---------------------------------------------------------------------------

struct RLStreamArgs {
  const double* x;
  int64_t n;
  Grid g;
  int thr32;
  void* out;
  uint16_t* scratch;  // [num_tiles][kSTile] staged local entries
  uint32_t* counts;   // [num_tiles]
  int64_t num_tiles;
  int32_t* err;
};

// One tile of the trainer pass: round, classify, store, stage logged
// elements (warp-local order == element order).  Returns the warp's count.
template <int OUT, bool FAST, bool FULL>
__device__ __forceinline__ uint32_t rl_tile(const RLStreamArgs& a, const double* src, void* o, int lim,
                                            uint16_t* stw, int warp, int lane, uint32_t lt, uint32_t& err) {
  uint32_t wcnt = 0;
#pragma unroll
  for (int j = 0; j < kSSlots; ++j) {
    const int e0 = warp * kSWarpElems + j * 64 + lane * 2;
    const double2 xv = *reinterpret_cast<const double2*>(src + e0);
    uint32_t c0, c1;
    if (FAST) {
      bool slow = false;
      float f0 = round_dir32_fast(xv.x, a.thr32, c0, slow);
      float f1 = round_dir32_fast(xv.y, a.thr32, c1, slow);
      if (slow) {
        f0 = round_dir32(xv.x, a.thr32, a.g.thr_sub, c0, err);
        f1 = round_dir32(xv.y, a.thr32, a.g.thr_sub, c1, err);
      }
      store2<OUT, FULL>(o, e0, lim, f0, f1);
    } else {
      const uint64_t r0 = round_dir(xv.x, a.g, c0, err);
      const uint64_t r1 = round_dir(xv.y, a.g, c1, err);
      store2<OUT, FULL>(o, e0, lim, r0, r1);
    }
    const uint32_t b0 = __ballot_sync(0xffffffffu, c0 != 1u);
    const uint32_t b1 = __ballot_sync(0xffffffffu, c1 != 1u);
    // branch-free staging: unlogged elements write into the trash slot
    // (index kSWarpElems of this warp's stage row)
    const uint32_t r0 = wcnt + __popc(b0 & lt) + __popc(b1 & lt);
    const uint32_t r1 = r0 + (c0 != 1u);
    stw[(c0 != 1u) ? r0 : kSWarpElems] = (uint16_t)(e0 | ((c0 == 2u) ? 0x8000 : 0));
    stw[(c1 != 1u) ? r1 : kSWarpElems] = (uint16_t)((e0 + 1) | ((c1 == 2u) ? 0x8000 : 0));
    wcnt += __popc(b0) + __popc(b1);
  }
  return wcnt;
}

template <int OUT, bool FAST>
__global__ void __launch_bounds__(kSThreads, 3) rl_stream_kernel(const RLStreamArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[kStages];
  __shared__ uint32_t s_cnt[2][kWarps];
  Ring ring{reinterpret_cast<double*>(sm), bars};
  uint16_t* st16 = reinterpret_cast<uint16_t*>(sm + kRingBytes);  // [2][kWarps][kStageRow]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t full_tiles = a.n / kSTile;
  const uint64_t pol = evict_first_policy();
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(bars + s, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < kStages; ++s) issue_tile(ring, a.x, blockIdx.x + (int64_t)s * gridDim.x, full_tiles, s, pol);

  const uint32_t lt = lanemask_lt();
  uint32_t err = 0;
  for (int64_t k = 0;; ++k) {
    const int64_t t = blockIdx.x + k * gridDim.x;
    if (t >= a.num_tiles) break;
    const int s = (int)(k % kStages);
    const int buf = (int)(k & 1);
    const double* src = acquire_tile(ring, a.x, a.n, t, full_tiles, s, (uint32_t)((k / kStages) & 1));
    const int64_t tbase = t * kSTile;
    uint16_t* stw = st16 + (buf * kWarps + warp) * kStageRow;
    void* o = tile_out<OUT>(a.out, tbase);
    const uint32_t wcnt = (t < full_tiles)
        ? rl_tile<OUT, FAST, true>(a, src, o, kSTile, stw, warp, lane, lt, err)
        : rl_tile<OUT, FAST, false>(a, src, o, (int)(a.n - tbase), stw, warp, lane, lt, err);
    if (lane == 0) s_cnt[buf][warp] = wcnt;
    __syncthreads();  // ring slot s fully consumed; warp counts visible
    if (tid == 0) {
      fence_proxy_async();
      issue_tile(ring, a.x, t + (int64_t)kStages * gridDim.x, full_tiles, s, pol);
    }
    uint32_t off = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = s_cnt[buf][w];
      off += (w < warp) ? c : 0u;
      total += c;
    }
    uint16_t* dst = a.scratch + t * kSTile + off;
    for (uint32_t i = lane; i < wcnt; i += 32) dst[i] = stw[i];
    if (tid == 0) a.counts[t] = total;
  }
  report_err(a.err, err);
}

// ---------------------------------------------------------------------------
// trainer: expand staged entries into the global log
// ---------------------------------------------------------------------------

constexpr uint64_t kSFlagAgg = 1ull << 62;
constexpr uint64_t kSFlagInc = 2ull << 62;
constexpr uint64_t kSValMask = (1ull << 62) - 1;

struct ExpandArgs {
  const uint16_t* scratch;
  const uint32_t* counts;
  int64_t num_tiles;
  uint64_t* status;  // [num_groups], zeroed
  int64_t global_base;
  const int64_t* cursor_in;
  int64_t* cursor_out;
  uint64_t* sparse;
  int64_t cap;
  int64_t* counters;
};

__global__ void __launch_bounds__(kSThreads) rl_expand_kernel(const ExpandArgs a) {
  __shared__ uint32_t s_off[kGroupTiles + 1];
  __shared__ int64_t s_base;
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t group = blockIdx.x;  // 1-D grid: dispatched in order, look-back is safe
  const int64_t t0 = group * kGroupTiles;
  const int nt = (int)std::min<int64_t>(kGroupTiles, a.num_tiles - t0);
  if (tid < 32) {
    // exclusive scan of the group's (<= 64) tile counts by warp 0
    const uint32_t c0 = (lane < nt) ? a.counts[t0 + lane] : 0u;
    const uint32_t c1 = (lane + 32 < nt) ? a.counts[t0 + lane + 32] : 0u;
    uint32_t i0 = c0, i1 = c1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u0 = __shfl_up_sync(0xffffffffu, i0, o);
      const uint32_t u1 = __shfl_up_sync(0xffffffffu, i1, o);
      if (lane >= o) {
        i0 += u0;
        i1 += u1;
      }
    }
    const uint32_t tot0 = __shfl_sync(0xffffffffu, i0, 31);
    s_off[lane] = i0 - c0;
    s_off[lane + 32] = tot0 + i1 - c1;
    const uint64_t agg = (uint64_t)tot0 + __shfl_sync(0xffffffffu, i1, 31);
    if (lane == 0) s_off[kGroupTiles] = (uint32_t)agg;
    // decoupled look-back over groups, 32 predecessors per round trip
    int64_t excl = 0;
    if (group == 0) {
      if (lane == 0) st_relaxed_u64(a.status, kSFlagInc | agg);
    } else {
      if (lane == 0) st_relaxed_u64(a.status + group, kSFlagAgg | agg);
      int64_t pred = group - 1;
      while (true) {
        const int64_t idx = pred - lane;
        const uint64_t s = (idx >= 0) ? ld_relaxed_u64(a.status + idx) : kSFlagInc;
        const uint64_t flag = s >> 62;
        const uint32_t inc = __ballot_sync(0xffffffffu, flag == 2);
        const uint32_t inv = __ballot_sync(0xffffffffu, flag == 0);
        const int first = inc ? (__ffs(inc) - 1) : 31;
        const uint32_t upto = (2u << first) - 1u;
        if (inv & upto) {
          __nanosleep(16);
          continue;
        }
        uint64_t v = (lane <= first) ? (s & kSValMask) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += (int64_t)v;
        if (inc) break;
        pred -= 32;
      }
      if (lane == 0) st_relaxed_u64(a.status + group, kSFlagInc | ((uint64_t)excl + agg));
    }
    if (lane == 0) {
      const int64_t cur = a.cursor_in ? *a.cursor_in : 0;
      s_base = cur + excl;
      if (t0 + nt == a.num_tiles) {
        atomicAdd(reinterpret_cast<unsigned long long*>(a.counters), (unsigned long long)(excl + (int64_t)agg));
        if (a.cursor_out) *a.cursor_out = cur + excl + (int64_t)agg;
      }
    }
  }
  __syncthreads();
  const int64_t base = s_base;
  const int warp = tid >> 5;
  // one warp per tile, unrolled so several independent loads are in flight
  for (int k = warp; k < nt; k += kWarps) {
    const int64_t t = t0 + k;
    const uint32_t cnt = s_off[k + 1] - s_off[k];
    const uint16_t* src = a.scratch + t * kSTile;
    const int64_t out0 = base + s_off[k];
    const uint64_t w0 = (uint64_t)(a.global_base + t * kSTile) << 1;
    if (out0 + cnt <= a.cap) {
#pragma unroll 4
      for (uint32_t i = lane; i < cnt; i += 32) {
        const uint32_t e = __ldg(src + i);
        a.sparse[out0 + i] = w0 + ((uint64_t)(e & 0x7fffu) << 1) + (e >> 15);
      }
    } else {
      for (uint32_t i = lane; i < cnt; i += 32) {
        const uint32_t e = __ldg(src + i);
        if (out0 + i < a.cap) a.sparse[out0 + i] = w0 + ((uint64_t)(e & 0x7fffu) << 1) + (e >> 15);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// auditor: streaming replay against the sparse log
// ---------------------------------------------------------------------------

struct RPStreamArgs {
  const double* x;
  int64_t n;
  Grid g;
  const uint64_t* log;
  int64_t log_base;
  const int64_t* offs;  // [num_tiles + 1] word ranges per tile
  void* out;
  int64_t num_tiles;
  int64_t* counters;
  int32_t* err;
};

__global__ void rp_tile_offsets_kernel(const uint64_t* __restrict__ w, int64_t n_words, int64_t base, int64_t n,
                                       int64_t num_tiles, int64_t* __restrict__ offs, int64_t* counters) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > num_tiles) return;
  const int64_t key = base + std::min<int64_t>(t * kSTile, n);
  int64_t lo = 0, hi = n_words;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)(__ldg(w + mid) >> 1) < key) lo = mid + 1;
    else hi = mid;
  }
  offs[t] = lo;
  if (t == 0) counters[1] = lo;
  if (t == num_tiles) counters[2] = lo;
}

// One tile of the auditor pass.  Each thread reads the codes of its own
// elements from the map and resets them to 1, so the map is all-ignore
// again for the next tile without an extra barrier.
template <int OUT, bool FAST, bool FULL>
__device__ __forceinline__ uint32_t rp_tile(const RPStreamArgs& a, const double* src, uint8_t* cs, void* o,
                                            int lim, int warp, int lane, uint32_t& err) {
  uint32_t flips = 0;
#pragma unroll
  for (int j = 0; j < kSSlots; ++j) {
    const int e0 = warp * kSWarpElems + j * 64 + lane * 2;
    const double2 xv = *reinterpret_cast<const double2*>(src + e0);
    uint16_t* cp = reinterpret_cast<uint16_t*>(cs + e0);
    const uint32_t cc = *cp;
    *cp = 0x0101;
    const uint32_t c0 = cc & 0xffu, c1 = cc >> 8;
    uint32_t f0, f1;
    if (FAST) {
      bool slow = false;
      float y0 = replay32_fast(xv.x, c0, slow, f0);
      float y1 = replay32_fast(xv.y, c1, slow, f1);
      if (slow) {
        y0 = replay32(xv.x, c0, err, f0);
        y1 = replay32(xv.y, c1, err, f1);
      }
      store2<OUT, FULL>(o, e0, lim, y0, y1);
    } else {
      const uint64_t r0 = replay_one(xv.x, c0, a.g, err, f0);
      const uint64_t r1 = replay_one(xv.y, c1, a.g, err, f1);
      store2<OUT, FULL>(o, e0, lim, r0, r1);
    }
    flips += f0 + f1;
  }
  return flips;
}

__device__ __forceinline__ void scatter_entry(uint8_t* cs, uint64_t word, uint64_t prev, int64_t i, int64_t key0,
                                              uint32_t& err) {
  const int64_t idx = (int64_t)(word >> 1) - key0;
  const bool ordered = (i == 0) || ((prev >> 1) < (word >> 1));
  if (idx >= 0 && idx < kSTile && ordered) cs[idx] = (word & 1ull) ? 2 : 0;
  else err |= VT_ERR_BAD_SPARSE;
}

template <int OUT, bool FAST>
__global__ void __launch_bounds__(kSThreads, 3) rp_stream_kernel(const RPStreamArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[kStages];
  __shared__ uint32_t s_red[kWarps];
  Ring ring{reinterpret_cast<double*>(sm), bars};
  uint8_t* cs = sm + kRingBytes;  // [kSTile] code map, all 1 between tiles

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t full_tiles = a.n / kSTile;
  const uint64_t pol = evict_first_policy();
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(bars + s, 1);
    fence_mbar_init();
  }
  reinterpret_cast<uint2*>(cs)[tid] = make_uint2(0x01010101u, 0x01010101u);
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < kStages; ++s) issue_tile(ring, a.x, blockIdx.x + (int64_t)s * gridDim.x, full_tiles, s, pol);

  // Log prefetch pipeline: the word range of tile k+2 and the first 256
  // words (plus predecessors, for the order check) of tile k+1 are loaded
  // while tile k is processed.
  const int64_t G = gridDim.x;
  int64_t t0 = blockIdx.x;
  int64_t p_lo = 0, p_hi = 0, q_lo = 0, q_hi = 0;
  uint64_t p_w = 0, p_prev = 0;
  if (t0 < a.num_tiles) {
    p_lo = a.offs[t0];
    p_hi = a.offs[t0 + 1];
    const int64_t i = p_lo + tid;
    if (i < p_hi) {
      p_w = __ldg(a.log + i);
      p_prev = i ? __ldg(a.log + i - 1) : 0ull;
    }
  }
  if (t0 + G < a.num_tiles) {
    q_lo = a.offs[t0 + G];
    q_hi = a.offs[t0 + G + 1];
  }

  uint32_t err = 0, flips = 0;
  for (int64_t k = 0;; ++k) {
    const int64_t t = blockIdx.x + k * G;
    if (t >= a.num_tiles) break;
    const int s = (int)(k % kStages);
    const int64_t tbase = t * kSTile;
    const int64_t c_lo = p_lo, c_hi = p_hi;
    const uint64_t c_w = p_w, c_prev = p_prev;
    p_lo = q_lo;
    p_hi = q_hi;
    p_w = p_prev = 0;
    {
      const int64_t i = p_lo + tid;
      if (i < p_hi) {
        p_w = __ldg(a.log + i);
        p_prev = i ? __ldg(a.log + i - 1) : 0ull;
      }
    }
    if (t + 2 * G < a.num_tiles) {
      q_lo = a.offs[t + 2 * G];
      q_hi = a.offs[t + 2 * G + 1];
    }
    const int64_t key0 = a.log_base + tbase;
    int64_t i = c_lo + tid;
    if (i < c_hi) scatter_entry(cs, c_w, c_prev, i, key0, err);
    for (i += kSThreads; i < c_hi; i += kSThreads) scatter_entry(cs, __ldg(a.log + i), __ldg(a.log + i - 1), i, key0, err);
    const double* src = acquire_tile(ring, a.x, a.n, t, full_tiles, s, (uint32_t)((k / kStages) & 1));
    __syncthreads();  // code map complete, x tile resident
    void* o = tile_out<OUT>(a.out, tbase);
    flips += (t < full_tiles) ? rp_tile<OUT, FAST, true>(a, src, cs, o, kSTile, warp, lane, err)
                              : rp_tile<OUT, FAST, false>(a, src, cs, o, (int)(a.n - tbase), warp, lane, err);
    __syncthreads();  // ring slot s consumed, code map reset
    if (tid == 0) {
      fence_proxy_async();
      issue_tile(ring, a.x, t + (int64_t)kStages * G, full_tiles, s, pol);
    }
  }
  report_err(a.err, err);
  uint32_t v = flips;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  if (tid == 0) {
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) tot += s_red[w];
    if (tot) atomicAdd(reinterpret_cast<unsigned long long*>(a.counters), (unsigned long long)tot);
  }
}

// ---------------------------------------------------------------------------
// host launchers (called from vt_round.cu's C ABI)
// ---------------------------------------------------------------------------

int64_t stream_tiles(int64_t n) { return (n + kSTile - 1) / kSTile; }

size_t rl_stream_workspace(int64_t n) {
  const int64_t t = stream_tiles(n);
  const int64_t groups = (t + kGroupTiles - 1) / kGroupTiles;
  return (size_t)(groups * 8 + t * 4 + 256) + (size_t)t * kSTile * 2 + 256;
}

size_t rp_stream_workspace(int64_t n) { return (size_t)(stream_tiles(n) + 1) * 8 + 256; }

static int resident_ctas(const void* fn, size_t smem) {
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kSThreads, smem);
  return std::max(1, per) * sms;
}

template <int OUT, bool FAST>
static int launch_rl_stream(const RLStreamArgs& a, const ExpandArgs& e, cudaStream_t st) {
  const size_t smem = kRingBytes + 2 * kWarps * kStageRow * sizeof(uint16_t);
  auto k = rl_stream_kernel<OUT, FAST>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = (int)std::min<int64_t>(a.num_tiles, resident_ctas((const void*)k, smem));
  k<<<grid, kSThreads, smem, st>>>(a);
  int rc = vt_check_launch("rl_stream_kernel");
  if (rc) return rc;
  const int64_t groups = (a.num_tiles + kGroupTiles - 1) / kGroupTiles;
  rl_expand_kernel<<<(unsigned)groups, kSThreads, 0, st>>>(e);
  return vt_check_launch("rl_expand_kernel");
}

int rl_stream(const double* x, int64_t n, const Grid& g, int thr32, bool fast, int out_kind, void* out,
              uint64_t* sparse, int64_t cap, int64_t global_base, const int64_t* cursor_in, int64_t* cursor_out,
              int64_t* counters, int32_t* err, void* ws, cudaStream_t st) {
  const int64_t tiles = stream_tiles(n);
  const int64_t groups = (tiles + kGroupTiles - 1) / kGroupTiles;
  uint8_t* w = static_cast<uint8_t*>(ws);
  uint64_t* status = reinterpret_cast<uint64_t*>(w);
  uint32_t* counts = reinterpret_cast<uint32_t*>(w + groups * 8);
  uint16_t* scratch = reinterpret_cast<uint16_t*>(w + ((groups * 8 + tiles * 4 + 255) & ~(int64_t)255));
  if (cudaMemsetAsync(status, 0, (size_t)groups * 8, st) != cudaSuccess) return vt_check_launch("memset");
  RLStreamArgs a{x, n, g, thr32, out, scratch, counts, tiles, err};
  ExpandArgs e{scratch, counts, tiles, status, global_base, cursor_in, cursor_out, sparse, cap, counters};
  if (fast) {
    return out_kind == VT_OUT_F32 ? launch_rl_stream<VT_OUT_F32, true>(a, e, st)
         : out_kind == VT_OUT_F64 ? launch_rl_stream<VT_OUT_F64, true>(a, e, st)
                                  : launch_rl_stream<VT_OUT_NONE, true>(a, e, st);
  }
  return out_kind == VT_OUT_F32 ? launch_rl_stream<VT_OUT_F32, false>(a, e, st)
       : out_kind == VT_OUT_F64 ? launch_rl_stream<VT_OUT_F64, false>(a, e, st)
                                : launch_rl_stream<VT_OUT_NONE, false>(a, e, st);
}

template <int OUT, bool FAST>
static int launch_rp_stream(const RPStreamArgs& a, cudaStream_t st) {
  const size_t smem = kRingBytes + kSTile;
  auto k = rp_stream_kernel<OUT, FAST>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = (int)std::min<int64_t>(a.num_tiles, resident_ctas((const void*)k, smem));
  k<<<grid, kSThreads, smem, st>>>(a);
  return vt_check_launch("rp_stream_kernel");
}

int rp_stream(const double* x, int64_t n, const Grid& g, bool fast, int out_kind, void* out, const uint64_t* log,
              int64_t n_words, int64_t log_base, int64_t* counters, int32_t* err, void* ws, cudaStream_t st) {
  const int64_t tiles = stream_tiles(n);
  int64_t* offs = static_cast<int64_t*>(ws);
  rp_tile_offsets_kernel<<<(unsigned)((tiles + 1 + 255) / 256), 256, 0, st>>>(log, n_words, log_base, n, tiles, offs,
                                                                              counters);
  int rc = vt_check_launch("rp_tile_offsets_kernel");
  if (rc) return rc;
  RPStreamArgs a{x, n, g, log, log_base, offs, out, tiles, counters, err};
  if (fast) {
    return out_kind == VT_OUT_F32 ? launch_rp_stream<VT_OUT_F32, true>(a, st)
         : out_kind == VT_OUT_F64 ? launch_rp_stream<VT_OUT_F64, true>(a, st)
                                  : launch_rp_stream<VT_OUT_NONE, true>(a, st);
  }
  return out_kind == VT_OUT_F32 ? launch_rp_stream<VT_OUT_F32, false>(a, st)
       : out_kind == VT_OUT_F64 ? launch_rp_stream<VT_OUT_F64, false>(a, st)
                                : launch_rp_stream<VT_OUT_NONE, false>(a, st);
}

}  // namespace vt
