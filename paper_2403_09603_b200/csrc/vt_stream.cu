// Persistent, TMA-pipelined streaming kernels for the north-star path
// (sparse log, FP32 / FP64 output):
//
//   rl_stream_kernel   trainer round-and-log (protocol._TrainerChannel.process,
//                      pkg/src/vtrain/protocol.py:198-202) -- rounds every element,
//                      and stages each tile's logged elements as 16-bit local
//                      entries (11-bit offset | up << 15) + a per-tile count;
//   rl_scan_kernel     block-level decoupled look-back prefix sum over the tile
//                      counts (the global log position of every tile);
//   rl_expand_kernel   expands the staged entries into the global ascending
//                      uint64 log (global_index << 1 | up);
//   rp_fused_kernel    auditor replay (protocol._AuditorChannel.process,
//                      protocol.py:212-216) -- scatters the tile's log slice into a
//                      shared-memory code map and replays every element.
//
// Streaming CTAs are persistent (grid = resident CTAs): the trainer walks
// tiles blockIdx.x, blockIdx.x + gridDim.x, ..., the auditor a contiguous
// range of tiles; the FP64 input of the next kStages tiles is in flight at
// all times through cp.async.bulk (TMA bulk copies, L2 evict-first) into a
// shared-memory ring guarded by mbarriers, so HBM streams continuously while
// the SM computes.  No CTA ever waits on another CTA in a streaming pass; the
// only cross-CTA wait is the look-back of the small scan pass.  (A single-
// launch variant that resolves each tile's log position a few waves later
// from epoch-tagged tile counts was measured 12-20% slower and dropped.)
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
// cross-CTA decoupled look-back with epoch-tagged status words
//
// status word = epoch (20 bits) | flag (2 bits) | value (42 bits).  A word
// whose epoch differs from the current call's is "not yet published", so the
// status array never needs clearing between calls: the workspace header keeps
// the epoch, every CTA reads it at start, and the last CTA bumps it after its
// own look-back (which completes only after every other CTA has published,
// hence after every CTA has read the old epoch).
// ---------------------------------------------------------------------------

constexpr int kEpochShift = 44;
constexpr uint64_t kEpochMask = (1ull << 20) - 1;
constexpr uint64_t kLBAgg = 1ull << 42;
constexpr uint64_t kLBInc = 2ull << 42;
constexpr uint64_t kLBVal = (1ull << 42) - 1;

struct WsHeader {
  uint32_t epoch;
  uint32_t pad[15];
};

__device__ __forceinline__ uint64_t lb_word(uint32_t epoch, uint64_t flag, uint64_t v) {
  return ((uint64_t)epoch << kEpochShift) | flag | (v & kLBVal);
}

// ---------------------------------------------------------------------------
// trainer: streaming pass (strided persistent tiles) + expand pass
// ---------------------------------------------------------------------------

struct RLArgs {
  const double* x;
  int64_t n;
  Grid g;
  int thr32;
  void* out;
  int64_t num_tiles;
  uint32_t* counts;   // [num_tiles] logged entries per tile
  uint16_t* scratch;  // [num_tiles][kSTile] staged entries: tile offset | up << 15
  int32_t* err;
  const DevThr* dthr;  // adaptive path: thresholds from the device bisection
};

// One tile: round, classify, store, stage logged elements (warp-local order
// == element order).  Returns the warp's count.
template <int OUT, bool FAST, bool FULL>
__device__ __forceinline__ uint32_t rl_tile(const Grid& g, int thr32, const double* src, void* o, int lim,
                                            uint16_t* stw, int warp, int lane, uint32_t lt, uint32_t& err) {
  uint32_t wcnt = 0;
  const int eb = warp * kSWarpElems + lane * 2;  // this lane's first element in the tile
  const uint32_t st_base = smem_u32(stw);       // shared-window address of the warp's stage row
  const uint32_t trash = st_base + 2u * kSWarpElems;
#pragma unroll
  for (int j = 0; j < kSSlots; ++j) {
    const int e0 = eb + j * 64;
    const double2 xv = *reinterpret_cast<const double2*>(src + e0);
    uint32_t c0, c1;
    if (FAST) {
      bool slow = false;
      float f0 = round_dir32_fast(xv.x, thr32, c0, slow);
      float f1 = round_dir32_fast(xv.y, thr32, c1, slow);
      if (slow) {
        f0 = round_dir32(xv.x, thr32, g.thr_sub, c0, err);
        f1 = round_dir32(xv.y, thr32, g.thr_sub, c1, err);
      }
      store2<OUT, FULL>(o, e0, lim, f0, f1);
    } else {
      const uint64_t r0 = round_dir(xv.x, g, c0, err);
      const uint64_t r1 = round_dir(xv.y, g, c1, err);
      store2<OUT, FULL>(o, e0, lim, r0, r1);
    }
    const bool l0 = c0 != 1u, l1 = c1 != 1u;
    const uint32_t b0 = __ballot_sync(0xffffffffu, l0);
    const uint32_t b1 = __ballot_sync(0xffffffffu, l1);
    // branch-free staging: unlogged elements write into the trash slot
    const uint32_t r0 = wcnt + __popc(b0 & lt) + __popc(b1 & lt);
    const uint32_t a0 = l0 ? st_base + 2u * r0 : trash;
    const uint32_t a1 = l1 ? st_base + 2u * (r0 + (l0 ? 1u : 0u)) : trash;
    const uint32_t v0 = (uint32_t)e0 | ((c0 == 2u) ? 0x8000u : 0u);
    const uint32_t v1 = (uint32_t)(e0 + 1) | ((c1 == 2u) ? 0x8000u : 0u);
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a0), "h"((uint16_t)v0) : "memory");
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(a1), "h"((uint16_t)v1) : "memory");
    wcnt += __popc(b0) + __popc(b1);
  }
  return wcnt;
}

// Tiles t = blockIdx.x + k * gridDim.x: at any moment the CTAs of the grid
// stream one contiguous window of x.  No cross-CTA waits.
template <int OUT, bool FAST>
__global__ void __launch_bounds__(kSThreads, 3) rl_stream_kernel(const RLArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[kStages];
  __shared__ uint32_t s_cnt[2][kWarps];
  Ring ring{reinterpret_cast<double*>(sm), bars};
  uint16_t* st16 = reinterpret_cast<uint16_t*>(sm + kRingBytes);  // [2][kWarps][kStageRow]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t G = gridDim.x;
  const int64_t full_tiles = a.n / kSTile;
  const uint64_t pol = evict_first_policy();
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(bars + s, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < kStages; ++s) issue_tile(ring, a.x, blockIdx.x + s * G, full_tiles, s, pol);

  const uint32_t lt = lanemask_lt();
  uint32_t err = 0;
  Grid g = a.g;
  int thr32 = a.thr32;
  if (a.dthr) {  // adaptive: tau was bisected on the device
    g.thr = a.dthr->thr;
    g.thr_sub = a.dthr->thr_sub;
    thr32 = a.dthr->thr32;
  }
  for (int64_t k = 0;; ++k) {
    const int64_t t = blockIdx.x + k * G;
    if (t >= a.num_tiles) break;
    const int s = (int)(k % kStages);
    const int buf = (int)(k & 1);
    const double* src = acquire_tile(ring, a.x, a.n, t, full_tiles, s, (uint32_t)((k / kStages) & 1));
    const int64_t tbase = t * kSTile;
    uint16_t* stw = st16 + (buf * kWarps + warp) * kStageRow;
    void* o = tile_out<OUT>(a.out, tbase);
    const uint32_t wcnt = (t < full_tiles)
        ? rl_tile<OUT, FAST, true>(g, thr32, src, o, kSTile, stw, warp, lane, lt, err)
        : rl_tile<OUT, FAST, false>(g, thr32, src, o, (int)(a.n - tbase), stw, warp, lane, lt, err);
    if (lane == 0) s_cnt[buf][warp] = wcnt;
    __syncthreads();  // ring slot s consumed; warp counts visible
    if (tid == 0) {
      fence_proxy_async();
      issue_tile(ring, a.x, t + kStages * G, full_tiles, s, pol);
    }
    uint32_t off = 0, total = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t c = s_cnt[buf][w];
      off += (w < warp) ? c : 0u;
      total += c;
    }
    uint16_t* dst = a.scratch + tbase + off;
    for (uint32_t i = lane; i < wcnt; i += 32) dst[i] = stw[i];
    if (tid == 0) a.counts[t] = total;
  }
  report_err(a.err, err);
}

// Scan: exclusive prefix of the per-tile counts by single-pass decoupled
// look-back (CTA per kScanTiles counts), giving every tile the global log
// position of its first entry.
constexpr int kScanPer = 8;                        // counts per thread
constexpr int kScanTiles = kSThreads * kScanPer;  // 2048 counts per CTA

struct ScanArgs {
  const uint32_t* counts;
  int64_t num_tiles;
  WsHeader* hdr;
  uint64_t* status;  // [num_scan_ctas] epoch-tagged
  int64_t* toffs;    // [num_tiles] global log position of each tile's entries
  const int64_t* cursor_in;
  int64_t* cursor_out;
  int64_t* counters;
};

__global__ void __launch_bounds__(kSThreads) rl_scan_kernel(const ScanArgs a) {
  __shared__ uint32_t s_warp[kWarps];
  __shared__ int64_t s_base;
  __shared__ uint32_t s_epoch;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t chunk = blockIdx.x;  // 1-D grid: dispatched in order, look-back is safe
  const int64_t t0 = chunk * kScanTiles + (int64_t)tid * kScanPer;
  uint32_t c[kScanPer];
  uint32_t sum = 0;
#pragma unroll
  for (int m = 0; m < kScanPer; ++m) {
    c[m] = (t0 + m < a.num_tiles) ? a.counts[t0 + m] : 0u;
    sum += c[m];
  }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) s_warp[warp] = inc;
  if (tid == 0) s_epoch = ((*(volatile uint32_t*)&a.hdr->epoch) + 1u) & (uint32_t)kEpochMask;
  __syncthreads();
  uint32_t wpre = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    wpre += (w < warp) ? s_warp[w] : 0u;
    agg += s_warp[w];
  }
  const uint32_t epoch = s_epoch;
  if (warp == 0) {
    int64_t excl = 0;
    if (chunk == 0) {
      if (lane == 0) st_relaxed_u64(a.status, lb_word(epoch, kLBInc, agg));
    } else {
      if (lane == 0) st_relaxed_u64(a.status + chunk, lb_word(epoch, kLBAgg, agg));
      int64_t pred = chunk - 1;
      while (true) {
        const int64_t idx = pred - lane;
        uint64_t s = lb_word(epoch, kLBInc, 0);
        if (idx >= 0) s = ld_relaxed_u64(a.status + idx);
        const bool valid = ((s >> kEpochShift) & kEpochMask) == epoch;
        const uint64_t flag = valid ? ((s >> 42) & 3ull) : 0ull;
        const uint32_t incm = __ballot_sync(0xffffffffu, flag == 2);
        const uint32_t inv = __ballot_sync(0xffffffffu, flag == 0);
        const int first = incm ? (__ffs(incm) - 1) : 31;
        const uint32_t upto = (2u << first) - 1u;
        if (inv & upto) {
          __nanosleep(32);
          continue;
        }
        uint64_t v = (lane <= first) ? (s & kLBVal) : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += (int64_t)v;
        if (incm) break;
        pred -= 32;
      }
      if (lane == 0) st_relaxed_u64(a.status + chunk, lb_word(epoch, kLBInc, (uint64_t)excl + agg));
    }
    if (lane == 0) {
      const int64_t cur = a.cursor_in ? *a.cursor_in : 0;
      s_base = cur + excl;
      if ((chunk + 1) * kScanTiles >= a.num_tiles) {
        atomicAdd(reinterpret_cast<unsigned long long*>(a.counters), (unsigned long long)(excl + (int64_t)agg));
        if (a.cursor_out) *a.cursor_out = cur + excl + (int64_t)agg;
        *(volatile uint32_t*)&a.hdr->epoch = epoch;
      }
    }
  }
  __syncthreads();
  int64_t off = s_base + wpre + (inc - sum);
#pragma unroll
  for (int m = 0; m < kScanPer; ++m) {
    if (t0 + m < a.num_tiles) a.toffs[t0 + m] = off;
    off += c[m];
  }
}

// Expand: warp per tile, no waits -- the staged 16-bit entries become
// global (index << 1 | up) words at the tile's scanned position.
constexpr int kExpTilesPerCta = kWarps;

struct ExpandArgs {
  const uint16_t* scratch;
  const uint32_t* counts;
  const int64_t* toffs;
  int64_t num_tiles;
  int64_t global_base;
  uint64_t* sparse;
  int64_t cap;
};

__global__ void __launch_bounds__(kSThreads) rl_expand_kernel(const ExpandArgs a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t t = (int64_t)blockIdx.x * kExpTilesPerCta + warp;
  if (t >= a.num_tiles) return;
  const uint32_t cnt = a.counts[t];
  const int64_t out0 = a.toffs[t];
  const uint16_t* src = a.scratch + t * kSTile;
  const uint64_t w0 = (uint64_t)(a.global_base + t * kSTile) << 1;
  if (out0 + cnt <= a.cap) {
    for (uint32_t i0 = 0; i0 < cnt; i0 += 4 * 32) {
      uint32_t e[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = i0 + u * 32 + lane;
        e[u] = (i < cnt) ? (uint32_t)__ldg(src + i) : 0u;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = i0 + u * 32 + lane;
        if (i < cnt) a.sparse[out0 + i] = w0 + ((uint64_t)(e[u] & 0x7fffu) << 1) + (e[u] >> 15);
      }
    }
  } else {
    for (uint32_t i = lane; i < cnt; i += 32) {
      const uint32_t e = __ldg(src + i);
      if (out0 + i < a.cap) a.sparse[out0 + i] = w0 + ((uint64_t)(e & 0x7fffu) << 1) + (e >> 15);
    }
  }
}

// ---------------------------------------------------------------------------
// auditor: streaming replay against the sparse log
// ---------------------------------------------------------------------------

struct RPArgs {
  const double* x;
  int64_t n;
  Grid g;
  const uint64_t* log;
  int64_t n_words;
  int64_t log_base;
  void* out;
  int64_t num_tiles;
  int64_t tiles_per_cta;
  int64_t* counters;
  int32_t* err;
};

// lower_bound over the sorted word indices by one warp, 32 probes per step
__device__ int64_t warp_lower_bound(const uint64_t* w, int64_t n, int64_t key, int lane) {
  int64_t lo = 0, hi = n;  // answer in [lo, hi]
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t p = lo + lane * step;
    const bool lt = (p < hi) && ((int64_t)(__ldg(w + p) >> 1) < key);
    const int c = __popc(__ballot_sync(0xffffffffu, lt));
    if (c == 0) return lo;
    const int64_t nlo = lo + (int64_t)(c - 1) * step + 1;
    hi = std::min<int64_t>(hi, lo + (int64_t)c * step);
    lo = nlo;
  }
  const int64_t p = lo + lane;
  const bool lt = (p < hi) && ((int64_t)(__ldg(w + p) >> 1) < key);
  return lo + __popc(__ballot_sync(0xffffffffu, lt));
}

// One tile of the auditor pass.  Each thread reads the codes of its own
// elements from the map and resets them to 1, so the map is all-ignore
// again for the next tile without an extra barrier.
template <int OUT, bool FAST, bool FULL>
__device__ __forceinline__ uint32_t rp_tile(const RPArgs& a, const double* src, uint8_t* cs, void* o, int lim,
                                            int warp, int lane, uint32_t& err) {
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

// Consume this tile's log words from the window [cur, cur + kSThreads)
// (prefetched in w/prev), scatter them into the code map; returns how many
// words belonged to the tile.  Entries must be a sorted prefix of the window.
__device__ __forceinline__ int scatter_window(uint8_t* cs, uint64_t w, uint64_t prev, int64_t i, int64_t n_words,
                                              int64_t key0, int64_t key1, uint32_t& err) {
  const bool have = i < n_words;
  const int64_t idx = (int64_t)(w >> 1);
  const bool in = have && idx < key1;
  const int cnt = __syncthreads_count(in);
  if (in) {
    const bool ordered = (i == 0) || ((prev >> 1) < (w >> 1));
    if (idx >= key0 && ordered && (int)threadIdx.x < cnt) cs[idx - key0] = (w & 1ull) ? 2 : 0;
    else err |= VT_ERR_BAD_SPARSE;
  }
  return cnt;
}

template <int OUT, bool FAST>
__global__ void __launch_bounds__(kSThreads, 3) rp_fused_kernel(const RPArgs a) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bars[kStages];
  __shared__ uint32_t s_red[kWarps];
  __shared__ int64_t s_lo;
  Ring ring{reinterpret_cast<double*>(sm), bars};
  uint8_t* cs = sm + kRingBytes;  // [kSTile] code map, all 1 between tiles

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t T0 = (int64_t)blockIdx.x * a.tiles_per_cta;
  const int64_t T1 = std::min<int64_t>(T0 + a.tiles_per_cta, a.num_tiles);
  const int64_t full_tiles = a.n / kSTile;
  const uint64_t pol = evict_first_policy();
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(bars + s, 1);
    fence_mbar_init();
  }
  reinterpret_cast<uint2*>(cs)[tid] = make_uint2(0x01010101u, 0x01010101u);
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < kStages && T0 + s < T1; ++s) issue_tile(ring, a.x, T0 + s, full_tiles, s, pol);
  if (warp == 0) {
    const int64_t lo = warp_lower_bound(a.log, a.n_words, a.log_base + T0 * kSTile, lane);
    if (lane == 0) s_lo = lo;
  }
  __syncthreads();
  int64_t cur = s_lo;  // first log word of the current tile (block-uniform)
  if (blockIdx.x == 0 && tid == 0) a.counters[1] = cur;
  uint64_t pw = 0, pp = 0;
  {
    const int64_t i = cur + tid;
    if (i < a.n_words) {
      pw = __ldg(a.log + i);
      pp = i ? __ldg(a.log + i - 1) : 0ull;
    }
  }

  uint32_t err = 0, flips = 0;
  for (int64_t t = T0; t < T1; ++t) {
    const int64_t k = t - T0;
    const int s = (int)(k % kStages);
    const int64_t tbase = t * kSTile;
    const int64_t key0 = a.log_base + tbase;
    const int64_t key1 = a.log_base + std::min<int64_t>(tbase + kSTile, a.n);
    int cnt = scatter_window(cs, pw, pp, cur + tid, a.n_words, key0, key1, err);
    cur += cnt;
    while (cnt == kSThreads) {  // more than one window of entries in this tile
      const int64_t i = cur + tid;
      uint64_t w = 0, p = 0;
      if (i < a.n_words) {
        w = __ldg(a.log + i);
        p = __ldg(a.log + i - 1);
      }
      cnt = scatter_window(cs, w, p, i, a.n_words, key0, key1, err);
      cur += cnt;
    }
    {  // prefetch the next tile's window while this tile computes
      const int64_t i = cur + tid;
      pw = pp = 0;
      if (i < a.n_words) {
        pw = __ldg(a.log + i);
        pp = i ? __ldg(a.log + i - 1) : 0ull;
      }
    }
    const double* src = acquire_tile(ring, a.x, a.n, t, full_tiles, s, (uint32_t)((k / kStages) & 1));
    __syncthreads();  // code map complete, x tile resident
    void* o = tile_out<OUT>(a.out, tbase);
    flips += (t < full_tiles) ? rp_tile<OUT, FAST, true>(a, src, cs, o, kSTile, warp, lane, err)
                              : rp_tile<OUT, FAST, false>(a, src, cs, o, (int)(a.n - tbase), warp, lane, err);
    __syncthreads();  // ring slot s consumed, code map reset
    if (tid == 0 && t + kStages < T1) {
      fence_proxy_async();
      issue_tile(ring, a.x, t + kStages, full_tiles, s, pol);
    }
  }
  if (blockIdx.x == gridDim.x - 1 && tid == 0) a.counters[2] = cur;
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

// [header 64 B][status: scan CTAs x 8][counts: T x 4][toffs: T x 8][scratch: T x kSTile x 2]
size_t rl_stream_workspace(int64_t n) {
  const int64_t t = stream_tiles(n);
  const int64_t chunks = (t + kScanTiles - 1) / kScanTiles;
  return (size_t)(64 + chunks * 8 + t * 12 + 512) + (size_t)t * kSTile * 2 + 256;
}

size_t rp_stream_workspace(int64_t n) {
  (void)n;
  return 0;
}

static int resident_ctas(const void* fn, size_t smem) {
  int dev = 0, sms = 148, per = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, kSThreads, smem);
  return std::max(1, per * sms);
}

template <int OUT, bool FAST>
static int launch_rl(const RLArgs& a, const ScanArgs& sc, const ExpandArgs& e, cudaStream_t st) {
  const size_t smem = kRingBytes + 2 * kWarps * kStageRow * sizeof(uint16_t);
  auto k = rl_stream_kernel<OUT, FAST>;
  static int resident = 0;  // one process per GPU: attribute + occupancy queried once
  if (!resident) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    resident = resident_ctas((const void*)k, smem);
  }
  const int grid = (int)std::min<int64_t>(a.num_tiles, resident);
  k<<<grid, kSThreads, smem, st>>>(a);
  int rc = vt_check_launch("rl_stream_kernel");
  if (rc) return rc;
  const int64_t chunks = (a.num_tiles + kScanTiles - 1) / kScanTiles;
  rl_scan_kernel<<<(unsigned)chunks, kSThreads, 0, st>>>(sc);
  if ((rc = vt_check_launch("rl_scan_kernel"))) return rc;
  const int64_t ectas = (a.num_tiles + kExpTilesPerCta - 1) / kExpTilesPerCta;
  rl_expand_kernel<<<(unsigned)ectas, kSThreads, 0, st>>>(e);
  return vt_check_launch("rl_expand_kernel");
}

int rl_stream(const double* x, int64_t n, const Grid& g, int thr32, bool fast, int out_kind, void* out,
              uint64_t* sparse, int64_t cap, int64_t global_base, const int64_t* cursor_in, int64_t* cursor_out,
              int64_t* counters, int32_t* err, void* ws, cudaStream_t st, const DevThr* dthr) {
  const int64_t tiles = stream_tiles(n);
  const int64_t chunks = (tiles + kScanTiles - 1) / kScanTiles;
  uint8_t* w = static_cast<uint8_t*>(ws);
  WsHeader* hdr = reinterpret_cast<WsHeader*>(w);
  uint64_t* status = reinterpret_cast<uint64_t*>(w + 64);
  int64_t* toffs = reinterpret_cast<int64_t*>(w + ((64 + chunks * 8 + 255) & ~(int64_t)255));
  uint32_t* counts = reinterpret_cast<uint32_t*>(toffs + tiles);
  uint16_t* scratch = reinterpret_cast<uint16_t*>(
      w + ((((64 + chunks * 8 + 255) & ~(int64_t)255) + tiles * 12 + 255) & ~(int64_t)255));
  RLArgs a{x, n, g, thr32, out, tiles, counts, scratch, err, dthr};
  ScanArgs sc{counts, tiles, hdr, status, toffs, cursor_in, cursor_out, counters};
  ExpandArgs e{scratch, counts, toffs, tiles, global_base, sparse, cap};
  if (fast) {
    return out_kind == VT_OUT_F32 ? launch_rl<VT_OUT_F32, true>(a, sc, e, st)
         : out_kind == VT_OUT_F64 ? launch_rl<VT_OUT_F64, true>(a, sc, e, st)
                                  : launch_rl<VT_OUT_NONE, true>(a, sc, e, st);
  }
  return out_kind == VT_OUT_F32 ? launch_rl<VT_OUT_F32, false>(a, sc, e, st)
       : out_kind == VT_OUT_F64 ? launch_rl<VT_OUT_F64, false>(a, sc, e, st)
                                : launch_rl<VT_OUT_NONE, false>(a, sc, e, st);
}

template <typename Args>
static void split_tiles(Args& a, int resident) {
  const int64_t grid = std::min<int64_t>(a.num_tiles, resident);
  a.tiles_per_cta = (a.num_tiles + grid - 1) / grid;
}

template <int OUT, bool FAST>
static int launch_rp(RPArgs a, cudaStream_t st) {
  const size_t smem = kRingBytes + kSTile;
  auto k = rp_fused_kernel<OUT, FAST>;
  static int resident = 0;
  if (!resident) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    resident = resident_ctas((const void*)k, smem);
  }
  split_tiles(a, resident);
  const int grid = (int)((a.num_tiles + a.tiles_per_cta - 1) / a.tiles_per_cta);
  k<<<grid, kSThreads, smem, st>>>(a);
  return vt_check_launch("rp_fused_kernel");
}

int rp_stream(const double* x, int64_t n, const Grid& g, bool fast, int out_kind, void* out, const uint64_t* log,
              int64_t n_words, int64_t log_base, int64_t* counters, int32_t* err, void* ws, cudaStream_t st) {
  (void)ws;
  RPArgs a{x, n, g, log, n_words, log_base, out, stream_tiles(n), 1, counters, err};
  if (fast) {
    return out_kind == VT_OUT_F32 ? launch_rp<VT_OUT_F32, true>(a, st)
         : out_kind == VT_OUT_F64 ? launch_rp<VT_OUT_F64, true>(a, st)
                                  : launch_rp<VT_OUT_NONE, true>(a, st);
  }
  return out_kind == VT_OUT_F32 ? launch_rp<VT_OUT_F32, false>(a, st)
       : out_kind == VT_OUT_F64 ? launch_rp<VT_OUT_F64, false>(a, st)
                                : launch_rp<VT_OUT_NONE, false>(a, st);
}

}  // namespace vt
