// Fused round-and-log (trainer) and replay (auditor) streaming kernels.
//
// round_log_kernel replaces protocol._TrainerChannel.process
// (pkg/src/vtrain/protocol.py:198-202): direction_array + LogWriter.write_array
// + rnd_array in ONE pass over the FP64 input.  replay_kernel replaces
// protocol._AuditorChannel.process (protocol.py:212-216): LogReader.read_array
// + rev_array + the correction count in ONE pass.
//
// HBM layout per call (element i of a contiguous FP64 tensor):
//   x[i]        FP64, read once with 256-bit L1::no_allocate loads
//   out[i]      FP32 (north-star form) or FP64 (drop-in form), 128/256-bit stores
//   sparse log  uint64 words (global_index << 1) | up, ascending, 8 B per logged element
//   codes[i]    optional uint8 ternary code
//   packed      optional .vtrl payload, 5 codes per byte
//
// The sparse log is emitted in index order by a single-pass decoupled
// look-back scan: each CTA publishes its tile's aggregate count and warp 0
// walks back over predecessors 32 at a time.
// Flag and value share one 64-bit word, so relaxed loads/stores suffice.
#include <algorithm>

#include "vt_common.cuh"

namespace vt {

constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

struct RoundLogArgs {
  const double* x;
  int64_t n;
  Grid g;
  void* out;
  uint64_t* sparse;
  int64_t sparse_cap;
  int64_t global_base;
  const int64_t* cursor_in;
  int64_t* cursor_out;
  uint8_t* codes;
  uint8_t* packed;
  int64_t head;   // elements before the first full .vtrl group
  int64_t nfull;  // full groups emitted by this call
  uint8_t* edge;  // head codes then tail codes (<= 8)
  int64_t* counters;
  int32_t* err;
  uint64_t* status;
  int64_t num_tiles;
  int thr32;  // b_r = 32 fast path: clamp(g.thr, 0, INT32_MAX)
};

__device__ __forceinline__ void load_slots(const double* __restrict__ x, int64_t n, int64_t wbase,
                                           int lane, D4 (&xv)[kSlots]) {
#pragma unroll
  for (int j = 0; j < kSlots; ++j) {
    const int64_t i0 = wbase + j * 128 + lane * 4;
    if (i0 + 3 < n) {
      xv[j] = ldg_stream4(x + i0);
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v) xv[j].v[v] = (i0 + v < n) ? x[i0 + v] : 0.0;
    }
  }
}

template <int OUT>
__device__ __forceinline__ void store_out(void* out, int64_t i0, int64_t n, const uint64_t (&rb)[4]) {
  if (OUT == VT_OUT_F32) {
    float* o = static_cast<float*>(out);
    float f[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) f[v] = __double2float_rn(__longlong_as_double((long long)rb[v]));
    if (i0 + 3 < n) {
      stg_stream4f(o + i0, f[0], f[1], f[2], f[3]);
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (i0 + v < n) o[i0 + v] = f[v];
    }
  } else if (OUT == VT_OUT_F64) {
    double* o = static_cast<double*>(out);
    double d[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) d[v] = __longlong_as_double((long long)rb[v]);
    if (i0 + 3 < n) {
      stg_stream4(o + i0, d[0], d[1], d[2], d[3]);
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (i0 + v < n) o[i0 + v] = d[v];
    }
  }
}

// FP32-valued results (b_r = 32 fast path)
template <int OUT>
__device__ __forceinline__ void store_out(void* out, int64_t i0, int64_t n, const float (&f)[4]) {
  if (OUT == VT_OUT_F32) {
    float* o = static_cast<float*>(out);
    if (i0 + 3 < n) {
      stg_stream4f(o + i0, f[0], f[1], f[2], f[3]);
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (i0 + v < n) o[i0 + v] = f[v];
    }
  } else if (OUT == VT_OUT_F64) {
    double* o = static_cast<double*>(out);
    if (i0 + 3 < n) {
      stg_stream4(o + i0, (double)f[0], (double)f[1], (double)f[2], (double)f[3]);
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (i0 + v < n) o[i0 + v] = (double)f[v];
    }
  }
}

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Decoupled look-back by the whole CTA: every thread reads one predecessor
// status word, so one L2 round trip covers 256 predecessors.  Returns the
// exclusive prefix of `tile` (all threads).  Called by all threads.
__device__ __forceinline__ int64_t lookback(uint64_t* status, int64_t tile, uint64_t agg) {
  __shared__ int s_first;
  __shared__ unsigned long long s_part[kWarps];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tile == 0) {
    if (tid == 0) st_relaxed_u64(status, kFlagInc | agg);
    return 0;
  }
  if (tid == 0) st_relaxed_u64(status + tile, kFlagAgg | agg);
  int64_t excl = 0;
  int64_t pred = tile - 1;
  while (true) {
    if (tid == 0) s_first = kThreads;
    __syncthreads();
    const int64_t idx = pred - tid;
    const uint64_t s = (idx >= 0) ? ld_relaxed_u64(status + idx) : kFlagInc;
    const uint64_t flag = s >> 62;
    const uint32_t inc = __ballot_sync(0xffffffffu, flag == 2);
    if (lane == 0 && inc) atomicMin(&s_first, warp * 32 + __ffs(inc) - 1);
    __syncthreads();
    const int first = s_first;  // nearest predecessor holding an inclusive prefix
    if (__syncthreads_or(flag == 0 && tid <= first)) {
      __nanosleep(32);
      continue;  // some needed predecessor has not published yet
    }
    uint64_t v = (tid <= first) ? (s & kValMask) : 0ull;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s_part[warp] = v;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kWarps; ++k) excl += (int64_t)s_part[k];
    if (first < kThreads) break;
    pred -= kThreads;
  }
  if (tid == 0) st_relaxed_u64(status + tile, kFlagInc | ((uint64_t)excl + agg));
  return excl;
}

template <int OUT, bool SPARSE, bool CODES, bool PACKED, bool FAST>
__global__ void __launch_bounds__(kThreads, 4) round_log_kernel(const RoundLogArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  __shared__ uint32_t s_warp[kWarps];
  __shared__ uint32_t s_total;
  __shared__ int64_t s_base;

  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  // Tile = blockIdx.x: 1-D grids are dispatched in increasing block order,
  // so every predecessor a tile waits on in the look-back is resident or done.
  const int64_t tile = blockIdx.x;
  const int64_t tile_base = tile * kTile;
  const int64_t wbase = tile_base + warp * kWarpElems;

  D4 xv[kSlots];
  load_slots(a.x, a.n, wbase, lane, xv);

  uint64_t* stage = reinterpret_cast<uint64_t*>(smem) + warp * kWarpElems;  // SPARSE
  uint8_t* cs = smem + (SPARSE ? kTile * sizeof(uint64_t) : 0);              // PACKED
  uint32_t err = 0;
  uint32_t cnt = 0;  // SPARSE: warp-uniform running count; else per-thread count
  const uint32_t lt = lanemask_lt();

#pragma unroll
  for (int j = 0; j < kSlots; ++j) {
    const int64_t i0 = wbase + j * 128 + lane * 4;
    uint32_t code[4];
    if (FAST) {
      float f[4];
      bool slow = false;
#pragma unroll
      for (int v = 0; v < 4; ++v) f[v] = round_dir32_fast(xv[j].v[v], a.thr32, code[v], slow);
      if (slow) {
#pragma unroll
        for (int v = 0; v < 4; ++v) f[v] = round_dir32(xv[j].v[v], a.thr32, a.g.thr_sub, code[v], err);
      }
      store_out<OUT>(a.out, i0, a.n, f);
    } else {
      uint64_t rb[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) rb[v] = round_dir(xv[j].v[v], a.g, code[v], err);
      store_out<OUT>(a.out, i0, a.n, rb);
    }
    if (CODES) {
      if (i0 + 3 < a.n) {
        *reinterpret_cast<uint32_t*>(a.codes + i0) = code[0] | (code[1] << 8) | (code[2] << 16) | (code[3] << 24);
      } else {
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (i0 + v < a.n) a.codes[i0 + v] = (uint8_t)code[v];
      }
    }
    if (PACKED) {
      const int e0 = warp * kWarpElems + j * 128 + lane * 4;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        cs[e0 + v] = (uint8_t)code[v];
        const int64_t i = i0 + v;
        if (i < a.n && (i < a.head || i >= a.head + 5 * a.nfull))
          a.edge[i < a.head ? i : i - 5 * a.nfull] = (uint8_t)code[v];
      }
    }
    if (SPARSE) {
      // warp-exclusive rank of this lane's logged elements: the lane's count
      // (0..4) is spread over three ballots, one per binary digit
      const uint32_t c = (code[0] != 1u) + (code[1] != 1u) + (code[2] != 1u) + (code[3] != 1u);
      const uint32_t b0 = __ballot_sync(0xffffffffu, c & 1u);
      const uint32_t b1 = __ballot_sync(0xffffffffu, c & 2u);
      const uint32_t b2 = __ballot_sync(0xffffffffu, c & 4u);
      uint32_t r = cnt + __popc(b0 & lt) + 2u * __popc(b1 & lt) + 4u * __popc(b2 & lt);
      if (c) {
        const uint64_t w0 = (uint64_t)(a.global_base + i0) << 1;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          if (code[v] != 1u) {
            stage[r] = w0 + ((uint64_t)v << 1) + (code[v] == 2u ? 1ull : 0ull);
            ++r;
          }
        }
      }
      cnt += __popc(b0) + 2u * __popc(b1) + 4u * __popc(b2);
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v) cnt += (code[v] != 1u) ? 1u : 0u;
    }
  }
  report_err(a.err, err);

  if (SPARSE) {
    if (lane == 0) s_warp[warp] = cnt;
    __syncthreads();
    if (warp == 0) {
      const uint32_t c = (lane < kWarps) ? s_warp[lane] : 0u;
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, kWarps - 1);
      __syncwarp();
      if (lane < kWarps) s_warp[lane] = incl - c;
      if (lane == 0) s_total = total;
    }
    __syncthreads();
    const uint32_t total = s_total;
    const int64_t excl = lookback(a.status, tile, total);
    if (threadIdx.x == 0) {
      const int64_t cur = a.cursor_in ? *a.cursor_in : 0;
      s_base = cur + excl;
      if (tile == a.num_tiles - 1) {
        atomicAdd(reinterpret_cast<unsigned long long*>(a.counters), (unsigned long long)(excl + (int64_t)total));
        if (a.cursor_out) *a.cursor_out = cur + excl + (int64_t)total;
      }
    }
    __syncthreads();
    const int64_t base = s_base + s_warp[warp];
    for (uint32_t i = lane; i < cnt; i += 32) {
      const int64_t pos = base + i;
      if (pos < a.sparse_cap) a.sparse[pos] = stage[i];
    }
  } else {
    const uint32_t w = warp_sum_u32(cnt);
    if (lane == 0) s_warp[warp] = w;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
#pragma unroll
      for (int k = 0; k < kWarps; ++k) t += s_warp[k];
      if (t) atomicAdd(reinterpret_cast<unsigned long long*>(a.counters), (unsigned long long)t);
    }
  }

  if (PACKED) {
    // A .vtrl group is owned by the tile holding its first element; groups
    // straddling the tile end need up to 4 codes from the next tile.
    if (threadIdx.x < 4) {
      const int64_t i = tile_base + kTile + threadIdx.x;
      uint32_t c = 1u, e2 = 0u;
      if (i < a.n) (void)round_dir(a.x[i], a.g, c, e2);
      cs[kTile + threadIdx.x] = (uint8_t)c;
    }
    __syncthreads();
    const int64_t g_lo = (tile_base <= a.head) ? 0 : (tile_base - a.head + 4) / 5;
    const int64_t g_hi = std::min<int64_t>(a.nfull, (tile_base + kTile - a.head + 4) / 5);
    for (int64_t gi = g_lo + threadIdx.x; gi < g_hi; gi += kThreads) {
      const int st = (int)(a.head + 5 * gi - tile_base);
      const uint32_t b = cs[st] + 3u * cs[st + 1] + 9u * cs[st + 2] + 27u * cs[st + 3] + 81u * cs[st + 4];
      a.packed[gi] = (uint8_t)b;
    }
  }
}

// ---------------------------------------------------------------------------
// replay
// ---------------------------------------------------------------------------

struct ReplayArgs {
  const double* x;
  int64_t n;
  Grid g;
  const void* log;
  int64_t log_len;
  int64_t log_base;
  void* out;
  int64_t* counters;
  int32_t* err;
};

// Dense-log replay (ternary codes, or the .vtrl payload); the sparse log
// goes through the persistent rp_fused_kernel (vt_stream.cu).
template <int OUT, int LOGK, bool FAST>
__global__ void __launch_bounds__(kThreads, 4) replay_kernel(const ReplayArgs a) {
  __shared__ uint32_t s_warp[kWarps];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int64_t tile = blockIdx.x;
  const int64_t tile_base = tile * kTile;
  const int64_t wbase = tile_base + warp * kWarpElems;

  D4 xv[kSlots];
  load_slots(a.x, a.n, wbase, lane, xv);
  uint32_t err = 0;

  // packed: a 256-entry table of each payload byte's five base-3 digits (3
  // bits each, roundlog.py:73-82); every thread then reads the one or two
  // payload bytes its 4 consecutive elements fall in -- no staging pass
  __shared__ uint16_t lut[256];
  int64_t qt = 0;
  int rt = 0;
  if (LOGK == VT_LOG_PACKED) {
    uint32_t t = threadIdx.x, v = 0;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      v |= (t % 3u) << (3 * k);
      t /= 3u;
    }
    lut[threadIdx.x] = (uint16_t)v;
    const int64_t pos_tile = a.log_base + tile_base;  // stream position of the tile's first element
    qt = pos_tile / 5;
    rt = (int)(pos_tile - 5 * qt);
    __syncthreads();
  }
  uint32_t flips = 0;
#pragma unroll
  for (int j = 0; j < kSlots; ++j) {
    const int64_t i0 = wbase + j * 128 + lane * 4;
    uint32_t code[4];
    if (LOGK == VT_LOG_CODES) {
      const uint8_t* cg = static_cast<const uint8_t*>(a.log);
      if (i0 + 3 < a.n) {
        const uint32_t c4 = *reinterpret_cast<const uint32_t*>(cg + i0);
#pragma unroll
        for (int v = 0; v < 4; ++v) code[v] = (c4 >> (8 * v)) & 0xffu;
      } else {
#pragma unroll
        for (int v = 0; v < 4; ++v) code[v] = (i0 + v < a.n) ? cg[i0 + v] : 1u;
      }
    } else {
      const uint8_t* p = static_cast<const uint8_t*>(a.log);
      const int rel = rt + warp * kWarpElems + j * 128 + lane * 4;  // < 2^16: 32-bit divisions by 5
      const int q0 = rel / 5, d0 = rel - 5 * q0;
      const int64_t bi0 = qt + q0;
      const int nv = (int)std::min<int64_t>(4, a.n - i0);  // valid elements of the four
      uint32_t b0 = 1u, b1 = 1u;  // bytes of the valid elements (past the end: unused)
      if (nv > 0) {
        b0 = (bi0 < a.log_len) ? (uint32_t)__ldg(p + bi0) : 255u;
        if (b0 > 242u) err |= VT_ERR_BAD_LOG_BYTE;
        if (d0 + nv > 5) {
          b1 = (bi0 + 1 < a.log_len) ? (uint32_t)__ldg(p + bi0 + 1) : 255u;
          if (b1 > 242u) err |= VT_ERR_BAD_LOG_BYTE;
        }
      }
      const uint32_t l0 = lut[b0 & 0xffu], l1 = lut[b1 & 0xffu];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int d = d0 + v;
        code[v] = v < nv ? (((d < 5 ? l0 : l1) >> (3 * (d < 5 ? d : d - 5))) & 7u) : 1u;
      }
    }
    if (FAST) {
      float y[4];
      uint32_t fl[4];
      bool slow = false;
#pragma unroll
      for (int v = 0; v < 4; ++v) y[v] = replay32_fast(xv[j].v[v], code[v], slow, fl[v]);
      if (slow) {
#pragma unroll
        for (int v = 0; v < 4; ++v) y[v] = replay32(xv[j].v[v], code[v], err, fl[v]);
      }
      flips += fl[0] + fl[1] + fl[2] + fl[3];  // padding lanes carry x = 0, code 1: never a flip
      store_out<OUT>(a.out, i0, a.n, y);
    } else {
      uint64_t rb[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        uint32_t f;
        rb[v] = replay_one(xv[j].v[v], code[v], a.g, err, f);
        flips += f;
      }
      store_out<OUT>(a.out, i0, a.n, rb);
    }
  }
  report_err(a.err, err);
  const uint32_t w = warp_sum_u32(flips);
  if (lane == 0) s_warp[warp] = w;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
#pragma unroll
    for (int k = 0; k < kWarps; ++k) t += s_warp[k];
    if (t) atomicAdd(reinterpret_cast<unsigned long long*>(a.counters), (unsigned long long)t);
  }
}

// ---------------------------------------------------------------------------
// elementwise helpers (not on the bandwidth-critical path)
// ---------------------------------------------------------------------------

__global__ void neighbors_kernel(const double* __restrict__ x, int64_t n, Grid g,
                                 double* __restrict__ below, double* __restrict__ above,
                                 int32_t* errp) {
  uint32_t err = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = x[i];
    const uint64_t bits = (uint64_t)__double_as_longlong(xi);
    const uint64_t mag = bits & kMag, sgn = bits & kSign;
    double lo, hi;
    if (mag >= kNormalMin) {
      err |= (mag >= kExpAllOnes) ? (uint32_t)VT_ERR_NONFINITE
                                  : ((mag > g.gmax_bits) ? (uint32_t)VT_ERR_RANGE_NEIGHBOR : 0u);
      const uint64_t trunc = mag & ~g.low_mask;
      const uint64_t away = trunc + (((mag & g.low_mask) != 0) ? g.one : 0ull);
      const double tv = __longlong_as_double((long long)(sgn | trunc));
      const double av = __longlong_as_double((long long)(sgn | away));
      const bool nonneg = !(xi < 0.0);
      lo = nonneg ? tv : av;
      hi = nonneg ? av : tv;
    } else {
      const double s = __dmul_rn(xi, g.sub_up);
      lo = __dmul_rn(floor(s), g.sub_dn);
      hi = __dmul_rn(ceil(s), g.sub_dn);
    }
    below[i] = lo;
    above[i] = hi;
  }
  report_err(errp, err);
}

__global__ void exponent_scale_kernel(const double* __restrict__ x, int64_t n,
                                      double* __restrict__ out, int32_t* errp) {
  uint32_t err = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = x[i];
    if (!isfinite(xi)) err |= VT_ERR_NONFINITE;
    int e = 0;
    (void)frexp(xi, &e);
    out[i] = (xi == 0.0) ? 0x1p-126 : ldexp(1.0, e - 1);
  }
  report_err(errp, err);
}

__global__ void on_grid_kernel(const double* __restrict__ x, int64_t n, uint32_t mask,
                               uint8_t* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = x[i];
    const float f = __double2float_rn(xi);
    const bool exact = isfinite(f) && ((double)f == xi);
    out[i] = (exact && ((__float_as_uint(f) & mask) == 0u)) ? 1 : 0;
  }
}

__global__ void norm_distance_kernel(const double* __restrict__ x, int64_t n, Grid g,
                                     double* __restrict__ out, int32_t* errp) {
  uint32_t err = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = x[i];
    const double r = __longlong_as_double((long long)round_only(xi, g, err));
    int e = 0;
    (void)frexp(xi, &e);
    double scale = (xi == 0.0) ? 0x1p-126 : ldexp(1.0, e - 1);
    scale = scale < 0x1p-126 ? 0x1p-126 : scale;
    out[i] = __ddiv_rn(fabs(__dsub_rn(xi, r)), scale);
  }
  report_err(errp, err);
}

}  // namespace vt

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------

using namespace vt;

namespace {

bool valid_b(int b_r) { return b_r >= 10 && b_r <= 32; }
bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }
int64_t num_tiles_for(int64_t n) { return (n + kTile - 1) / kTile; }

template <int OUT, bool S, bool C, bool P, bool F>
void launch_rl(const RoundLogArgs& a, int64_t tiles, cudaStream_t st) {
  size_t smem = (S ? (size_t)kTile * sizeof(uint64_t) : 0) + (P ? (size_t)kTile + 8 : 0);
  auto k = round_log_kernel<OUT, S, C, P, F>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k<<<(unsigned)tiles, kThreads, smem, st>>>(a);
}

typedef void (*rl_fn)(const RoundLogArgs&, int64_t, cudaStream_t);

template <int OUT, bool F>
rl_fn pick_rl2(int key) {
  switch (key) {
    case 0: return launch_rl<OUT, false, false, false, F>;
    case 1: return launch_rl<OUT, false, false, true, F>;
    case 2: return launch_rl<OUT, false, true, false, F>;
    case 3: return launch_rl<OUT, false, true, true, F>;
    case 4: return launch_rl<OUT, true, false, false, F>;
    case 5: return launch_rl<OUT, true, false, true, F>;
    case 6: return launch_rl<OUT, true, true, false, F>;
    default: return launch_rl<OUT, true, true, true, F>;
  }
}

rl_fn pick_rl(int out_kind, bool fast, bool s, bool c, bool p) {
  const int key = (s ? 4 : 0) | (c ? 2 : 0) | (p ? 1 : 0);
  if (fast) {
    return out_kind == VT_OUT_F32 ? pick_rl2<VT_OUT_F32, true>(key)
         : out_kind == VT_OUT_F64 ? pick_rl2<VT_OUT_F64, true>(key)
                                  : pick_rl2<VT_OUT_NONE, true>(key);
  }
  return out_kind == VT_OUT_F32 ? pick_rl2<VT_OUT_F32, false>(key)
       : out_kind == VT_OUT_F64 ? pick_rl2<VT_OUT_F64, false>(key)
                                : pick_rl2<VT_OUT_NONE, false>(key);
}

}  // namespace

extern "C" int vt_tile_elems(void) { return kTile; }

extern "C" size_t vt_round_log_workspace(int64_t n) {
  return std::max((size_t)(num_tiles_for(n) * 8 + 256), rl_stream_workspace(n));
}

extern "C" int vt_round_log(const double* x, int64_t n, int b_r, double tau, int out_kind, void* out,
                            uint64_t* sparse, int64_t sparse_cap, int64_t global_base,
                            const int64_t* cursor_in, int64_t* cursor_out, uint8_t* codes,
                            uint8_t* packed, int64_t log_pos, uint8_t* edge_codes,
                            int64_t* counters, int32_t* err, void* ws, size_t ws_bytes,
                            vt_stream_t stream) {
  if (n < 0 || !valid_b(b_r) || out_kind < 0 || out_kind > 2 || !counters || !err) {
    vt_set_error("vt_round_log: bad argument");
    return VT_EINVAL;
  }
  if (n == 0) return VT_OK;
  if (!x || !aligned(x, 32) || (out_kind == VT_OUT_F32 && !aligned(out, 16)) ||
      (out_kind == VT_OUT_F64 && !aligned(out, 32)) || (codes && !aligned(codes, 4)) ||
      (packed && !edge_codes) || log_pos < 0) {
    vt_set_error("vt_round_log: null or misaligned buffer (x needs 32 B, f32 out 16 B, f64 out 32 B, codes 4 B)");
    return VT_EINVAL;
  }
  const int64_t tiles = num_tiles_for(n);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  RoundLogArgs a;
  a.x = x;
  a.n = n;
  a.g = make_grid(b_r, tau);
  a.out = out;
  a.sparse = sparse;
  a.sparse_cap = sparse_cap;
  a.global_base = global_base;
  a.cursor_in = cursor_in;
  a.cursor_out = cursor_out;
  a.codes = codes;
  a.packed = packed;
  const int64_t head = std::min<int64_t>((5 - log_pos % 5) % 5, n);
  a.head = head;
  a.nfull = (n - head) / 5;
  a.edge = edge_codes;
  a.counters = counters;
  a.err = err;
  a.num_tiles = tiles;
  a.status = nullptr;
  a.thr32 = (int)std::min<int64_t>(std::max<int64_t>(a.g.thr, 0), INT32_MAX);
  if (sparse) {
    if (!ws || ws_bytes < vt_round_log_workspace(n)) {
      vt_set_error("vt_round_log: workspace too small");
      return VT_EINVAL;
    }
    if (!codes && !packed) {  // north-star path: persistent TMA streaming + look-back expand
      return rl_stream(x, n, a.g, a.thr32, b_r == 32, out_kind, out, sparse, sparse_cap, global_base, cursor_in,
                       cursor_out, counters, err, ws, st);
    }
    a.status = static_cast<uint64_t*>(ws);
    if (cudaMemsetAsync(ws, 0, (size_t)tiles * 8, st) != cudaSuccess) return vt_check_launch("memset");
  }
  rl_fn f = pick_rl(out_kind, b_r == 32, sparse != nullptr, codes != nullptr, packed != nullptr);
  f(a, tiles, st);
  return vt_check_launch("round_log_kernel");
}

extern "C" size_t vt_exchange_words(int world) { return world > 0 ? (size_t)(1 + 2 * world) : 0; }

extern "C" int vt_round_log_exchange(const double* x, int64_t n, int b_r, double tau, int out_kind, void* out,
                                     uint64_t* sparse, int64_t sparse_cap, int64_t global_base, int64_t* counters,
                                     int32_t* err, void* ws, size_t ws_bytes, uint64_t* const* xpeers, int world,
                                     int rank, vt_stream_t stream) {
  if (n < 0 || !valid_b(b_r) || out_kind < 0 || out_kind > 2 || !counters || !err || !xpeers || world <= 0 ||
      rank < 0 || rank >= world) {
    vt_set_error("vt_round_log_exchange: bad argument (n >= 0, 0 <= rank < world)");
    return VT_EINVAL;
  }
  if (n == 0)  // an empty shard still takes part: it publishes a count of 0
    return exchange_publish_empty(XPeers{xpeers, world, rank}, static_cast<cudaStream_t>(stream));
  if (!sparse || !ws || ws_bytes < vt_round_log_workspace(n)) {
    vt_set_error("vt_round_log_exchange: bad argument (sparse log, workspace)");
    return VT_EINVAL;
  }
  if (!aligned(x, 32) || (out_kind == VT_OUT_F32 && !aligned(out, 16)) || (out_kind == VT_OUT_F64 && !aligned(out, 32))) {
    vt_set_error("vt_round_log_exchange: misaligned buffer");
    return VT_EINVAL;
  }
  const Grid g = make_grid(b_r, tau);
  const int thr32 = (int)std::min<int64_t>(std::max<int64_t>(g.thr, 0), INT32_MAX);
  return rl_stream(x, n, g, thr32, b_r == 32, out_kind, out, sparse, sparse_cap, global_base, nullptr, nullptr,
                   counters, err, ws, static_cast<cudaStream_t>(stream), nullptr, nullptr, nullptr,
                   XPeers{xpeers, world, rank});
}

extern "C" int vt_counts_wait(uint64_t* const* xpeers, int world, int rank, int64_t* counts_out, int32_t* err,
                              vt_stream_t stream) {
  if (!xpeers || world <= 0 || rank < 0 || rank >= world || !counts_out || !err) {
    vt_set_error("vt_counts_wait: bad argument");
    return VT_EINVAL;
  }
  return counts_wait(XPeers{xpeers, world, rank}, counts_out, err, static_cast<cudaStream_t>(stream));
}

namespace {
template <int OUT, int L, bool F>
void launch_rp(const ReplayArgs& a, int64_t tiles, cudaStream_t st) {
  replay_kernel<OUT, L, F><<<(unsigned)tiles, kThreads, 0, st>>>(a);
}
typedef void (*rp_fn)(const ReplayArgs&, int64_t, cudaStream_t);
template <int OUT, bool F>
rp_fn pick_rp2(int lk) {
  return lk == VT_LOG_CODES ? launch_rp<OUT, VT_LOG_CODES, F> : launch_rp<OUT, VT_LOG_PACKED, F>;
}
rp_fn pick_rp(int out_kind, bool fast, int lk) {
  if (fast) {
    return out_kind == VT_OUT_F32 ? pick_rp2<VT_OUT_F32, true>(lk)
         : out_kind == VT_OUT_F64 ? pick_rp2<VT_OUT_F64, true>(lk)
                                  : pick_rp2<VT_OUT_NONE, true>(lk);
  }
  return out_kind == VT_OUT_F32 ? pick_rp2<VT_OUT_F32, false>(lk)
       : out_kind == VT_OUT_F64 ? pick_rp2<VT_OUT_F64, false>(lk)
                                : pick_rp2<VT_OUT_NONE, false>(lk);
}
}  // namespace

extern "C" size_t vt_replay_workspace(int64_t n) { return rp_stream_workspace(n); }

extern "C" int vt_replay(const double* x, int64_t n, int b_r, int log_kind, const void* log,
                         int64_t log_len, int64_t log_base, int out_kind, void* out,
                         int64_t* counters, int32_t* err, void* ws, size_t ws_bytes,
                         vt_stream_t stream) {
  if (n < 0 || !valid_b(b_r) || out_kind < 0 || out_kind > 2 || log_kind < 0 || log_kind > 2 ||
      !counters || !err || log_len < 0 || log_base < 0) {
    vt_set_error("vt_replay: bad argument");
    return VT_EINVAL;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t tiles = num_tiles_for(n);
  if (n == 0) return VT_OK;
  if (!x || !aligned(x, 32) || (out_kind == VT_OUT_F32 && !aligned(out, 16)) ||
      (out_kind == VT_OUT_F64 && !aligned(out, 32)) || (!log && (log_len > 0 || log_kind == VT_LOG_CODES)) ||
      (log_kind == VT_LOG_CODES && !aligned(log, 4))) {
    vt_set_error("vt_replay: null or misaligned buffer");
    return VT_EINVAL;
  }
  ReplayArgs a;
  a.x = x;
  a.n = n;
  a.g = make_grid(b_r, 0.0);
  a.log = log;
  a.log_len = log_len;
  a.log_base = log_base;
  a.out = out;
  a.counters = counters;
  a.err = err;
  if (log_kind == VT_LOG_SPARSE) {
    if (!ws || ws_bytes < vt_replay_workspace(n)) {
      vt_set_error("vt_replay: workspace too small");
      return VT_EINVAL;
    }
    return rp_stream(x, n, a.g, b_r == 32, out_kind, out, static_cast<const uint64_t*>(log), log_len, log_base,
                     counters, err, ws, st);
  }
  if (log_kind == VT_LOG_PACKED && n >= (1 << 18) && ws && ws_bytes >= vt_replay_workspace(n)) {
    // the persistent TMA-pipelined replay, decoding the payload a tile ahead
    // (2^26: 86% vs 79% of the copy peak for replay_kernel<PACKED>); small
    // tensors keep the per-tile kernel, which spreads them over more SMs
    return rp_stream_packed(x, n, a.g, b_r == 32, out_kind, out, static_cast<const uint8_t*>(log), log_len,
                            log_base, counters, err, ws, st);
  }
  rp_fn f = pick_rp(out_kind, b_r == 32, log_kind);
  f(a, tiles, st);
  return vt_check_launch("replay_kernel");
}

namespace {
unsigned ew_blocks(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}
}  // namespace

extern "C" int vt_grid_neighbors(const double* x, int64_t n, int b_r, double* below, double* above,
                                 int32_t* err, vt_stream_t stream) {
  if (n < 0 || !valid_b(b_r) || !err) {
    vt_set_error("vt_grid_neighbors: bad argument");
    return VT_EINVAL;
  }
  if (n == 0) return VT_OK;
  neighbors_kernel<<<ew_blocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      x, n, make_grid(b_r, 0.0), below, above, err);
  return vt_check_launch("neighbors_kernel");
}

extern "C" int vt_exponent_scale(const double* x, int64_t n, double* out, int32_t* err,
                                 vt_stream_t stream) {
  if (n < 0 || !err) {
    vt_set_error("vt_exponent_scale: bad argument");
    return VT_EINVAL;
  }
  if (n == 0) return VT_OK;
  exponent_scale_kernel<<<ew_blocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(x, n, out, err);
  return vt_check_launch("exponent_scale_kernel");
}

extern "C" int vt_is_on_grid(const double* x, int64_t n, int b_r, uint8_t* out, vt_stream_t stream) {
  if (n < 0 || !valid_b(b_r)) {
    vt_set_error("vt_is_on_grid: bad argument");
    return VT_EINVAL;
  }
  if (n == 0) return VT_OK;
  const uint32_t mask = (b_r < 32) ? ((1u << (32 - b_r)) - 1u) : 0u;
  on_grid_kernel<<<ew_blocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(x, n, mask, out);
  return vt_check_launch("on_grid_kernel");
}

extern "C" int vt_norm_distance(const double* x, int64_t n, int b_r, double* out, int32_t* err,
                                vt_stream_t stream) {
  if (n < 0 || !valid_b(b_r) || !err) {
    vt_set_error("vt_norm_distance: bad argument");
    return VT_EINVAL;
  }
  if (n == 0) return VT_OK;
  norm_distance_kernel<<<ew_blocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      x, n, make_grid(b_r, 0.0), out, err);
  return vt_check_launch("norm_distance_kernel");
}
