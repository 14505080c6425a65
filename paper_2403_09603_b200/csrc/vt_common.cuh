// Shared device code: grid parameters, bit-exact rounding / direction /
// replay primitives, streaming load/store wrappers, error plumbing.
//
// Semantics follow the reference (vtrain 0.1.0, pkg/src/vtrain/fpround.py):
//   rnd        fpround.py:99-135   RNE on the kept mantissa bits, absolute grid below 2^-126
//   direction  fpround.py:164-177  strict |x - rnd(x)| > max(scale(x), 2^-126) * tau
//   neighbours fpround.py:185-218  truncate + one step in magnitude space
//   rev        fpround.py:227-247  neighbour on the coded side when rnd disagrees
// The integer forms used here are derived in SURVEY.md Appendix B and are
// checked bit for bit against the oracle by tests/test_gpu_*.py.
//
// Build flags never include --use_fast_math / -ftz: FP32/FP64 subnormals must
// survive, and FP64 arithmetic below uses explicit _rn intrinsics so nothing
// is contracted into an FMA.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/vtrain_b200.h"

namespace vt {

constexpr uint64_t kSign = 0x8000000000000000ull;
constexpr uint64_t kMag = 0x7fffffffffffffffull;
constexpr uint64_t kNormalMin = 0x3810000000000000ull;  // bits of 2^-126
constexpr uint64_t kExpAllOnes = 0x7ff0000000000000ull;  // inf / nan threshold

// Tile geometry shared by every streaming kernel: 8 warps x 5 slots x
// 32 lanes x 4 consecutive FP64 (one 256-bit load per lane per slot).
// 640 = lcm(5, 128) elements per warp keeps .vtrl byte groups and 128-bit
// vectors aligned to warp boundaries.
constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kVec = 4;
constexpr int kSlots = 5;
constexpr int kWarpElems = 32 * kVec * kSlots;  // 640
constexpr int kTile = kWarps * kWarpElems;      // 5120

struct Grid {
  int drop;             // 52 - (b_r - 9) mantissa bits dropped
  int _pad;
  uint64_t low_mask;    // (1 << drop) - 1
  uint64_t half;        // 1 << (drop - 1)
  uint64_t one;         // 1 << drop
  uint64_t gmax_bits;   // bit pattern of grid_max(b_r)
  double sub_up;        // 2^-q, q = (32 - b_r) - 149
  double sub_dn;        // 2^q
  int64_t thr;          // integer threshold on d (units of ulp(x) in FP64)
  double thr_sub;       // 2^-126 * tau, the FP64 threshold below 2^-126
};

// Host-side construction (also used by the C ABI wrappers).
inline Grid make_grid(int b_r, double tau) {
  Grid g;
  g.drop = 52 - (b_r - 9);
  g._pad = 0;
  g.one = 1ull << g.drop;
  g.low_mask = g.one - 1;
  g.half = 1ull << (g.drop - 1);
  // grid_max = (2 - 2^-(b_r-9)) * 2^127: FP64 biased exponent 1023 + 127,
  // the kept mantissa bits all ones
  g.gmax_bits = (1150ull << 52) | (((1ull << (b_r - 9)) - 1) << g.drop);
  int q = (32 - b_r) - 149;
  g.sub_up = ldexp(1.0, -q);
  g.sub_dn = ldexp(1.0, q);
  // Normal range: |x - r| = d * 2^(E-52) exactly and scale*tau = 2^E * tau,
  // so (strict) |x - r| > scale * tau  <=>  d > tau * 2^52  <=>  d > floor(tau * 2^52).
  // Degenerate taus are mapped so the comparison keeps the FP64 outcome.
  if (tau != tau) {
    g.thr = INT64_MAX;  // NaN: comparison always false
  } else if (tau < 0.0) {
    g.thr = -1;  // every d >= 0 passes; d == 0 still yields IGNORE
  } else if (tau < 0x1p-800) {
    g.thr = 0;  // tau * 2^E may underflow, but any d >= 1 exceeds it
  } else {
    double t = floor(ldexp(tau, 52));
    g.thr = (t >= 0x1p62) ? INT64_MAX : (int64_t)t;
  }
  g.thr_sub = 0x1p-126 * tau;
  return g;
}

// Thresholds derived from a tau that lives on the device (adaptive path:
// the bisection result never visits the host).  Same mapping as make_grid.
struct DevThr {
  double tau;
  int64_t thr;
  double thr_sub;
  int32_t thr32;
  int32_t _pad;
};

__host__ __device__ inline DevThr thresholds_for(double tau) {
  DevThr d;
  d.tau = tau;
  if (tau != tau) {
    d.thr = INT64_MAX;
  } else if (tau < 0.0) {
    d.thr = -1;
  } else if (tau < 0x1p-800) {
    d.thr = 0;
  } else {
    const double t = floor(ldexp(tau, 52));
    d.thr = (t >= 0x1p62) ? INT64_MAX : (int64_t)t;
  }
  d.thr_sub = 0x1p-126 * tau;
  d.thr32 = (int32_t)(d.thr < 0 ? 0 : (d.thr > INT32_MAX ? INT32_MAX : d.thr));
  d._pad = 0;
  return d;
}

// ---------------------------------------------------------------------------
// element primitives
// ---------------------------------------------------------------------------

// Round x onto the grid and classify it.  Returns the rounded FP64 bits;
// `code` gets 0 (DOWN: x > r), 1 (IGNORE), 2 (UP: x < r); `err` collects
// VT_ERR_NONFINITE / VT_ERR_RANGE.
__device__ __forceinline__ uint64_t round_dir(double x, const Grid& g, uint32_t& code,
                                              uint32_t& err) {
  const uint64_t bits = (uint64_t)__double_as_longlong(x);
  const uint64_t mag = bits & kMag;
  const uint64_t sgn = bits & kSign;
  if (mag >= kNormalMin) {
    const uint64_t low = mag & g.low_mask;
    const uint64_t base = mag >> g.drop;
    const bool up = (low > g.half) || ((low == g.half) && (base & 1ull));
    const uint64_t rmag = (base + (up ? 1ull : 0ull)) << g.drop;
    err |= (mag >= kExpAllOnes) ? (uint32_t)VT_ERR_NONFINITE
                                : ((rmag > g.gmax_bits) ? (uint32_t)VT_ERR_RANGE : 0u);
    const int64_t d = (int64_t)(up ? (g.one - low) : low);
    const bool logged = (d > g.thr) && (low != 0);
    const bool r_above = up != (sgn != 0);  // x < r
    code = logged ? (r_above ? 2u : 0u) : 1u;
    return sgn | rmag;
  }
  const double s = __dmul_rn(x, g.sub_up);
  const double r = __dmul_rn(rint(s), g.sub_dn);
  const double dist = fabs(__dsub_rn(x, r));
  const bool logged = dist > g.thr_sub;
  code = logged ? ((x < r) ? 2u : ((x > r) ? 0u : 1u)) : 1u;
  return (uint64_t)__double_as_longlong(r);
}

// Plain rounding (no classification).
__device__ __forceinline__ uint64_t round_only(double x, const Grid& g, uint32_t& err) {
  const uint64_t bits = (uint64_t)__double_as_longlong(x);
  const uint64_t mag = bits & kMag;
  if (mag >= kNormalMin) {
    const uint64_t low = mag & g.low_mask;
    const uint64_t base = mag >> g.drop;
    const bool up = (low > g.half) || ((low == g.half) && (base & 1ull));
    const uint64_t rmag = (base + (up ? 1ull : 0ull)) << g.drop;
    err |= (mag >= kExpAllOnes) ? (uint32_t)VT_ERR_NONFINITE
                                : ((rmag > g.gmax_bits) ? (uint32_t)VT_ERR_RANGE : 0u);
    return (bits & kSign) | rmag;
  }
  const double r = __dmul_rn(rint(__dmul_rn(x, g.sub_up)), g.sub_dn);
  return (uint64_t)__double_as_longlong(r);
}

// Replay: rnd(x) unless the recorded code points at the other neighbour.
// `flip` is set when the output differs from rnd(x) (an auditor correction).
__device__ __forceinline__ uint64_t replay_one(double x, uint32_t c, const Grid& g,
                                               uint32_t& err, uint32_t& flip) {
  const uint64_t bits = (uint64_t)__double_as_longlong(x);
  const uint64_t mag = bits & kMag;
  const uint64_t sgn = bits & kSign;
  err |= (c > 2u) ? (uint32_t)VT_ERR_BAD_CODE : 0u;
  if (mag >= kNormalMin) {
    const uint64_t low = mag & g.low_mask;
    const uint64_t base = mag >> g.drop;
    const bool up = (low > g.half) || ((low == g.half) && (base & 1ull));
    err |= (mag >= kExpAllOnes) ? (uint32_t)VT_ERR_NONFINITE
                                : ((mag > g.gmax_bits) ? (uint32_t)VT_ERR_RANGE_NEIGHBOR : 0u);
    const bool off = low != 0;
    const bool r_above = up != (sgn != 0);  // x < r when off grid
    const bool f = off && ((c == 0u && r_above) || (c == 2u && !r_above));
    flip = f ? 1u : 0u;
    return sgn | ((base + ((up != f) ? 1ull : 0ull)) << g.drop);
  }
  const double s = __dmul_rn(x, g.sub_up);
  const double r = __dmul_rn(rint(s), g.sub_dn);
  if (c == 0u && x < r) {
    flip = 1u;
    return (uint64_t)__double_as_longlong(__dmul_rn(floor(s), g.sub_dn));
  }
  if (c == 2u && x > r) {
    flip = 1u;
    return (uint64_t)__double_as_longlong(__dmul_rn(ceil(s), g.sub_dn));
  }
  flip = 0u;
  return (uint64_t)__double_as_longlong(r);
}

// ---------------------------------------------------------------------------
// b_r = 32 fast path: the grid is exactly the FP32 value set, so
// rnd(x) == (double)cvt.rn.f32.f64(x) for every finite x, FP32 subnormals
// included (no FTZ) -- SURVEY.md Appendix A.1 / B.1, pinned by the GPU
// parity tests.  Direction and replay decisions then need only the low
// 32 bits of x (normal range) or one FP64 compare (below 2^-126).
// ---------------------------------------------------------------------------

constexpr double kFltMax = 3.4028234663852886e38;

// thr32 = clamp(Grid::thr, 0, INT32_MAX): d is an integer in [0, 2^28], so
// d > thr  <=>  d > max(thr, 0) whenever d != 0, and d == 0 is never logged.
__device__ __forceinline__ float round_dir32(double x, int thr32, double thr_sub, uint32_t& code,
                                             uint32_t& err) {
  const float f = __double2float_rn(x);
  const int hi = __double2hiint(x);
  const uint32_t lo = (uint32_t)__double2loint(x);
  const uint32_t ahi = (uint32_t)hi & 0x7fffffffu;
  if (ahi >= 0x38100000u) {  // |x| >= 2^-126 (incl. inf / nan)
    const uint32_t low = lo & 0x1fffffffu;  // the 29 dropped mantissa bits
    // RNE: round magnitude up iff low > half, or low == half and the kept lsb is odd
    const bool up = (low + ((lo >> 29) & 1u)) > 0x10000000u;
    const int d = (int)(up ? (0x20000000u - low) : low);
    const bool r_above = up != (hi < 0);
    code = (d > thr32) ? (r_above ? 2u : 0u) : 1u;
    if (ahi >= 0x47efffffu)  // |x| >= FLT_MAX + half ulp (0x47efffff00000000) possible
      err |= (ahi >= 0x7ff00000u) ? (uint32_t)VT_ERR_NONFINITE : (isinf(f) ? (uint32_t)VT_ERR_RANGE : 0u);
  } else {  // absolute grid below 2^-126: FP64 test exactly as the reference
    const double r = (double)f;
    const bool logged = fabs(__dsub_rn(x, r)) > thr_sub;
    code = logged ? ((x < r) ? 2u : ((x > r) ? 0u : 1u)) : 1u;
  }
  return f;
}

// Branch-free variants for the common case 2^-126 <= |x| < FLT_MAX + half ulp.
// `slow` is raised for anything else (FP32-subnormal range, overflow,
// inf/nan, bad code); the caller then redoes the element group with the
// exact general routines above / below.
__device__ __forceinline__ bool outside_normal32(uint32_t ahi) {
  return (ahi - 0x38100000u) >= (0x47efffffu - 0x38100000u);
}

__device__ __forceinline__ float round_dir32_fast(double x, int thr32, uint32_t& code, bool& slow) {
  const float f = __double2float_rn(x);
  const int hi = __double2hiint(x);
  const uint32_t lo = (uint32_t)__double2loint(x);
  slow |= outside_normal32((uint32_t)hi & 0x7fffffffu);
  const uint32_t low = lo & 0x1fffffffu;
  const bool up = (low + ((lo >> 29) & 1u)) > 0x10000000u;
  const int d = (int)(up ? (0x20000000u - low) : low);
  code = (d > thr32) ? ((up != (hi < 0)) ? 2u : 0u) : 1u;
  return f;
}

__device__ __forceinline__ float replay32_fast(double x, uint32_t c, bool& slow, uint32_t& flip) {
  const float f = __double2float_rn(x);
  const int hi = __double2hiint(x);
  const uint32_t lo = (uint32_t)__double2loint(x);
  slow |= outside_normal32((uint32_t)hi & 0x7fffffffu) | (c > 2u);
  const uint32_t low = lo & 0x1fffffffu;
  const bool up = (low + ((lo >> 29) & 1u)) > 0x10000000u;
  const bool r_above = up != (hi < 0);  // x < rnd(x) when off grid
  const bool fl = (low != 0u) && ((c == 0u && r_above) || (c == 2u && !r_above));
  flip = fl ? 1u : 0u;
  // sign-magnitude: one FP32 ulp of magnitude is +-1 on the bit pattern
  return fl ? __int_as_float(__float_as_int(f) + (up ? -1 : 1)) : f;
}

__device__ __forceinline__ float replay32(double x, uint32_t c, uint32_t& err, uint32_t& flip) {
  float f = __double2float_rn(x);
  const double r = (double)f;
  const bool above = r > x;
  const bool below = r < x;
  const bool fl = (c == 0u && above) || (c == 2u && below);
  err |= (c > 2u) ? (uint32_t)VT_ERR_BAD_CODE : 0u;
  if (!(fabs(x) <= kFltMax))
    err |= (isnan(x) || isinf(x)) ? (uint32_t)VT_ERR_NONFINITE : (uint32_t)VT_ERR_RANGE_NEIGHBOR;
  if (fl) f = __int_as_float(__float_as_int(f) + ((above != (x < 0.0)) ? -1 : 1));
  flip = fl ? 1u : 0u;
  return f;
}

// ---------------------------------------------------------------------------
// memory helpers
// ---------------------------------------------------------------------------

struct D4 {
  double v[4];
};

// 256-bit streaming load (LDG.E.NA...256 on sm_100a), read-once data.
__device__ __forceinline__ D4 ldg_stream4(const double* p) {
  D4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
               : "l"(p));
  return r;
}

__device__ __forceinline__ void stg_stream4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b),
               "d"(c), "d"(d)
               : "memory");
}

__device__ __forceinline__ void stg_stream4f(float* p, float a, float b, float c, float d) {
  asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b),
               "f"(c), "f"(d)
               : "memory");
}

__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// system scope: peer GPUs' memory over NVLink (symmetric-memory exchange)
__device__ __forceinline__ uint64_t ld_acquire_sys_u64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys_u64(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ void report_err(int32_t* err, uint32_t e) {
  if (e) atomicOr(reinterpret_cast<int*>(err), (int)e);
}

// persistent TMA-pipelined kernels of the north-star path (vt_stream.cu)
size_t rl_stream_workspace(int64_t n);
size_t rp_stream_workspace(int64_t n);
// dthr: nullable device thresholds overriding g.thr / g.thr_sub / thr32;
// gate: nullable device flag, the kernel does nothing while *gate == 0
// The per-rank count exchange over peer memory (vt_round_log_exchange):
// xpeers = device array of `world` pointers to every rank's exchange buffer
// (symmetric memory, vt_exchange_words(world) uint64 words each).
struct XPeers {
  uint64_t* const* peers;
  int world, rank;
};

int rl_stream(const double* x, int64_t n, const Grid& g, int thr32, bool fast, int out_kind, void* out,
              uint64_t* sparse, int64_t cap, int64_t global_base, const int64_t* cursor_in, int64_t* cursor_out,
              int64_t* counters, int32_t* err, void* ws, cudaStream_t st, const DevThr* dthr = nullptr,
              const int32_t* gate = nullptr, uint64_t* keys = nullptr, XPeers xp = XPeers{nullptr, 0, 0});
int counts_wait(XPeers xp, int64_t* counts_out, int32_t* err, cudaStream_t st);
int exchange_publish_empty(XPeers xp, cudaStream_t st);
int rp_stream(const double* x, int64_t n, const Grid& g, bool fast, int out_kind, void* out, const uint64_t* log,
              int64_t n_words, int64_t log_base, int64_t* counters, int32_t* err, void* ws, cudaStream_t st);
int rp_stream_packed(const double* x, int64_t n, const Grid& g, bool fast, int out_kind, void* out,
                     const uint8_t* payload, int64_t nbytes, int64_t pos, int64_t* counters, int32_t* err, void* ws,
                     cudaStream_t st);

// Batched trainer pass: up to kMaxBatch tensors in one launch of the fused
// round-and-log.  The table travels by value as a __grid_constant__ kernel
// parameter (no descriptor upload, so batches are graph-capturable).  Each
// tensor owns a contiguous run of tickets [tick0, tick0 + its super-tiles)
// and the look-back words at the same offsets; its log is its own.
constexpr int kMaxBatch = 224;

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

// rl_batch_kernel<..., KEYS>: a candidate whose x was not staged (its row
// overflowed the staging slots); the adaptive histogram gathers it
constexpr uint64_t kKeyMissing = ~0ull;

struct RLSeg {
  const double* x;
  void* out;
  uint64_t* sparse;
  int64_t* cursor_out;  // nullable: entries written (the adaptive candidate count)
  int64_t* counters;    // counters[0] += entries
  int32_t* err;
  const DevThr* dthr;   // nullable: thresholds from the device instead of thr / thr_sub / thr32
  const int32_t* gate;  // nullable: the tensor is skipped while *gate == 0
  uint64_t* keys;       // KEYS launches: x bits of each logged element (or kKeyMissing), at its log position
  int64_t n, cap, global_base, tick0;
  int64_t thr;
  double thr_sub;
  int32_t thr32, pad;
};

struct RLBatch {
  Grid g;            // b_r-dependent fields (thr / thr_sub per tensor)
  void* hdr;         // FusedHeader + look-back words (vt_round_log_workspace layout)
  const int32_t* any;  // nullable: the whole launch does nothing while *any == 0
  int32_t nseg, pad;
  int64_t total;     // tickets over all tensors
  RLSeg seg[kMaxBatch];
};

// tiles (of 2048 elements) per round-and-log ticket / look-back word
#ifndef VT_RL_SUPER  // A/B: tiles per round-and-log ticket
#define VT_RL_SUPER 4
#endif
constexpr int kRLSuper = VT_RL_SUPER;
__host__ __device__ inline int64_t rl_batch_tickets(int64_t n) {
  const int64_t tiles = (n + 2047) / 2048;
  return tiles / kRLSuper + tiles % kRLSuper;
}
// the batch's look-back words come after a 64-byte header
inline size_t rl_batch_workspace(int64_t total_tickets) { return (size_t)(64 + total_tickets * 8 + 256); }
int rl_stream_batch(const RLBatch& b, bool fast, int out_kind, cudaStream_t st, bool keys = false);

}  // namespace vt

// host-side error bookkeeping shared by the ABI translation units
void vt_set_error(const char* what);
int vt_check_launch(const char* what);
