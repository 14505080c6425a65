// Persistent, TMA-pipelined streaming kernels for the north-star path
// (sparse log, FP32 / FP64 output):
//
//   rl_fused_kernel    trainer round-and-log (protocol._TrainerChannel.process,
//                      pkg/src/vtrain/protocol.py:198-202) in ONE pass: rounds
//                      every element, and writes the ascending uint64 log
//                      (global_index << 1 | up) at its global position, found by
//                      an in-kernel decoupled look-back over 8192-element
//                      super-tiles (warp-specialised; see the section below);
//   rp_fused_kernel    auditor replay (protocol._AuditorChannel.process,
//                      protocol.py:212-216) -- scatters the tile's log slice into a
//                      shared-memory code map and replays every element.
//
// Streaming CTAs are persistent (grid = resident CTAs): the trainer draws
// super-tiles from an atomic ticket counter, the auditor walks a contiguous
// range of tiles; the FP64 input of the next tiles is in flight at all times
// through cp.async.bulk (TMA bulk copies, L2 evict-first) into a shared-memory
// ring guarded by mbarriers, so HBM streams continuously while the SM computes.
#include <algorithm>
#include <cstdlib>

#include "vt_common.cuh"

#ifndef VT_L2_PREFETCH  // round-and-log producer: L2 prefetch of each ticket's tiles when drawn
#define VT_L2_PREFETCH 1
#endif
#ifndef VT_RP_L2_PREFETCH  // replay producer: the same (measured slower; off)
#define VT_RP_L2_PREFETCH 0
#endif


namespace vt {

constexpr int kSThreads = 256;
constexpr int kSTile = 2048;  // elements per tile (16 KiB of FP64)
constexpr int kSWarpElems = kSTile / kWarps;  // 256
constexpr int kSSlots = kSWarpElems / 64;     // 4 slots x 32 lanes x 2 elements

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

// L2 prefetch of a ticket's tiles ahead of their TMA copies (no shared memory,
// no barrier): the ring holds only kFStages tiles, so without it too few
// bytes are in flight per SM to cover the loaded HBM latency.
__device__ __forceinline__ void l2_prefetch(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
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
// the epoch, every CTA reads it at start, and the last CTA to finish bumps it
// (after every CTA has read the old one).
// ---------------------------------------------------------------------------

constexpr int kEpochShift = 44;
// exchange words: sequence number (24 bits) << 40 | entry count (40 bits)
constexpr int kXSeqShift = 40;
constexpr uint64_t kXSeqMask = (1ull << 24) - 1;
constexpr uint64_t kXCountMask = (1ull << 40) - 1;

// The last CTA of an exchanging round-and-log (or an empty shard's one
// thread): this call's entry count into slot [parity][rank] of every rank's
// exchange buffer, tagged with this rank's next sequence number.
__device__ __forceinline__ void exchange_publish(const XPeers& xp, uint64_t total) {
  uint64_t* mine = xp.peers[xp.rank];
  const uint64_t seq = mine[0] + 1ull;
  mine[0] = seq;
  const uint64_t word = ((seq & kXSeqMask) << kXSeqShift) | (total & kXCountMask);
  const int par = (int)(seq & 1ull);
  for (int p = 0; p < xp.world; ++p) st_release_sys_u64(xp.peers[p] + 1 + par * xp.world + xp.rank, word);
}

__global__ void exchange_publish_kernel(const XPeers xp, uint64_t total) { exchange_publish(xp, total); }


constexpr uint64_t kEpochMask = (1ull << 20) - 1;
constexpr uint64_t kLBAgg = 1ull << 42;
constexpr uint64_t kLBInc = 2ull << 42;
constexpr uint64_t kLBVal = (1ull << 42) - 1;

__device__ __forceinline__ uint64_t lb_word(uint32_t epoch, uint64_t flag, uint64_t v) {
  return ((uint64_t)epoch << kEpochShift) | flag | (v & kLBVal);
}

// ---------------------------------------------------------------------------
// trainer, single pass: warp-specialised round-and-log with an in-kernel
// decoupled look-back
//
//   warps 0..7  compute: round every element of a 2048-element tile staged by
//               TMA, store y, and ballot two masks per 64-element group
//               (logged, UP) into a shared-memory mask slot -- no compaction,
//               no per-element shared stores;
//   warp 8      log writer: per 8192-element super-tile (4 tiles), popc the
//               masks, publish the super-tile count, look back over the
//               predecessors' epoch-tagged status words for its global log
//               position, and write the final (index << 1 | up) words
//               (staged in shared memory, then coalesced stores);
//   warp 9      producer: grabs super-tile tickets (atomic counter: a CTA
//               only ever waits on lower tickets, which running CTAs hold, so
//               the kernel cannot deadlock even when not all CTAs are
//               resident) and keeps kFStages TMA bulk copies in flight.
//
// Compute warps never wait on another CTA: the look-back latency is absorbed
// by kMaskSlots super-tiles of mask slack.  The CTA that finishes last
// resets the ticket counter and bumps the epoch for the next call.
// ---------------------------------------------------------------------------

#ifdef VT_TIMELINE  // development builds only (tools/timeline.py): per-CTA globaltimer stamps
__device__ uint64_t g_tl[1024][64];
__device__ __forceinline__ void tl_mark(int i) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  if (i < 64) g_tl[blockIdx.x & 1023][i] = t;
}
__device__ __forceinline__ void tl_put(int i, uint64_t v) { g_tl[blockIdx.x & 1023][i] = v; }
extern "C" int vt_debug_timeline(uint64_t* host) {
  return (int)cudaMemcpyFromSymbol(host, g_tl, sizeof(g_tl));
}
#define TL(i) tl_mark(i)
#define TLV(i, v) tl_put(i, v)
__device__ __forceinline__ uint64_t tl_now() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TWAIT(acc, stmt)            \
  do {                              \
    const uint64_t t_ = tl_now();   \
    stmt;                           \
    acc += tl_now() - t_;           \
  } while (0)
#else
#define TL(i)
#define TLV(i, v)
#define TWAIT(acc, stmt) stmt
#endif

// A ticket ("super-tile") is kSuper tiles: the unit of the dynamic schedule
// and of the look-back; kMaskSlots tickets of staged masks / rows give the
// look-back ~3 ordinals (~20 us) of slack.  Measured and not kept: 2-tile
// tickets with 6 slots (same slack in time, half the tail granularity):
// 2^26 78% vs 81%, 2^28 85% vs 90% -- twice the look-backs and ordinal
// overheads, and the tail spread (CTA speeds differ ~1.6x) barely moved.
constexpr int kSuper = kRLSuper;                 // tiles per super-tile / status word
#ifndef VT_MASK_SLOTS  // A/B
#define VT_MASK_SLOTS 3
#endif
#ifndef VT_RL_STAGES  // A/B
#define VT_RL_STAGES 3
#endif
constexpr int kMaskSlots = VT_MASK_SLOTS;        // super-tiles of masks in flight
constexpr int kFStages = VT_RL_STAGES;           // TMA ring depth of the fused kernel
constexpr int kRow = 64;                         // staged entries per warp-tile (else from masks)
// KEYS launches reuse a row's 128 bytes as kRowK {key, entry} pairs: 8-byte
// keys first, then the 16-bit entries
constexpr int kRowK = 12;
static_assert(kRowK * 10 <= kRow * 2, "keyed staging must fit a row");
constexpr int kRows = kSuper * kWarps;           // warp-tiles per super-tile
static_assert(kRows <= 32, "the log warp scans a super-tile's rows one per lane");
constexpr int kFCompute = kSThreads;             // 8 compute warps
constexpr int kFThreads = kFCompute + 64;        // + log warp + producer warp
constexpr int kLogWarp = kWarps;                 // warp 8
constexpr int kProdWarp = kWarps + 1;            // warp 9
constexpr int kGroups = kSTile / 64;             // 32 groups of 64 elements per tile

struct FusedHeader {
  uint32_t epoch;
  uint32_t ticket;  // next super-tile to hand out
  uint32_t done;    // CTAs finished
  uint32_t hwm;     // most status words any call has written
  uint64_t total;   // this call's log entries (written with the last super-tile's look-back)
  uint32_t pad[10];
};
static_assert(sizeof(FusedHeader) == 64, "the look-back words start at byte 64");

struct FusedSmem {
  double ring[kFStages][kSTile];
  uint4 masks[kMaskSlots][kSuper][kGroups];    // {logged even, logged odd, up even, up odd} lanes
  uint16_t rows[kMaskSlots][kRows][kRow];      // staged entries: super-tile offset << 1 | up
  uint32_t cnts[kMaskSlots][kRows];            // entries per warp-tile (tile-major)
  uint32_t rpos[kMaskSlots][kRows];            // log warp: row start inside the super-tile
  int64_t sbase[kMaskSlots];                   // log warp: global log position of the super-tile
  int64_t slot_id[kMaskSlots];
  int32_t slot_seg[kMaskSlots];   // batched kernel: tensor of slot_id[]
  int64_t ids[4];
  int32_t sids[4];                // batched kernel: tensor of ids[]
  uint32_t slot_cnt[kMaskSlots];  // (warps arrived << 24) + logged entries, by the compute warps
  uint64_t full[kFStages], empty[kFStages], mfull[kMaskSlots], ofull[kMaskSlots];
  uint32_t epoch;
};

struct RLFArgs {
  const double* x;
  int64_t n;
  Grid g;
  int thr32;
  void* out;
  int64_t num_tiles;
  int64_t num_super;  // tickets: n4 super-tiles of kSuper tiles, then one per remaining tile
  int64_t n4;
  FusedHeader* hdr;
  uint64_t* status;  // [num_super] epoch-tagged look-back words
  uint64_t* sparse;
  int64_t cap;
  int64_t global_base;
  const int64_t* cursor_in;
  int64_t* cursor_out;
  int64_t* counters;
  int32_t* err;
  const DevThr* dthr;
  const int32_t* gate;  // nullable: the kernel returns at once when *gate == 0
  uint64_t* keys;       // KEYS launches only
  XPeers xp;            // nullable peers: the last CTA publishes the call's entry count to every rank
};

// Ticket s -> its first tile and tile count: n4 super-tiles of kSuper tiles,
// then the remaining (< kSuper) tiles one per ticket.
__device__ __forceinline__ int64_t st_first(const RLFArgs& a, int64_t s) {
  return s < a.n4 ? s * kSuper : a.n4 * kSuper + (s - a.n4);
}
__device__ __forceinline__ int st_ntiles(const RLFArgs& a, int64_t s) { return s < a.n4 ? kSuper : 1; }

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// bit i of x (< 2^16) -> bit 2i
__device__ __forceinline__ uint32_t spread16(uint32_t x) {
  x = (x | (x << 8)) & 0x00ff00ffu;
  x = (x | (x << 4)) & 0x0f0f0f0fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

// One tile, compute warp: round, store, ballot.  `gx` non-null = partial
// tile read straight from global memory (elements >= lim are zero, which is
// on the grid and never logged).
template <int OUT, bool FAST, bool FULL, bool KEYS = false>
__device__ __forceinline__ uint32_t rlf_tile(const Grid& g, uint32_t c8, uint32_t w8, int thr32, const double* src,
                                         void* o, int lim, uint4* mslot, uint16_t* row, uint32_t sbase, int warp,
                                         int lane, uint32_t lt, uint32_t& err) {
  uint32_t wcnt = 0;
  // staged entry of this lane's first element in slot 0: super-tile offset << 1
  const uint32_t eb = (sbase + (uint32_t)(warp * kSWarpElems + lane * 2)) << 1;
#pragma unroll
  for (int j = 0; j < kSSlots; ++j) {
    const int e0 = warp * kSWarpElems + j * 64 + lane * 2;
    double2 xv;
    if (FULL) {
      xv = *reinterpret_cast<const double2*>(src + e0);
    } else {
      xv.x = (e0 < lim) ? src[e0] : 0.0;
      xv.y = (e0 + 1 < lim) ? src[e0 + 1] : 0.0;
    }
    bool l0, l1, u0, u1;
    if (FAST) {
      float f0 = __double2float_rn(xv.x), f1 = __double2float_rn(xv.y);
      const uint32_t lo0 = (uint32_t)__double2loint(xv.x), lo1 = (uint32_t)__double2loint(xv.y);
      const uint32_t hi0 = (uint32_t)__double2hiint(xv.x), hi1 = (uint32_t)__double2hiint(xv.y);
      // normal range: logged <=> thr32 < low29 < 2^29 - thr32 (SURVEY App. B.2,
      // d = min(low, 2^29 - low) split by the rounding side); the magnitude
      // rounded up iff the FP32 lsb differs from the FP64 bit 29, and the
      // code is UP iff that XOR the sign.
      l0 = (lo0 << 3) - c8 < w8;
      l1 = (lo1 << 3) - c8 < w8;
      const uint32_t fb0 = (uint32_t)__float_as_int(f0), fb1 = (uint32_t)__float_as_int(f1);
      u0 = (int32_t)((fb0 << 31) ^ (lo0 << 2) ^ fb0) < 0;
      u1 = (int32_t)((fb1 << 31) ^ (lo1 << 2) ^ fb1) < 0;
      // outside the FP32 normal range (subnormal results, overflow, inf / nan):
      // the whole warp takes the exact routine -- a warp-uniform branch keeps
      // the common path free of per-lane reconvergence and predicate spills
      if (__any_sync(0xffffffffu, outside_normal32(hi0 & 0x7fffffffu) | outside_normal32(hi1 & 0x7fffffffu))) {
        uint32_t c0, c1;
        f0 = round_dir32(xv.x, thr32, g.thr_sub, c0, err);
        f1 = round_dir32(xv.y, thr32, g.thr_sub, c1, err);
        l0 = c0 != 1u;
        l1 = c1 != 1u;
        u0 = c0 == 2u;
        u1 = c1 == 2u;
      }
      store2<OUT, FULL>(o, e0, lim, f0, f1);
    } else {
      uint32_t c0, c1;
      const uint64_t r0 = round_dir(xv.x, g, c0, err);
      const uint64_t r1 = round_dir(xv.y, g, c1, err);
      store2<OUT, FULL>(o, e0, lim, r0, r1);
      l0 = c0 != 1u;
      l1 = c1 != 1u;
      u0 = c0 == 2u;
      u1 = c1 == 2u;
    }
    const uint32_t L0 = __ballot_sync(0xffffffffu, l0), L1 = __ballot_sync(0xffffffffu, l1);
    const uint32_t U0 = __ballot_sync(0xffffffffu, u0), U1 = __ballot_sync(0xffffffffu, u1);
    if (lane == 0) mslot[warp * kSSlots + j] = make_uint4(L0, L1, U0, U1);
    // ballot-rank staging of the warp-tile's entries (first kRow only)
    const uint32_t r0 = wcnt + __popc(L0 & lt) + __popc(L1 & lt);
    const uint32_t r1 = r0 + (l0 ? 1u : 0u);
    const uint32_t v0 = eb + (uint32_t)(j * 128) + (u0 ? 1u : 0u);
    const uint32_t v1 = eb + (uint32_t)(j * 128 + 2) + (u1 ? 1u : 0u);
    if (KEYS) {  // also each entry's x (the adaptive selection then needs no gather of x)
      double* rk = reinterpret_cast<double*>(row);
      uint16_t* re = row + 4 * kRowK;
      if (l0 && r0 < (uint32_t)kRowK) {
        re[r0] = (uint16_t)v0;
        rk[r0] = xv.x;
      }
      if (l1 && r1 < (uint32_t)kRowK) {
        re[r1] = (uint16_t)v1;
        rk[r1] = xv.y;
      }
    } else {
      if (l0 && r0 < (uint32_t)kRow) row[r0] = (uint16_t)v0;
      if (l1 && r1 < (uint32_t)kRow) row[r1] = (uint16_t)v1;
    }
    wcnt += __popc(L0) + __popc(L1);
  }
  return wcnt;
}

// Look-back window: words per lane per round trip (window = 32 x this).
// One word per lane measured best (pair step, graph-timed, round-and-log /
// copy peak): 2^26 0.918 vs 0.870 for 4 words per lane, 2^28 1.022 vs
// 0.978, 2^24 0.63 vs 0.59; 8 and 16 words: 0.81 at 2^26.  Most look-backs
// find an inclusive prefix within the first few predecessors, and the wider
// window's loads (and re-loads while a predecessor is unpublished) only
// lengthen each round trip of the log warp, whose placement gates the row
// writes.  The poll interval (0-512 ns) does not matter.
#ifndef VT_LB_WORDS
#define VT_LB_WORDS 1
#endif
#ifndef VT_LB_SLEEP  // ns between look-back polls of an unpublished word
#define VT_LB_SLEEP 32
#endif

// Look-back by one warp over up to 32 * VT_LB_WORDS predecessors per round
// trip (the super-tile's own aggregate was published by its compute warps).
// Valid aggregates before the first unpublished word are kept, so every retry
// starts at the first word still missing.  Returns the exclusive prefix of
// super-tile s (same value in every lane) and publishes its inclusive prefix.
__device__ __forceinline__ int64_t lookback(uint64_t* status, int64_t s, uint64_t agg, uint32_t epoch,
                                               int lane) {
  constexpr int M = VT_LB_WORDS, WIN = 32 * M;
  if (s == 0) return 0;
  int64_t excl = 0, pred = s - 1;
  while (true) {
    uint64_t w[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int64_t idx = pred - (m * 32 + lane);
      w[m] = (idx >= 0) ? ld_relaxed_u64(status + idx) : lb_word(epoch, kLBInc, 0);
    }
    int p_inc = WIN, p_inv = WIN;  // first INC / first unpublished window position
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const bool valid = ((w[m] >> kEpochShift) & kEpochMask) == epoch;
      const uint64_t flag = valid ? ((w[m] >> 42) & 3ull) : 0ull;
      const uint32_t inc = __ballot_sync(0xffffffffu, flag == 2);
      const uint32_t inv = __ballot_sync(0xffffffffu, flag == 0);
      if (p_inc == WIN && inc) p_inc = m * 32 + __ffs(inc) - 1;
      if (p_inv == WIN && inv) p_inv = m * 32 + __ffs(inv) - 1;
    }
    const bool done = p_inc < p_inv;
    const int upto = done ? p_inc + 1 : p_inv;  // positions [0, upto) are summed
    uint64_t v = 0;
#pragma unroll
    for (int m = 0; m < M; ++m)
      if (m * 32 + lane < upto) v += w[m] & kLBVal;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    excl += (int64_t)v;
    if (done) break;
    pred -= upto;
    if (upto < WIN) __nanosleep(VT_LB_SLEEP);
  }
  if (lane == 0) st_relaxed_u64(status + s, lb_word(epoch, kLBInc, (uint64_t)excl + agg));
  return excl;
}

// Log warp, overflow path: warp-tile q had more than kRow entries, so its
// words come from the ballot masks, one 64-element group per step.
// `dst` = the row's first log position, `lim` = positions still in capacity.
__device__ __noinline__ void rlf_row_from_masks(const FusedSmem& S, int slot, int q, uint64_t gw, uint64_t* dst,
                                                int64_t lim, int lane, uint32_t lt, uint64_t* kdst = nullptr) {
  const int tile = q / kWarps, w = q % kWarps;
  uint32_t r = 0;
  for (int j = 0; j < kSSlots; ++j) {
    const uint4 m = S.masks[slot][tile][w * kSSlots + j];
    const bool l0 = (m.x >> lane) & 1u, l1 = (m.y >> lane) & 1u;
    const uint32_t r0 = r + __popc(m.x & lt) + __popc(m.y & lt);
    const uint64_t e0 = (uint64_t)(tile * kSTile + w * kSWarpElems + j * 64 + lane * 2);
    if (l0 && (int64_t)r0 < lim) dst[r0] = gw + (e0 << 1) + ((m.z >> lane) & 1u);
    const uint32_t r1 = r0 + (l0 ? 1u : 0u);
    if (l1 && (int64_t)r1 < lim) dst[r1] = gw + ((e0 + 1) << 1) + ((m.w >> lane) & 1u);
    if (kdst) {
      if (l0 && (int64_t)r0 < lim) kdst[r0] = kKeyMissing;
      if (l1 && (int64_t)r1 < lim) kdst[r1] = kKeyMissing;
    }
    r += __popc(m.x) + __popc(m.y);
  }
}

// Compute warp: once the log warp has placed ordinal k (super-tile s) of this
// CTA (ofull), write this warp's four rows of it -- staged entries by
// coalesced stores, an overflowing row from its ballot masks.
template <bool KEYS = false>
__device__ __forceinline__ void rlf_write_rows(const RLFArgs& a, FusedSmem& S, int64_t k, int64_t s, int warp,
                                               int lane, uint32_t lt) {
  const int slot = (int)(k % kMaskSlots);
  mbar_wait(S.ofull + slot, (uint32_t)((k / kMaskSlots) & 1));
  if (warp == 0 && lane == 0 && k + kMaskSlots < 14) TL(5 + 4 * (int)(k + kMaskSlots));
  const int64_t off = S.sbase[slot];
  uint64_t* dst = a.sparse + off;
  const int64_t lim = a.cap - off;  // positions >= lim are beyond the log capacity
  const uint64_t gw = (uint64_t)(a.global_base + st_first(a, s) * kSTile) << 1;
  const int nt = st_ntiles(a, s);
#pragma unroll
  for (int i = 0; i < kSuper; ++i) {
    const int q = i * kWarps + warp;
    if (i >= nt) break;
    const uint32_t cq = S.cnts[slot][q];
    const uint32_t pq = S.rpos[slot][q];
    if (KEYS) {
      uint64_t* kd = a.keys + off;
      if (cq <= (uint32_t)kRowK) {
        const uint64_t* rk = reinterpret_cast<const uint64_t*>(S.rows[slot][q]);
        const uint16_t* re = S.rows[slot][q] + 4 * kRowK;
        if ((uint32_t)lane < cq && (int64_t)(pq + lane) < lim) {
          dst[pq + lane] = gw + re[lane];
          kd[pq + lane] = rk[lane];
        }
      } else {
        rlf_row_from_masks(S, slot, q, gw, dst + pq, lim - (int64_t)pq, lane, lt, kd + pq);
      }
      continue;
    }
    if (cq <= (uint32_t)kRow) {
      const uint16_t* row = S.rows[slot][q];
      if ((uint32_t)lane < cq && (int64_t)(pq + lane) < lim) dst[pq + lane] = gw + row[lane];
      if (cq > 32u && (uint32_t)lane + 32u < cq && (int64_t)(pq + lane + 32) < lim)
        dst[pq + lane + 32] = gw + row[lane + 32];
    } else {
      rlf_row_from_masks(S, slot, q, gw, dst + pq, lim - (int64_t)pq, lane, lt);
    }
  }
}

template <int OUT, bool FAST, bool KEYS = false>
__global__ void __launch_bounds__(kFThreads, 3) rl_fused_kernel(const RLFArgs a) {
  extern __shared__ __align__(128) uint8_t smraw[];
  FusedSmem& S = *reinterpret_cast<FusedSmem*>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (a.gate && *a.gate == 0) return;
  if (tid == 0) {
    TL(0);
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    TLV(63, smid);
  }
  const int64_t full_tiles = a.n / kSTile;
  if (tid == 0) {
    for (int s = 0; s < kFStages; ++s) {
      mbar_init(S.full + s, 1);
      mbar_init(S.empty + s, kWarps);
    }
    for (int m = 0; m < kMaskSlots; ++m) {
      mbar_init(S.mfull + m, kWarps);
      mbar_init(S.ofull + m, 1);
    }
    for (int m = 0; m < kMaskSlots; ++m) S.slot_cnt[m] = 0u;
    fence_mbar_init();
    S.epoch = ((*(volatile uint32_t*)&a.hdr->epoch) + 1u) & (uint32_t)kEpochMask;
  }
  __syncthreads();

  if (warp == kProdWarp) {
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      // a ticket's whole tiles (from its tile `from` on) into L2 as soon as it is drawn
      auto prefetch = [&](int64_t s, int from) {
        if (s < 0 || s >= a.num_super) return;
        const int64_t t0 = st_first(a, s) + from;
        const int64_t t1 = min(st_first(a, s) + (int64_t)st_ntiles(a, s), full_tiles);
        if (t1 > t0) l2_prefetch(a.x + t0 * kSTile, (uint32_t)((t1 - t0) * kSTile * sizeof(double)));
      };
      int64_t s = (int64_t)atomicAdd(&a.hdr->ticket, 1u);
      uint32_t q = 0;  // ring sequence number (32-bit: q % 3 and q / 3 are one multiply-high)
      for (int64_t k = 0;; ++k) {
        if (s >= a.num_super) s = -1;
        int64_t nxt = -1;
        const int nt = (s >= 0) ? st_ntiles(a, s) : 1;
        const int64_t t0 = (s >= 0) ? st_first(a, s) : 0;
#pragma unroll 1
        for (int i = 0; i < nt; ++i, ++q) {
          const int st = (int)(q % kFStages);
          mbar_wait(S.empty + st, (uint32_t)(((q / kFStages) & 1) ^ 1));
          if (i == 0) S.ids[k & 3] = s;
          // draw the next ticket with this ordinal's last tile: late enough that
          // the grid runs dry together, early enough to hide the atomic
          if (i == nt - 1 && s >= 0) {
            nxt = (int64_t)atomicAdd(&a.hdr->ticket, 1u);
            if (VT_L2_PREFETCH) prefetch(nxt, 0);
          }
          const int64_t t = t0 + i;
          if (s >= 0 && t < full_tiles) {
            fence_proxy_async();
            tma_load(S.ring[st], a.x + t * kSTile, kSTile * sizeof(double), S.full + st, pol);
          } else {
            mbar_arrive(S.full + st);
          }
          // the first ticket: its tiles beyond the ring, once the ring's copies are issued
          if (VT_L2_PREFETCH && k == 0 && i == kFStages - 1) prefetch(s, kFStages);
        }
        if (s < 0) break;
        s = nxt;
      }
    }
    __syncwarp();
  } else if (warp == kLogWarp) {  // scan + look-back only; compute warps write the words
    const int64_t cur = a.cursor_in ? *a.cursor_in : 0;
    const uint32_t epoch = S.epoch;
    for (int64_t k = 0;; ++k) {
      const int slot = (int)(k % kMaskSlots);
      mbar_wait(S.mfull + slot, (uint32_t)((k / kMaskSlots) & 1));
      const int64_t s = S.slot_id[slot];
      if (s < 0) break;
      // lane = warp-tile (tile-major): exclusive position of each row inside the super-tile
      const uint32_t c = (lane < kRows && lane / kWarps < st_ntiles(a, s)) ? S.cnts[slot][lane] : 0u;
      uint32_t inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      const uint64_t agg = __shfl_sync(0xffffffffu, inc, 31);
      if (lane < kRows) S.rpos[slot][lane] = inc - c;
      const int64_t excl = lookback(a.status, s, agg, epoch, lane);
      if (lane == 0) {
        if (s == a.num_super - 1) {
          atomicAdd(reinterpret_cast<unsigned long long*>(a.counters), (unsigned long long)(excl + (int64_t)agg));
          if (a.cursor_out) *a.cursor_out = cur + excl + (int64_t)agg;
          a.hdr->total = (uint64_t)(excl + (int64_t)agg);
        }
        S.sbase[slot] = cur + excl;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(S.ofull + slot);
    }
  } else {  // compute warps
    uint32_t err = 0;
    Grid g = a.g;
    int thr32 = a.thr32;
    if (a.dthr) {
      g.thr = a.dthr->thr;
      g.thr_sub = a.dthr->thr_sub;
      thr32 = a.dthr->thr32;
    }
    const uint32_t lt = lanemask_lt();
    const uint32_t c8 = ((uint32_t)thr32 + 1u) << 3;
    const uint32_t w8 = (thr32 >= (1 << 28)) ? 0u : ((0x20000000u - 2u * (uint32_t)thr32 - 1u) << 3);
    const uint32_t epoch = S.epoch;
    int64_t hist[kMaskSlots];  // super-tile of ordinal kk at hist[kk % kMaskSlots]
    uint32_t q = 0;            // ring sequence number (32-bit, as the producer's)
    for (int64_t k = 0;; ++k) {
      // this warp's rows of ordinal k - kMaskSlots leave slot k % kMaskSlots before it is reused
      if (warp == 0 && lane == 0 && k < 14) TL(4 + 4 * (int)k);
      if (k >= kMaskSlots) rlf_write_rows<KEYS>(a, S, k - kMaskSlots, hist[k % kMaskSlots], warp, lane, lt);
      if (warp == 0 && lane == 0 && k < 14) TL(6 + 4 * (int)k);
      const int slot = (int)(k % kMaskSlots);
      int64_t s = -1, t0 = 0;
      int nt = 1;
      uint32_t wcnt = 0;
#pragma unroll 1
      for (int i = 0; i < nt; ++i, ++q) {
        const int st = (int)(q % kFStages);
        mbar_wait(S.full + st, (uint32_t)((q / kFStages) & 1));
        if (q == 0 && warp == 0 && lane == 0) TL(1);
        if (i == 0) {
          s = S.ids[k & 3];
          if (s < 0) {
            ++q;
            break;
          }
          nt = st_ntiles(a, s);
          t0 = st_first(a, s);
        }
        const int64_t t = t0 + i;
        {
          const int64_t tbase = t * kSTile;
          void* o = tile_out<OUT>(a.out, tbase);
          uint16_t* row = S.rows[slot][i * kWarps + warp];
          const uint32_t tc =
              (t < full_tiles)
                  ? rlf_tile<OUT, FAST, true, KEYS>(g, c8, w8, thr32, S.ring[st], o, kSTile, S.masks[slot][i], row,
                                              (uint32_t)(i * kSTile), warp, lane, lt, err)
                  : rlf_tile<OUT, FAST, false, KEYS>(g, c8, w8, thr32, a.x + tbase, o, (int)(a.n - tbase),
                                               S.masks[slot][i], row, (uint32_t)(i * kSTile), warp, lane, lt, err);
          if (lane == 0) S.cnts[slot][i * kWarps + warp] = tc;
          wcnt += tc;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(S.empty + st);
      }
      if (lane == 0) {
        if (s >= 0) {  // the last warp of the super-tile publishes its aggregate right away
          const uint32_t prev = atomicAdd(&S.slot_cnt[slot], wcnt + (1u << 24));
          if ((prev >> 24) == kWarps - 1) {
            const uint64_t agg = (prev & 0xffffffu) + wcnt;
            st_relaxed_u64(a.status + s, lb_word(epoch, s == 0 ? kLBInc : kLBAgg, agg));
            S.slot_cnt[slot] = 0u;
          }
        }
        if (warp == 0) S.slot_id[slot] = s;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(S.mfull + slot);
      if (warp == 0 && lane == 0 && k < 14) TL(7 + 4 * (int)k);
      if (warp == 0 && lane == 0 && s >= 0) {
        TL(58);
        TLV(56, (uint64_t)k + 1);
        TLV(55, (uint64_t)s);
      }
      if (warp == 0 && lane == 0 && s < 0) TL(60);
      if (s < 0) {  // drain ordinals k - kMaskSlots + 1 .. k - 1
        for (int64_t kk = k >= kMaskSlots - 1 ? k - kMaskSlots + 1 : 0; kk < k; ++kk) {
          rlf_write_rows<KEYS>(a, S, kk, hist[kk % kMaskSlots], warp, lane, lt);
          if (warp == 0 && lane == 0 && kk == k - 2) TL(61);
        }
        if (warp == 0 && lane == 0) TL(62);
        break;
      }
      hist[k % kMaskSlots] = s;
    }
    report_err(a.err, err);
  }

  if (tid == 0) TL(2);
  __syncthreads();
  __shared__ uint32_t s_last;
  if (tid == 0) {
    TL(3);
    __threadfence();
    s_last = atomicAdd(&a.hdr->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  // the last CTA out: every CTA has drawn its last ticket and read the epoch
  const uint32_t hwm = max(a.hdr->hwm, (uint32_t)a.num_super);
  if (S.epoch == (uint32_t)kEpochMask) {
    // the next epoch value wraps: clear every status word any call has
    // written, so no word from 2^20 calls ago can pass for a current one
    __threadfence();
    for (uint32_t i = tid; i < hwm; i += blockDim.x) a.status[i] = 0ull;
    __threadfence();
    __syncthreads();
  }
  if (tid == 0) {
    if (a.xp.peers) {
      // the exchange step fused into the kernel: the call's entry count goes
      // to every rank's exchange buffer over peer memory (NVLink), tagged
      // with this rank's exchange sequence number; slots alternate by parity
      // so a rank one exchange ahead cannot overwrite a slot still awaited
      __threadfence();
      exchange_publish(a.xp, *(volatile uint64_t*)&a.hdr->total);
    }
    a.hdr->ticket = 0u;
    a.hdr->done = 0u;
    a.hdr->hwm = hwm;
    a.hdr->epoch = S.epoch == (uint32_t)kEpochMask ? 0u : S.epoch;
    __threadfence();
  }
}

int exchange_publish_empty(XPeers xp, cudaStream_t st) {
  exchange_publish_kernel<<<1, 1, 0, st>>>(xp, 0ull);
  return vt_check_launch("exchange_publish_kernel");
}

// The other half of the exchange: wait until every rank's count for this
// rank's current sequence number has arrived (bounded spin: after
// timeout_ns the error bit VT_ERR_EXCHANGE is raised instead of hanging).
__global__ void counts_wait_kernel(const XPeers xp, int64_t* counts_out, int32_t* err, uint64_t timeout_ns) {
  const uint64_t* mine = xp.peers[xp.rank];
  const uint64_t seq = *(volatile const uint64_t*)mine;
  const int par = (int)(seq & 1ull);
  for (int q = threadIdx.x; q < xp.world; q += blockDim.x) {
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    uint64_t w;
    while (true) {
      w = ld_acquire_sys_u64(mine + 1 + par * xp.world + q);
      if ((w >> kXSeqShift) == (seq & kXSeqMask)) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        atomicOr(err, VT_ERR_EXCHANGE);
        w = 0;
        break;
      }
      __nanosleep(100);
    }
    counts_out[q] = (int64_t)(w & kXCountMask);
  }
}

int counts_wait(XPeers xp, int64_t* counts_out, int32_t* err, cudaStream_t st) {
  counts_wait_kernel<<<1, 32, 0, st>>>(xp, counts_out, err, 10ull * 1000 * 1000 * 1000);
  return vt_check_launch("counts_wait_kernel");
}

// ---------------------------------------------------------------------------
// trainer, batched: the same warp-specialised pipeline over many tensors in
// one launch (configs[2]: 161 tensors of 32 K .. 25.7 M elements).  One
// persistent grid streams every tensor back to back, so the per-tensor ramp
// and drain of a separate launch is paid once per batch.
//
// Tickets run over all tensors: tensor j owns [tick0_j, tick0_j + its
// super-tiles) and the look-back words at the same offsets, so the look-back
// of a ticket stops at its tensor's first super-tile (local ticket 0 = INC 0)
// and every tensor's log is ordered and positioned on its own.  A gated-off
// tensor (fallback pass, *gate == 0) is skipped whole: the producer that
// draws one of its tickets raises the counter to the next tensor's first
// ticket (atomicMax), so only the tickets of skipped tensors are ever jumped.
// ---------------------------------------------------------------------------

// the fields rlf_write_rows / st_first / st_ntiles read, for tensor j
__device__ __forceinline__ RLFArgs seg_view(const RLBatch& b, int j) {
  RLFArgs v{};
  const RLSeg& sg = b.seg[j];
  v.x = sg.x;
  v.n = sg.n;
  v.num_tiles = (sg.n + kSTile - 1) / kSTile;
  v.n4 = v.num_tiles / kSuper;
  v.num_super = v.n4 + v.num_tiles % kSuper;
  v.sparse = sg.sparse;
  v.cap = sg.cap;
  v.global_base = sg.global_base;
  v.keys = sg.keys;
  return v;
}

template <int OUT, bool FAST, bool KEYS>
__global__ void __launch_bounds__(kFThreads, 3) rl_batch_kernel(const __grid_constant__ RLBatch b) {
  extern __shared__ __align__(128) uint8_t smraw[];
  FusedSmem& S = *reinterpret_cast<FusedSmem*>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (b.any && *b.any == 0) return;
  FusedHeader* hdr = static_cast<FusedHeader*>(b.hdr);
  uint64_t* status = reinterpret_cast<uint64_t*>(static_cast<uint8_t*>(b.hdr) + 64);
  if (tid == 0) {
    for (int s = 0; s < kFStages; ++s) {
      mbar_init(S.full + s, 1);
      mbar_init(S.empty + s, kWarps);
    }
    for (int m = 0; m < kMaskSlots; ++m) {
      mbar_init(S.mfull + m, kWarps);
      mbar_init(S.ofull + m, 1);
    }
    for (int m = 0; m < kMaskSlots; ++m) S.slot_cnt[m] = 0u;
    fence_mbar_init();
    S.epoch = ((*(volatile uint32_t*)&hdr->epoch) + 1u) & (uint32_t)kEpochMask;
  }
  __syncthreads();

  if (warp == kProdWarp) {
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      // the next ticket of a tensor that runs (skips gated-off tensors whole);
      // a CTA's tickets ascend, so its tensor index only moves forward
      int jc = 0;
      auto draw = [&]() -> int64_t {
        while (true) {
          const int64_t s = (int64_t)atomicAdd(&hdr->ticket, 1u);
          if (s >= b.total) return -1;
          while (jc + 1 < b.nseg && b.seg[jc + 1].tick0 <= s) ++jc;
          const int32_t* gate = b.seg[jc].gate;
          if (!gate || *gate != 0) return s;
          const int64_t next = jc + 1 < b.nseg ? b.seg[jc + 1].tick0 : b.total;
          atomicMax(&hdr->ticket, (uint32_t)next);
        }
      };
      // a ticket's tensor and tiles, looked up once it is drawn (off the path
      // from a free ring slot to the next copy)
      struct TicketInfo {
        int64_t s, t0, full_tiles;
        const double* x;
        int nt, j;
      };
      auto lookup = [&](int64_t s) {
        TicketInfo ti{s, 0, 0, nullptr, 1, jc};  // draw() left jc at the tensor of s
        if (s >= 0) {
          const RLFArgs v = seg_view(b, jc);
          const int64_t ls = s - b.seg[jc].tick0;
          ti.nt = st_ntiles(v, ls);
          ti.t0 = st_first(v, ls);
          ti.full_tiles = v.n / kSTile;
          ti.x = v.x;
        }
        return ti;
      };
      // a ticket's whole tiles into L2 as soon as it is drawn (as rl_fused_kernel)
      auto prefetch = [&](const TicketInfo& ti) {
        if (!VT_L2_PREFETCH || ti.s < 0) return;
        const int64_t t1 = min(ti.t0 + (int64_t)ti.nt, ti.full_tiles);
        if (t1 > ti.t0) l2_prefetch(ti.x + ti.t0 * kSTile, (uint32_t)((t1 - ti.t0) * kSTile * sizeof(double)));
      };
      TicketInfo cur = lookup(draw());
      prefetch(cur);
      uint32_t q = 0;  // ring sequence number (32-bit)
      for (int64_t k = 0;; ++k) {
        const int64_t s = cur.s;
        const int nt = cur.nt, j = cur.j;
        const int64_t t0 = cur.t0, full_tiles = cur.full_tiles;
        const double* x = cur.x;
        TicketInfo nxt{-1, 0, 0, nullptr, 1, 0};
#pragma unroll 1
        for (int i = 0; i < nt; ++i, ++q) {
          const int st = (int)(q % kFStages);
          mbar_wait(S.empty + st, (uint32_t)(((q / kFStages) & 1) ^ 1));
          if (i == 0) {
            S.ids[k & 3] = s;
            S.sids[k & 3] = j;
          }
          const int64_t t = t0 + i;
          if (s >= 0 && t < full_tiles) {
            fence_proxy_async();
            tma_load(S.ring[st], x + t * kSTile, kSTile * sizeof(double), S.full + st, pol);
          } else {
            mbar_arrive(S.full + st);
          }
          // the next ticket after this tile's copy is in flight: draw() waits
          // on its atomic and the tensor lookup, the TMA must not
          if (i == nt - 1 && s >= 0) {
            nxt = lookup(draw());
            prefetch(nxt);
          }
        }
        if (s < 0) break;
        cur = nxt;
      }
    }
    __syncwarp();
  } else if (warp == kLogWarp) {
    const uint32_t epoch = S.epoch;
    for (int64_t k = 0;; ++k) {
      const int slot = (int)(k % kMaskSlots);
      mbar_wait(S.mfull + slot, (uint32_t)((k / kMaskSlots) & 1));
      const int64_t s = S.slot_id[slot];
      if (s < 0) break;
      const int j = S.slot_seg[slot];
      const RLSeg& sg = b.seg[j];
      const RLFArgs v = seg_view(b, j);
      const int64_t ls = s - sg.tick0;
      const uint32_t c = (lane < kRows && lane / kWarps < st_ntiles(v, ls)) ? S.cnts[slot][lane] : 0u;
      uint32_t inc = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += u;
      }
      const uint64_t agg = __shfl_sync(0xffffffffu, inc, 31);
      if (lane < kRows) S.rpos[slot][lane] = inc - c;
      const int64_t excl = lookback(status + sg.tick0, ls, agg, epoch, lane);
      if (lane == 0) {
        if (ls == v.num_super - 1) {
          if (sg.counters)
            atomicAdd(reinterpret_cast<unsigned long long*>(sg.counters), (unsigned long long)(excl + (int64_t)agg));
          if (sg.cursor_out) *sg.cursor_out = excl + (int64_t)agg;
        }
        S.sbase[slot] = excl;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(S.ofull + slot);
    }
  } else {  // compute warps
    const uint32_t lt = lanemask_lt();
    const uint32_t epoch = S.epoch;
    int64_t hist[kMaskSlots];  // ticket of ordinal kk at hist[kk % kMaskSlots]
    int histj[kMaskSlots];     // and its tensor
    uint32_t q = 0;  // ring sequence number (32-bit)
    auto write_rows = [&](int64_t kk, int64_t s, int j) {
      rlf_write_rows<KEYS>(seg_view(b, j), S, kk, s - b.seg[j].tick0, warp, lane, lt);
    };
    for (int64_t k = 0;; ++k) {
      if (k >= kMaskSlots) write_rows(k - kMaskSlots, hist[k % kMaskSlots], histj[k % kMaskSlots]);
      const int slot = (int)(k % kMaskSlots);
      int64_t s = -1, t0 = 0, ls = 0;
      int nt = 1, j = 0;
      uint32_t wcnt = 0;
      // the ordinal's tensor constants, loaded once per super-tile
      Grid g = b.g;
      int thr32 = 0;
      uint32_t c8 = 0, w8 = 0;
      int64_t full_tiles = 0;
      const RLSeg* sgp = b.seg;
#pragma unroll 1
      for (int i = 0; i < nt; ++i, ++q) {
        const int st = (int)(q % kFStages);
        mbar_wait(S.full + st, (uint32_t)((q / kFStages) & 1));
        if (i == 0) {
          s = S.ids[k & 3];
          if (s < 0) {
            ++q;
            break;
          }
          j = S.sids[k & 3];
          sgp = b.seg + j;
          ls = s - sgp->tick0;
          const RLFArgs v = seg_view(b, j);
          nt = st_ntiles(v, ls);
          t0 = st_first(v, ls);
          thr32 = sgp->thr32;
          g.thr = sgp->thr;
          g.thr_sub = sgp->thr_sub;
          if (sgp->dthr) {
            g.thr = sgp->dthr->thr;
            g.thr_sub = sgp->dthr->thr_sub;
            thr32 = sgp->dthr->thr32;
          }
          c8 = ((uint32_t)thr32 + 1u) << 3;
          w8 = (thr32 >= (1 << 28)) ? 0u : ((0x20000000u - 2u * (uint32_t)thr32 - 1u) << 3);
          full_tiles = sgp->n / kSTile;
        }
        const RLSeg& sg = *sgp;
        uint32_t err = 0;
        const int64_t t = t0 + i;
        const int64_t tbase = t * kSTile;
        void* o = tile_out<OUT>(sg.out, tbase);
        uint16_t* row = S.rows[slot][i * kWarps + warp];
        const uint32_t tc =
            (t < full_tiles)
                ? rlf_tile<OUT, FAST, true, KEYS>(g, c8, w8, thr32, S.ring[st], o, kSTile, S.masks[slot][i], row,
                                                  (uint32_t)(i * kSTile), warp, lane, lt, err)
                : rlf_tile<OUT, FAST, false, KEYS>(g, c8, w8, thr32, sg.x + tbase, o, (int)(sg.n - tbase),
                                                   S.masks[slot][i], row, (uint32_t)(i * kSTile), warp, lane, lt, err);
        if (lane == 0) S.cnts[slot][i * kWarps + warp] = tc;
        wcnt += tc;
        report_err(sg.err, err);
        __syncwarp();
        if (lane == 0) mbar_arrive(S.empty + st);
      }
      if (lane == 0) {
        if (s >= 0) {
          const uint32_t prev = atomicAdd(&S.slot_cnt[slot], wcnt + (1u << 24));
          if ((prev >> 24) == kWarps - 1) {
            const uint64_t agg = (prev & 0xffffffu) + wcnt;
            st_relaxed_u64(status + s, lb_word(epoch, ls == 0 ? kLBInc : kLBAgg, agg));
            S.slot_cnt[slot] = 0u;
          }
        }
        if (warp == 0) {
          S.slot_id[slot] = s;
          S.slot_seg[slot] = j;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(S.mfull + slot);
      if (s < 0) {
        for (int64_t kk = k >= kMaskSlots - 1 ? k - kMaskSlots + 1 : 0; kk < k; ++kk)
          write_rows(kk, hist[kk % kMaskSlots], histj[kk % kMaskSlots]);
        break;
      }
      hist[k % kMaskSlots] = s;
      histj[k % kMaskSlots] = j;
    }
  }

  __syncthreads();
  __shared__ uint32_t s_last;
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(&hdr->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  const uint32_t hwm = max(hdr->hwm, (uint32_t)b.total);
  if (S.epoch == (uint32_t)kEpochMask) {
    __threadfence();
    for (uint32_t i = tid; i < hwm; i += blockDim.x) status[i] = 0ull;
    __threadfence();
    __syncthreads();
  }
  if (tid == 0) {
    hdr->ticket = 0u;
    hdr->done = 0u;
    hdr->hwm = hwm;
    hdr->epoch = S.epoch == (uint32_t)kEpochMask ? 0u : S.epoch;
    __threadfence();
  }
}

// ---------------------------------------------------------------------------
// auditor: streaming replay against the sparse log
// ---------------------------------------------------------------------------

struct RPArgs {
  const double* x;
  int64_t n;
  Grid g;
  const uint64_t* log;  // sparse words; PACKED: the .vtrl payload (bytes)
  int64_t n_words;      // sparse words; PACKED: payload bytes
  int64_t log_base;     // global index of element 0; PACKED: its stream position in the payload
  void* out;
  int64_t num_tiles;
  int64_t num_super;  // tickets, as for the trainer: n4 chunks of kSuper tiles, then single tiles
  int64_t n4;
  FusedHeader* hdr;   // ticket + done counters
  int64_t* counters;
  int32_t* err;
};

constexpr int kRStages = 4;
constexpr int kRThreads = kSThreads + 64;  // 8 compute warps + producer warp + log-search warp
constexpr int kRIds = 8;                   // ordinals in flight between the three roles

struct ReplaySmem {
  double ring[kRStages][kSTile];
  uint8_t cmap[kSTile];             // code map of the current tile, all 1 between tiles (sparse)
  uint16_t lut[256];                // PACKED: a payload byte's five base-3 digits, 2 bits each; bit 15 = invalid
  int64_t ids[kRIds], curs[kRIds];  // ticket (producer) and first log word (search warp) of ordinal k
  uint64_t full[kRStages], empty[kRStages], tfull[kRIds], nfull[kRIds];
  uint32_t red[kWarps];
};

constexpr int kRSuper = 4;  // tiles per replay ticket (no look-back: only the dynamic schedule)
__device__ __forceinline__ int64_t rp_first(const RPArgs& a, int64_t s) {
  return s < a.n4 ? s * kRSuper : a.n4 * kRSuper + (s - a.n4);
}
__device__ __forceinline__ int rp_ntiles(const RPArgs& a, int64_t s) { return s < a.n4 ? kRSuper : 1; }

// named barrier over the 256 compute threads (barrier 0 is the whole CTA)
__device__ __forceinline__ void compute_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ int compute_sync_count(bool p) {
  int r;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %1, 0;\n\tbar.red.popc.u32 %0, 1, 256, q;\n}"
               : "=r"(r)
               : "r"((uint32_t)p)
               : "memory");
  return r;
}

// lower_bound over the sorted word indices by one warp, 32 probes per step;
// the answer is known to lie in [lo, hi]
__device__ int64_t warp_lower_bound(const uint64_t* w, int64_t lo, int64_t hi, int64_t key, int lane) {
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

// First log word with index >= key.  Entries are spread over the tensor's
// index range: for uniformly scattered entries the word count below key is
// binomial around the interpolated position, with sd <= sqrt(nw) / 2, so 32
// probes spaced sqrt(nw) / 8 (+-4 sd) usually bracket the answer; otherwise
// (skewed logs) the bracket is one side of the probes.  Then the 32-ary search.
// Measured and not kept: two-round forms (128 probes then the bracket, or 32
// probes then the whole bracket in one round of up to 12 loads per lane):
// the first search of each CTA still waits behind the TMA burst, and the
// extra scattered probes cost 1-8% at 2^26.
__device__ int64_t log_lower_bound(const RPArgs& a, int64_t key, int lane) {
  const int64_t nw = a.n_words;
  if (nw == 0) return 0;
  const int64_t g = (int64_t)((double)(key - a.log_base) / (double)a.n * (double)nw);
  const int64_t d = std::max<int64_t>(64, (int64_t)(sqrt((double)nw) * 0.125));
  const int64_t p = g + (int64_t)(lane - 16) * d;
  const bool lt = (p < 0) || (p < nw && (int64_t)(__ldg(a.log + p) >> 1) < key);
  const int c = __popc(__ballot_sync(0xffffffffu, lt));
  const int64_t p0 = g - 16 * d;
  int64_t lo = (c == 0) ? 0 : p0 + (int64_t)(c - 1) * d + 1;
  int64_t hi = (c == 32) ? nw : p0 + (int64_t)c * d;
  lo = std::max<int64_t>(lo, 0);
  hi = std::min<int64_t>(std::max<int64_t>(hi, lo), nw);
  return warp_lower_bound(a.log, lo, hi, key, lane);
}

// One tile of the auditor pass.  Each thread reads the codes of its own
// elements from the map and resets them to 1, so the map is all-ignore
// again for the next tile without an extra barrier.
template <int OUT, bool FAST, bool FULL, bool RESET = true>
__device__ __forceinline__ uint32_t rp_tile(const RPArgs& a, const double* src, uint8_t* cs, void* o, int lim,
                                            int warp, int lane, uint32_t& err) {
  uint32_t flips = 0;
#pragma unroll
  for (int j = 0; j < kSSlots; ++j) {
    const int e0 = warp * kSWarpElems + j * 64 + lane * 2;
    const double2 xv = *reinterpret_cast<const double2*>(src + e0);
    uint16_t* cp = reinterpret_cast<uint16_t*>(cs + e0);
    const uint32_t cc = *cp;
    if (RESET) *cp = 0x0101;
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
  const int cnt = compute_sync_count(in);
  if (in) {
    const bool ordered = (i == 0) || ((prev >> 1) < (w >> 1));
    if (idx >= key0 && ordered && (int)threadIdx.x < cnt) cs[idx - key0] = (w & 1ull) ? 2 : 0;
    else err |= VT_ERR_BAD_SPARSE;
  }
  return cnt;
}

// PACKED (.vtrl payload, roundlog.py:67-82): the three payload bytes holding
// the codes of this thread's 8 consecutive elements [e8, e8 + 8) of a tile,
// loaded a tile ahead (they sit at stream positions pos .. pos + 7).
struct PackedWin {
  uint32_t b0, b1, b2;
  int ph;   // digit of the first element inside b0
  int nv;   // valid elements of the 8
};

__device__ __forceinline__ PackedWin packed_load(const RPArgs& a, int64_t tbase, int tid) {
  PackedWin w{1u, 1u, 1u, 0, 0};
  const int64_t e = tbase + (int64_t)tid * 8;
  w.nv = (int)std::max<int64_t>(0, std::min<int64_t>(8, a.n - e));
  if (w.nv == 0) return w;
  const int64_t pos = a.log_base + e;
  const int64_t bi = pos / 5;
  w.ph = (int)(pos - 5 * bi);
  const uint8_t* p = reinterpret_cast<const uint8_t*>(a.log);
  const int last = (w.ph + w.nv - 1) / 5;  // byte offset of the last valid digit
  w.b0 = bi < a.n_words ? (uint32_t)__ldg(p + bi) : 255u;
  if (last >= 1) w.b1 = bi + 1 < a.n_words ? (uint32_t)__ldg(p + bi + 1) : 255u;
  if (last >= 2) w.b2 = bi + 2 < a.n_words ? (uint32_t)__ldg(p + bi + 2) : 255u;
  return w;
}

// decode the window into the code map: 8 code bytes, one 8-byte store
__device__ __forceinline__ void packed_decode(const PackedWin& w, const uint16_t* lut, uint8_t* cs, int tid,
                                              uint32_t& err) {
  if (w.nv == 0) {
    *reinterpret_cast<uint2*>(cs + tid * 8) = make_uint2(0x01010101u, 0x01010101u);
    return;
  }
  const uint32_t l0 = lut[w.b0 & 0xffu], l1 = lut[w.b1 & 0xffu], l2 = lut[w.b2 & 0xffu];
  if ((l0 | l1 | l2) & 0x8000u) err |= VT_ERR_BAD_LOG_BYTE;  // a byte > 242 (corrupt log byte)
  // 15 digits of 2 bits, starting at this thread's first element
  uint32_t c = ((l0 & 0x3ffu) | ((l1 & 0x3ffu) << 10) | ((l2 & 0x3ffu) << 20)) >> (2 * w.ph);
  if (w.nv < 8) c = (c & ((1u << (2 * w.nv)) - 1u)) | (0x5555u & ~((1u << (2 * w.nv)) - 1u));  // past n: code 1
  auto spread = [](uint32_t x) {  // four 2-bit codes -> four bytes
    return (x & 3u) | ((x & 0xcu) << 6) | ((x & 0x30u) << 12) | ((x & 0xc0u) << 18);
  };
  *reinterpret_cast<uint2*>(cs + tid * 8) = make_uint2(spread(c & 0xffu), spread((c >> 8) & 0xffu));
}

// Auditor kernel, warp-specialised like the trainer's: the producer warp
// draws tickets (super-tiles of kSuper tiles) and keeps kRStages TMA copies in
// flight; the search warp finds each ordinal's first log word
// (log_lower_bound) as soon as its ticket is known and publishes it (nfull);
// the compute warps scatter each tile's log slice into the code map and
// replay the tile, prefetching the next tile's window of log words while the
// current one computes (across ordinals too, through nfull).
template <int OUT, bool FAST, bool PACKED = false>
__global__ void __launch_bounds__(kRThreads, 3) rp_fused_kernel(const RPArgs a) {
  extern __shared__ __align__(128) uint8_t smraw[];
  ReplaySmem& S = *reinterpret_cast<ReplaySmem*>(smraw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t full_tiles = a.n / kSTile;
  if (tid == 0) TL(0);
  if (tid < kSThreads) reinterpret_cast<uint2*>(S.cmap)[tid] = make_uint2(0x01010101u, 0x01010101u);
  if (PACKED && tid < 256) {
    uint32_t t = (uint32_t)tid, v = 0;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      v |= (t % 3u) << (2 * k);
      t /= 3u;
    }
    S.lut[tid] = (uint16_t)(v | (tid > 242 ? 0x8000u : 0u));
  }
  if (tid == 0) {
    for (int st = 0; st < kRStages; ++st) {
      mbar_init(S.full + st, 1);
      mbar_init(S.empty + st, 1);
    }
    for (int m = 0; m < kRIds; ++m) {
      mbar_init(S.tfull + m, 1);
      mbar_init(S.nfull + m, 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kWarps) {  // producer: tickets and TMA
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      // a ticket's whole tiles into L2 as soon as it is drawn -- off: the
      // replay's 4-stage ring already covers the latency, and the prefetch
      // cost it 2-8% (2^24: 0.66 vs 0.75 of the copy peak; the round-and-log
      // gains 8-10%, see rl_fused_kernel)
      auto prefetch = [&](int64_t s) {
        if (!VT_RP_L2_PREFETCH || s < 0 || s >= a.num_super) return;
        const int64_t t0 = rp_first(a, s);
        const int64_t t1 = min(t0 + (int64_t)rp_ntiles(a, s), full_tiles);
        if (t1 > t0) l2_prefetch(a.x + t0 * kSTile, (uint32_t)((t1 - t0) * kSTile * sizeof(double)));
      };
      int64_t s = (int64_t)atomicAdd(&a.hdr->ticket, 1u);
      prefetch(s);
      int64_t q = 0;
      for (int64_t k = 0;; ++k) {
        if (s >= a.num_super) s = -1;
        S.ids[k % kRIds] = s;
        mbar_arrive(S.tfull + (k % kRIds));
        // the first ticket's log search (2-3 dependent loads) runs before this
        // CTA's TMA burst instead of queueing behind it: 2^22 0.37 vs 0.33 of
        // the copy peak, no change from 2^24 up
        if (k == 0) mbar_wait(S.nfull, 0u);
        const int nt = (s >= 0) ? rp_ntiles(a, s) : 1;
        const int64_t t0 = (s >= 0) ? rp_first(a, s) : 0;
        int64_t nxt = -1;
#pragma unroll 1
        for (int i = 0; i < nt; ++i, ++q) {
          const int st = (int)(q % kRStages);
          mbar_wait(S.empty + st, (uint32_t)(((q / kRStages) & 1) ^ 1));
          if (i == nt - 1 && s >= 0) {
            nxt = (int64_t)atomicAdd(&a.hdr->ticket, 1u);
            prefetch(nxt);
          }
          const int64_t t = t0 + i;
          if (s >= 0 && t < full_tiles) {
            fence_proxy_async();
            tma_load(S.ring[st], a.x + t * kSTile, kSTile * sizeof(double), S.full + st, pol);
          } else {
            mbar_arrive(S.full + st);
          }
        }
        if (s < 0) break;
        s = nxt;
      }
    }
    __syncwarp();
  } else if (warp == kWarps + 1) {  // log search: each ordinal's first log word, ahead of the compute warps
    for (int64_t k = 0;; ++k) {
      const int m = (int)(k % kRIds);
      mbar_wait(S.tfull + m, (uint32_t)((k / kRIds) & 1));
      const int64_t s = S.ids[m];
      const int64_t cur = (!PACKED && s >= 0) ? log_lower_bound(a, a.log_base + rp_first(a, s) * kSTile, lane) : 0;
      if (lane == 0) {
        S.curs[m] = cur;
        mbar_arrive(S.nfull + m);
      }
      if (s < 0) break;
    }
  } else {  // compute warps
    uint32_t err = 0, flips = 0;
    int64_t q = 0;
    uint64_t tw_top = 0, tw_next = 0, tw_full = 0;  // timeline builds: ns waited (thread 0)
    (void)tw_top, (void)tw_next, (void)tw_full;
    uint64_t pw = 0, pp = 0;  // prefetched window for the next tile (word at cur + tid, its predecessor)
    PackedWin pwin{1u, 1u, 1u, 0, 0};  // PACKED: the next tile's payload bytes
    bool pref = false;
    int64_t cur = 0;
    for (int64_t k = 0;; ++k) {
      TWAIT(tw_top, mbar_wait(S.nfull + (k % kRIds), (uint32_t)((k / kRIds) & 1)));
      const int64_t s = S.ids[k % kRIds];
      if (s < 0) break;
      const int nt = rp_ntiles(a, s);
      const int64_t t0 = rp_first(a, s);
      if (PACKED) {
#pragma unroll 1
        for (int i = 0; i < nt; ++i, ++q) {
          const int64_t t = t0 + i;
          const int64_t tbase = t * kSTile;
          // this tile's payload window (loaded a tile ahead, except the first)
          if (!pref) pwin = packed_load(a, tbase, tid);
          const PackedWin cw = pwin;
          // the next tile of this ticket, or of the next ticket once it is known
          int64_t nbase = -1;
          if (i + 1 < nt) {
            nbase = tbase + kSTile;
          } else {
            mbar_wait(S.nfull + ((k + 1) % kRIds), (uint32_t)(((k + 1) / kRIds) & 1));
            const int64_t s2 = S.ids[(k + 1) % kRIds];
            if (s2 >= 0) nbase = rp_first(a, s2) * kSTile;
          }
          pref = nbase >= 0;
          if (pref) pwin = packed_load(a, nbase, tid);
          packed_decode(cw, S.lut, S.cmap, tid, err);
          const int st = (int)(q % kRStages);
          const double* src = S.ring[st];
          mbar_wait(S.full + st, (uint32_t)((q / kRStages) & 1));
          if (t >= full_tiles) {  // partial last tile: plain loads into the (unused) ring slot
            double* dst = S.ring[st];
            for (int e = tid; e < kSTile; e += kSThreads) dst[e] = (tbase + e < a.n) ? a.x[tbase + e] : 0.0;
          }
          compute_sync();  // code map decoded, x tile resident
          void* o = tile_out<OUT>(a.out, tbase);
          flips += (t < full_tiles)
                       ? rp_tile<OUT, FAST, true, false>(a, src, S.cmap, o, kSTile, warp, lane, err)
                       : rp_tile<OUT, FAST, false, false>(a, src, S.cmap, o, (int)(a.n - tbase), warp, lane, err);
          compute_sync();  // ring slot and code map consumed
          if (tid == 0) mbar_arrive(S.empty + st);
        }
        continue;
      }
      if (!pref) {
        cur = S.curs[k % kRIds];
        const int64_t i = cur + tid;
        pw = pp = 0;
        if (i < a.n_words) {
          pw = __ldg(a.log + i);
          pp = i ? __ldg(a.log + i - 1) : 0ull;
        }
      }
      if (s == 0 && tid == 0) a.counters[1] = cur;
#pragma unroll 1
      for (int i = 0; i < nt; ++i, ++q) {
        const int64_t t = t0 + i;
        const int64_t tbase = t * kSTile;
        const int64_t key0 = a.log_base + tbase;
        const int64_t key1 = a.log_base + std::min<int64_t>(tbase + kSTile, a.n);
        int cnt = scatter_window(S.cmap, pw, pp, cur + tid, a.n_words, key0, key1, err);
        cur += cnt;
        while (cnt == kSThreads) {  // more than one window of entries in this tile
          const int64_t j = cur + tid;
          uint64_t w = 0, p = 0;
          if (j < a.n_words) {
            w = __ldg(a.log + j);
            p = __ldg(a.log + j - 1);
          }
          cnt = scatter_window(S.cmap, w, p, j, a.n_words, key0, key1, err);
          cur += cnt;
        }
        // prefetch the next tile's window while this tile computes
        pref = true;
        int64_t ncur = cur;
        if (i == nt - 1) {  // next ordinal: its first word comes from the producer's search
          TWAIT(tw_next, mbar_wait(S.nfull + ((k + 1) % kRIds), (uint32_t)(((k + 1) / kRIds) & 1)));
          if (S.ids[(k + 1) % kRIds] >= 0) ncur = S.curs[(k + 1) % kRIds];
          if (s == a.num_super - 1 && tid == 0) a.counters[2] = cur;
        }
        {
          const int64_t j = ncur + tid;
          pw = pp = 0;
          if (j < a.n_words) {
            pw = __ldg(a.log + j);
            pp = j ? __ldg(a.log + j - 1) : 0ull;
          }
        }
        const int st = (int)(q % kRStages);
        const double* src = S.ring[st];
        if (t < full_tiles) {
          TWAIT(tw_full, mbar_wait(S.full + st, (uint32_t)((q / kRStages) & 1)));
        } else {  // partial last tile: plain loads into the (unused) ring slot
          mbar_wait(S.full + st, (uint32_t)((q / kRStages) & 1));
          double* dst = S.ring[st];
          for (int e = tid; e < kSTile; e += kSThreads) dst[e] = (tbase + e < a.n) ? a.x[tbase + e] : 0.0;
        }
        if (tid == 0 && q == 0) TL(1);
        compute_sync();  // code map complete, x tile resident
        void* o = tile_out<OUT>(a.out, tbase);
        flips += (t < full_tiles) ? rp_tile<OUT, FAST, true>(a, src, S.cmap, o, kSTile, warp, lane, err)
                                  : rp_tile<OUT, FAST, false>(a, src, S.cmap, o, (int)(a.n - tbase), warp, lane, err);
        compute_sync();  // ring slot consumed, code map reset
        if (tid == 0) mbar_arrive(S.empty + (int)(q % kRStages));
        cur = ncur;
      }
    }
    report_err(a.err, err);
    if (tid == 0) {
      TLV(10, tw_top);
      TLV(11, tw_next);
      TLV(12, tw_full);
      TLV(13, (uint64_t)q);
    }
    uint32_t v = flips;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) S.red[warp] = v;
    compute_sync();
    if (tid == 0) {
      uint32_t tot = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) tot += S.red[w];
      if (tot) atomicAdd(reinterpret_cast<unsigned long long*>(a.counters), (unsigned long long)tot);
    }
  }
  __syncthreads();
  if (tid == 0) {
    TL(3);
    __threadfence();
    const uint32_t prev = atomicAdd(&a.hdr->done, 1u);
    if (prev == gridDim.x - 1) {  // every CTA has drawn its last ticket
      a.hdr->ticket = 0u;
      a.hdr->done = 0u;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------
// host launchers (called from vt_round.cu's C ABI)
// ---------------------------------------------------------------------------

int64_t stream_tiles(int64_t n) { return (n + kSTile - 1) / kSTile; }

// fused: [header 64 B][status: one word per ticket (at most one per tile)]
static size_t rl_fused_workspace(int64_t n) { return (size_t)(64 + stream_tiles(n) * 8 + 256); }

size_t rl_stream_workspace(int64_t n) { return rl_fused_workspace(n); }

size_t rp_stream_workspace(int64_t n) {
  (void)n;
  return 64;  // ticket header
}

template <int OUT, bool FAST, bool KEYS = false>
static int launch_rlf(RLFArgs a, cudaStream_t st) {
  const size_t smem = sizeof(FusedSmem);
  static_assert(sizeof(FusedSmem) <= 74 * 1024, "three fused CTAs per SM");
  auto k = rl_fused_kernel<OUT, FAST, KEYS>;
  static int resident = 0;
  if (!resident) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kFThreads, smem);
    if (const char* e = getenv("VT_RL_CTAS_PER_SM")) per = std::max(1, std::min(per, atoi(e)));  // A/B only
    resident = std::max(1, per * sms);
  }
  a.n4 = a.num_tiles / kSuper;
  a.num_super = a.n4 + a.num_tiles % kSuper;
  const int grid = (int)std::min<int64_t>(a.num_super, resident);
  k<<<grid, kFThreads, smem, st>>>(a);
  return vt_check_launch("rl_fused_kernel");
}

int rl_stream(const double* x, int64_t n, const Grid& g, int thr32, bool fast, int out_kind, void* out,
              uint64_t* sparse, int64_t cap, int64_t global_base, const int64_t* cursor_in, int64_t* cursor_out,
              int64_t* counters, int32_t* err, void* ws, cudaStream_t st, const DevThr* dthr,
              const int32_t* gate, uint64_t* keys, XPeers xp) {
  uint8_t* w = static_cast<uint8_t*>(ws);
  RLFArgs f{x, n, g, thr32, out, stream_tiles(n), 0, 0, reinterpret_cast<FusedHeader*>(w),
            reinterpret_cast<uint64_t*>(w + 64), sparse, cap, global_base, cursor_in, cursor_out, counters, err,
            dthr, gate, keys, xp};
  if (keys) {  // the adaptive candidate pass (b_r = 32 or not)
    if (fast)
      return out_kind == VT_OUT_F32 ? launch_rlf<VT_OUT_F32, true, true>(f, st)
           : out_kind == VT_OUT_F64 ? launch_rlf<VT_OUT_F64, true, true>(f, st)
                                    : launch_rlf<VT_OUT_NONE, true, true>(f, st);
    return out_kind == VT_OUT_F32 ? launch_rlf<VT_OUT_F32, false, true>(f, st)
         : out_kind == VT_OUT_F64 ? launch_rlf<VT_OUT_F64, false, true>(f, st)
                                  : launch_rlf<VT_OUT_NONE, false, true>(f, st);
  }
  if (fast) {
    return out_kind == VT_OUT_F32 ? launch_rlf<VT_OUT_F32, true>(f, st)
         : out_kind == VT_OUT_F64 ? launch_rlf<VT_OUT_F64, true>(f, st)
                                  : launch_rlf<VT_OUT_NONE, true>(f, st);
  }
  return out_kind == VT_OUT_F32 ? launch_rlf<VT_OUT_F32, false>(f, st)
       : out_kind == VT_OUT_F64 ? launch_rlf<VT_OUT_F64, false>(f, st)
                                : launch_rlf<VT_OUT_NONE, false>(f, st);
}

template <int OUT, bool FAST, bool KEYS>
static int launch_rlb(const RLBatch& b, cudaStream_t st) {
  static_assert(sizeof(RLBatch) <= 32000, "batch table must fit the kernel parameter space");
  const size_t smem = sizeof(FusedSmem);
  auto k = rl_batch_kernel<OUT, FAST, KEYS>;
  static int resident = 0;
  if (!resident) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kFThreads, smem);
    resident = std::max(1, per * sms);
  }
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(b.total, resident));
  k<<<grid, kFThreads, smem, st>>>(b);
  return vt_check_launch("rl_batch_kernel");
}

template <bool KEYS>
static int rl_stream_batch_t(const RLBatch& b, bool fast, int out_kind, cudaStream_t st) {
  if (fast) {
    return out_kind == VT_OUT_F32 ? launch_rlb<VT_OUT_F32, true, KEYS>(b, st)
         : out_kind == VT_OUT_F64 ? launch_rlb<VT_OUT_F64, true, KEYS>(b, st)
                                  : launch_rlb<VT_OUT_NONE, true, KEYS>(b, st);
  }
  return out_kind == VT_OUT_F32 ? launch_rlb<VT_OUT_F32, false, KEYS>(b, st)
       : out_kind == VT_OUT_F64 ? launch_rlb<VT_OUT_F64, false, KEYS>(b, st)
                                : launch_rlb<VT_OUT_NONE, false, KEYS>(b, st);
}

int rl_stream_batch(const RLBatch& b, bool fast, int out_kind, cudaStream_t st, bool keys) {
  return keys ? rl_stream_batch_t<true>(b, fast, out_kind, st) : rl_stream_batch_t<false>(b, fast, out_kind, st);
}

template <int OUT, bool FAST, bool PACKED = false>
static int launch_rp(RPArgs a, cudaStream_t st) {
  const size_t smem = sizeof(ReplaySmem);
  static_assert(sizeof(ReplaySmem) <= 74 * 1024, "three replay CTAs per SM");
  auto k = rp_fused_kernel<OUT, FAST, PACKED>;
  static int resident = 0;
  if (!resident) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kRThreads, smem);
    resident = std::max(1, per * sms);
  }
  a.n4 = a.num_tiles / kRSuper;
  a.num_super = a.n4 + a.num_tiles % kRSuper;
  const int grid = (int)std::min<int64_t>(a.num_super, resident);
  k<<<grid, kRThreads, smem, st>>>(a);
  return vt_check_launch("rp_fused_kernel");
}

int rp_stream_packed(const double* x, int64_t n, const Grid& g, bool fast, int out_kind, void* out,
                     const uint8_t* payload, int64_t nbytes, int64_t pos, int64_t* counters, int32_t* err, void* ws,
                     cudaStream_t st) {
  RPArgs a{x, n, g, reinterpret_cast<const uint64_t*>(payload), nbytes, pos, out, stream_tiles(n), 0, 0,
           static_cast<FusedHeader*>(ws), counters, err};
  if (fast) {
    return out_kind == VT_OUT_F32 ? launch_rp<VT_OUT_F32, true, true>(a, st)
         : out_kind == VT_OUT_F64 ? launch_rp<VT_OUT_F64, true, true>(a, st)
                                  : launch_rp<VT_OUT_NONE, true, true>(a, st);
  }
  return out_kind == VT_OUT_F32 ? launch_rp<VT_OUT_F32, false, true>(a, st)
       : out_kind == VT_OUT_F64 ? launch_rp<VT_OUT_F64, false, true>(a, st)
                                : launch_rp<VT_OUT_NONE, false, true>(a, st);
}

int rp_stream(const double* x, int64_t n, const Grid& g, bool fast, int out_kind, void* out, const uint64_t* log,
              int64_t n_words, int64_t log_base, int64_t* counters, int32_t* err, void* ws, cudaStream_t st) {
  RPArgs a{x, n, g, log, n_words, log_base, out, stream_tiles(n), 0, 0, static_cast<FusedHeader*>(ws), counters,
           err};
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
