// SHA-256 Merkle hashing of checkpoint bytes (FIPS 180-4 compression).
//
// Leaves: SHA-256 of each `leaf_bytes` chunk of the FP32 little-endian
// weight serialization (north-star chunked leaf, SURVEY.md Appendix A.5;
// the per-leaf hash is merkle._sha256, pkg/src/vtrain/merkle.py:24-25).
// Internal nodes: SHA-256(left || right), an unpaired last node promoted
// unchanged, every level kept (merkle.build, merkle.py:55-72).
//
// One message per thread with a register-resident 16-word rolling schedule;
// rotations are funnel shifts (SHF), Ch/Maj/Sigma fold into LOP3, byte swaps
// are PRMT.  A message whose length is a multiple of 64 ends in a padding
// block of constant content, so its schedule W[t] + K[t] is precomputed on
// the host once per length and passed in the kernel parameters.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "vt_common.cuh"

namespace vt {

__constant__ uint32_t kK[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
    0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
    0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
    0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
    0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
    0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
    0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
    0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};

static const uint32_t kKHost[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
    0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
    0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
    0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
    0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
    0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
    0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
    0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};

__constant__ uint32_t kIV[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                             0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};

struct PadWK {
  uint32_t wk[64];  // W[t] + K[t] of a constant padding block
};

__device__ __forceinline__ uint32_t rotr(uint32_t x, int n) { return __funnelshift_r(x, x, n); }
__device__ __forceinline__ uint32_t bswap(uint32_t x) { return __byte_perm(x, 0, 0x0123); }

// Adds: on the ALU pipe (IADD3) or, with FMA_ADDS, as IMADs by a runtime 1 on
// the FMA pipe.  The rotates and Ch/Maj/Sigma (SHF, LOP3) can only use the
// ALU pipe, which a plain compress() saturates (ncu: ALU 97% active, FMA 5%);
// moving the adds off it balances the two pipes.
template <bool FMA_ADDS>
__device__ __forceinline__ uint32_t vadd(uint32_t x, uint32_t y, uint32_t one) {
  if (FMA_ADDS) return x * one + y;
  return x + y;
}

#define VT_ROUND(a, b, c, d, e, f, g, h, wk)                                                              \
  {                                                                                                      \
    const uint32_t t1 = vadd<FMA>(h, vadd<FMA>(rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25),                  \
                                               vadd<FMA>((e & f) ^ (~e & g), (wk), one), one), one);    \
    const uint32_t t2 = vadd<FMA>(rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22), (a & b) ^ (a & c) ^ (b & c), one); \
    d = vadd<FMA>(d, t1, one);                                                                           \
    h = vadd<FMA>(t1, t2, one);                                                                          \
  }

// One compression of a data block held in w[16] (consumed).
template <bool FMA>
__device__ __forceinline__ void compress(uint32_t (&s)[8], uint32_t (&w)[16], uint32_t one) {
  uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#pragma unroll
  for (int t = 0; t < 64; t += 8) {
    if (t >= 16) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int j = (t + k) & 15;
        const uint32_t w15 = w[(j + 1) & 15], w2 = w[(j + 14) & 15];
        w[j] = vadd<FMA>(w[j], vadd<FMA>(rotr(w2, 17) ^ rotr(w2, 19) ^ (w2 >> 10),
                                         vadd<FMA>(w[(j + 9) & 15], rotr(w15, 7) ^ rotr(w15, 18) ^ (w15 >> 3), one),
                                         one), one);
      }
    }
    VT_ROUND(a, b, c, d, e, f, g, h, vadd<FMA>(kK[t + 0], w[(t + 0) & 15], one));
    VT_ROUND(h, a, b, c, d, e, f, g, vadd<FMA>(kK[t + 1], w[(t + 1) & 15], one));
    VT_ROUND(g, h, a, b, c, d, e, f, vadd<FMA>(kK[t + 2], w[(t + 2) & 15], one));
    VT_ROUND(f, g, h, a, b, c, d, e, vadd<FMA>(kK[t + 3], w[(t + 3) & 15], one));
    VT_ROUND(e, f, g, h, a, b, c, d, vadd<FMA>(kK[t + 4], w[(t + 4) & 15], one));
    VT_ROUND(d, e, f, g, h, a, b, c, vadd<FMA>(kK[t + 5], w[(t + 5) & 15], one));
    VT_ROUND(c, d, e, f, g, h, a, b, vadd<FMA>(kK[t + 6], w[(t + 6) & 15], one));
    VT_ROUND(b, c, d, e, f, g, h, a, vadd<FMA>(kK[t + 7], w[(t + 7) & 15], one));
  }
  s[0] += a; s[1] += b; s[2] += c; s[3] += d; s[4] += e; s[5] += f; s[6] += g; s[7] += h;
}

// Compression of a constant block whose W+K schedule is precomputed.
template <bool FMA>
__device__ __forceinline__ void compress_wk(uint32_t (&s)[8], const PadWK& p, uint32_t one) {
  uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
#pragma unroll
  for (int t = 0; t < 64; t += 8) {
    VT_ROUND(a, b, c, d, e, f, g, h, p.wk[t + 0]);
    VT_ROUND(h, a, b, c, d, e, f, g, p.wk[t + 1]);
    VT_ROUND(g, h, a, b, c, d, e, f, p.wk[t + 2]);
    VT_ROUND(f, g, h, a, b, c, d, e, p.wk[t + 3]);
    VT_ROUND(e, f, g, h, a, b, c, d, p.wk[t + 4]);
    VT_ROUND(d, e, f, g, h, a, b, c, p.wk[t + 5]);
    VT_ROUND(c, d, e, f, g, h, a, b, p.wk[t + 6]);
    VT_ROUND(b, c, d, e, f, g, h, a, p.wk[t + 7]);
  }
  s[0] += a; s[1] += b; s[2] += c; s[3] += d; s[4] += e; s[5] += f; s[6] += g; s[7] += h;
}

__device__ __forceinline__ void store_digest(uint8_t* dst, const uint32_t (&s)[8]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
  d[0] = make_uint4(bswap(s[0]), bswap(s[1]), bswap(s[2]), bswap(s[3]));
  d[1] = make_uint4(bswap(s[4]), bswap(s[5]), bswap(s[6]), bswap(s[7]));
}

struct LeafArgs {
  const uint8_t* data;
  int64_t nbytes;
  int64_t leaf_bytes;
  int64_t n_leaves;
  uint8_t* out;
  PadWK pad;  // padding block for a full leaf when leaf_bytes % 64 == 0
  uint32_t one;  // 1 (a runtime value: the FMA-pipe adds multiply by it)
};

// Generic tail: `rem` (< 64) trailing bytes at p, total message length len.
template <bool FMA>
__device__ __forceinline__ void finish_generic(uint32_t (&s)[8], const uint8_t* p, int rem, int64_t len,
                                               uint32_t one) {
  uint32_t w[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) w[k] = 0u;
  for (int k = 0; k < rem; ++k) w[k >> 2] |= (uint32_t)p[k] << (24 - 8 * (k & 3));
  w[rem >> 2] |= 0x80u << (24 - 8 * (rem & 3));
  const uint64_t bitlen = (uint64_t)len * 8ull;
  if (rem >= 56) {
    compress<FMA>(s, w, one);
#pragma unroll
    for (int k = 0; k < 16; ++k) w[k] = 0u;
  }
  w[14] = (uint32_t)(bitlen >> 32);
  w[15] = (uint32_t)bitlen;
  compress<FMA>(s, w, one);
}

template <bool FMA>
__global__ void __launch_bounds__(128) sha256_leaves_kernel(const LeafArgs a) {
  const uint32_t one = a.one;
  const int64_t leaf = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (leaf >= a.n_leaves) return;
  const int64_t off = leaf * a.leaf_bytes;
  const int64_t len = std::min<int64_t>(a.leaf_bytes, a.nbytes - off);
  const uint8_t* p = a.data + off;
  uint32_t s[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) s[k] = kIV[k];
  const int64_t nblk = len >> 6;
  const bool vec = ((reinterpret_cast<uintptr_t>(p) & 15) == 0);
  const uint4* p4 = reinterpret_cast<const uint4*>(p);
  for (int64_t blk = 0; blk < nblk; ++blk) {
    uint32_t w[16];
    if (vec) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 v = __ldg(p4 + blk * 4 + q);
        w[4 * q + 0] = bswap(v.x);
        w[4 * q + 1] = bswap(v.y);
        w[4 * q + 2] = bswap(v.z);
        w[4 * q + 3] = bswap(v.w);
      }
    } else {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const uint8_t* b = p + blk * 64 + 4 * k;
        w[k] = ((uint32_t)b[0] << 24) | ((uint32_t)b[1] << 16) | ((uint32_t)b[2] << 8) | b[3];
      }
    }
    compress<FMA>(s, w, one);
  }
  const int rem = (int)(len - (nblk << 6));
  if (rem == 0 && len == a.leaf_bytes && (a.leaf_bytes & 63) == 0) {
    compress_wk<FMA>(s, a.pad, one);
  } else {
    finish_generic<FMA>(s, p + (nblk << 6), rem, len, one);
  }
  store_digest(a.out + leaf * 32, s);
}

struct NodeArgs {
  const uint8_t* in;
  int64_t n_in;
  uint8_t* out;
  PadWK pad;  // padding block of a 64-byte message
  uint32_t one;
};

template <bool FMA>
__global__ void __launch_bounds__(128) merkle_level_kernel(const NodeArgs a) {
  const uint32_t one = a.one;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n_out = (a.n_in + 1) >> 1;
  if (i >= n_out) return;
  const uint4* src = reinterpret_cast<const uint4*>(a.in + 64 * i);
  uint4* dst = reinterpret_cast<uint4*>(a.out + 32 * i);
  if (2 * i + 1 >= a.n_in) {  // unpaired: promoted unchanged (merkle.py:66-67)
    dst[0] = src[0];
    dst[1] = src[1];
    return;
  }
  uint32_t w[16];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 v = src[q];
    w[4 * q + 0] = bswap(v.x);
    w[4 * q + 1] = bswap(v.y);
    w[4 * q + 2] = bswap(v.z);
    w[4 * q + 3] = bswap(v.w);
  }
  uint32_t s[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) s[k] = kIV[k];
  compress<FMA>(s, w, one);
  compress_wk<FMA>(s, a.pad, one);
  store_digest(a.out + 32 * i, s);
  (void)dst;
}

// Host: W+K schedule of the padding block that follows a message of `len`
// bytes when len % 64 == 0.
PadWK make_pad(int64_t len) {
  uint32_t w[64];
  for (int k = 0; k < 16; ++k) w[k] = 0u;
  w[0] = 0x80000000u;
  const uint64_t bits = (uint64_t)len * 8ull;
  w[14] = (uint32_t)(bits >> 32);
  w[15] = (uint32_t)bits;
  auto r = [](uint32_t x, int n) { return (x >> n) | (x << (32 - n)); };
  for (int t = 16; t < 64; ++t) {
    const uint32_t s0 = r(w[t - 15], 7) ^ r(w[t - 15], 18) ^ (w[t - 15] >> 3);
    const uint32_t s1 = r(w[t - 2], 17) ^ r(w[t - 2], 19) ^ (w[t - 2] >> 10);
    w[t] = w[t - 16] + s0 + w[t - 7] + s1;
  }
  PadWK p;
  for (int t = 0; t < 64; ++t) p.wk[t] = w[t] + kKHost[t];
  return p;
}

// Which add placement the Merkle kernels use: FMA-pipe adds unless
// VT_SHA_ALU_ADDS=1 (A/B switch for measurement).
bool sha_fma_adds() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("VT_SHA_ALU_ADDS");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

}  // namespace vt

using namespace vt;

extern "C" int vt_sha256_leaves(const uint8_t* data, int64_t nbytes, int64_t leaf_bytes, uint8_t* digests,
                                vt_stream_t stream) {
  if (nbytes <= 0 || leaf_bytes <= 0 || !data || !digests || (reinterpret_cast<uintptr_t>(digests) & 15)) {
    vt_set_error("vt_sha256_leaves: bad argument (nbytes, leaf_bytes > 0; digests 16-byte aligned)");
    return VT_EINVAL;
  }
  LeafArgs a;
  a.data = data;
  a.nbytes = nbytes;
  a.leaf_bytes = leaf_bytes;
  a.n_leaves = (nbytes + leaf_bytes - 1) / leaf_bytes;
  a.out = digests;
  a.pad = make_pad(leaf_bytes);
  a.one = 1u;
  const unsigned grid = (unsigned)((a.n_leaves + 127) / 128);
  if (sha_fma_adds())
    sha256_leaves_kernel<true><<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(a);
  else
    sha256_leaves_kernel<false><<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return vt_check_launch("sha256_leaves_kernel");
}

extern "C" int vt_merkle_level(const uint8_t* in, int64_t n_in, uint8_t* out, vt_stream_t stream) {
  if (n_in <= 0 || !in || !out || (reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(out) & 15)) {
    vt_set_error("vt_merkle_level: bad argument (16-byte aligned digests)");
    return VT_EINVAL;
  }
  NodeArgs a;
  a.in = in;
  a.n_in = n_in;
  a.out = out;
  a.pad = make_pad(64);
  a.one = 1u;
  const int64_t n_out = (n_in + 1) / 2;
  const unsigned grid = (unsigned)((n_out + 127) / 128);
  if (sha_fma_adds())
    merkle_level_kernel<true><<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(a);
  else
    merkle_level_kernel<false><<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(a);
  return vt_check_launch("merkle_level_kernel");
}

// ---------------------------------------------------------------------------
// Block-root exchange of the sharded Merkle tree over peer
// memory: the level kernel that produces a rank's block roots also stores
// every root into EVERY rank's exchange buffer (symmetric memory mapped over
// NVLink) at its global block index, and its last CTA publishes the rank's
// arrival with st.release.sys; a one-CTA wait kernel then gathers all roots.
// Replaces the ncclAllGather of the block roots.
//
// Buffer (uint64 words): [0] this rank's exchange sequence number, [1] CTA
// done counter (local), [2 + par * world + r] rank r's arrival tag for
// parity par, then the digests [par][n_total][4 words].  Digest areas and
// tags alternate by the parity of the sequence number: a rank can only run
// one exchange ahead of a peer after that peer has published, i.e. after its
// wait kernel (and every reader of its roots, stream-ordered before its next
// publish) is done -- the argument of the count exchange (vt_stream.cu).
// ---------------------------------------------------------------------------
struct DXPeers {
  uint64_t* const* peers;
  int world, rank;
  int64_t dst;      // this rank's first block index
  int64_t n_total;  // block roots over all ranks
};

__device__ __forceinline__ uint64_t* dx_digest(const DXPeers& xp, int p, int par, int64_t j) {
  return xp.peers[p] + 2 + 2 * xp.world + ((int64_t)par * xp.n_total + j) * 4;
}

__device__ __forceinline__ void dx_store(const DXPeers& xp, int par, int64_t j, const uint32_t* h) {
  // the digest's 32 bytes, big-endian words as in store_digest
  uint4 d0, d1;
  d0.x = bswap(h[0]); d0.y = bswap(h[1]); d0.z = bswap(h[2]); d0.w = bswap(h[3]);
  d1.x = bswap(h[4]); d1.y = bswap(h[5]); d1.z = bswap(h[6]); d1.w = bswap(h[7]);
  for (int p = 0; p < xp.world; ++p) {
    uint4* q = reinterpret_cast<uint4*>(dx_digest(xp, p, par, xp.dst + j));
    q[0] = d0;
    q[1] = d1;
  }
}

// every thread of the grid calls this once, after its stores
__device__ __forceinline__ void dx_finish(const DXPeers& xp, int par) {
  __shared__ unsigned s_last;
  __threadfence_system();
  __syncthreads();
  uint64_t* mine = xp.peers[xp.rank];
  if (threadIdx.x == 0)
    s_last = atomicAdd(reinterpret_cast<unsigned long long*>(mine + 1), 1ull) == (unsigned long long)gridDim.x - 1;
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  __threadfence_system();
  const uint64_t seq = mine[0] + 1ull;
  mine[0] = seq;
  mine[1] = 0ull;
  for (int p = 0; p < xp.world; ++p) st_release_sys_u64(xp.peers[p] + 2 + par * xp.world + xp.rank, seq);
}

template <bool FMA>
__global__ void __launch_bounds__(128) merkle_level_xchg_kernel(const NodeArgs a, const DXPeers xp) {
  const int par = (int)((xp.peers[xp.rank][0] + 1ull) & 1ull);  // this exchange's parity
  const uint32_t one = a.one;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n_out = (a.n_in + 1) >> 1;
  if (i < n_out) {
    uint32_t s[8];
    if (2 * i + 1 >= a.n_in) {  // unpaired: promoted unchanged (merkle.py:66-67)
      const uint4* src = reinterpret_cast<const uint4*>(a.in + 64 * i);
      uint4* dst = reinterpret_cast<uint4*>(a.out + 32 * i);
      const uint4 v0 = src[0], v1 = src[1];
      dst[0] = v0;
      dst[1] = v1;
      s[0] = bswap(v0.x); s[1] = bswap(v0.y); s[2] = bswap(v0.z); s[3] = bswap(v0.w);
      s[4] = bswap(v1.x); s[5] = bswap(v1.y); s[6] = bswap(v1.z); s[7] = bswap(v1.w);
    } else {
      const uint4* src = reinterpret_cast<const uint4*>(a.in + 64 * i);
      uint32_t w[16];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 v = src[q];
        w[4 * q + 0] = bswap(v.x);
        w[4 * q + 1] = bswap(v.y);
        w[4 * q + 2] = bswap(v.z);
        w[4 * q + 3] = bswap(v.w);
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) s[k] = kIV[k];
      compress<FMA>(s, w, one);
      compress_wk<FMA>(s, a.pad, one);
      store_digest(a.out + 32 * i, s);
    }
    dx_store(xp, par, i, s);
  }
  dx_finish(xp, par);
}

// roots that need no hashing at this rank (one node, depth 0, or none)
__global__ void __launch_bounds__(128) digests_publish_kernel(const uint8_t* in, int64_t n, const DXPeers xp) {
  const int par = (int)((xp.peers[xp.rank][0] + 1ull) & 1ull);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4* src = reinterpret_cast<const uint4*>(in + 32 * i);
    const uint4 v0 = src[0], v1 = src[1];
    const uint32_t s[8] = {bswap(v0.x), bswap(v0.y), bswap(v0.z), bswap(v0.w),
                           bswap(v1.x), bswap(v1.y), bswap(v1.z), bswap(v1.w)};
    dx_store(xp, par, i, s);
  }
  dx_finish(xp, par);
}

__global__ void __launch_bounds__(256) digests_wait_kernel(const DXPeers xp, uint8_t* out, int32_t* err,
                                                           uint64_t timeout_ns) {
  __shared__ int s_ok;
  const uint64_t* mine = xp.peers[xp.rank];
  const uint64_t seq = *(volatile const uint64_t*)mine;
  const int par = (int)(seq & 1ull);
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  for (int q = threadIdx.x; q < xp.world; q += blockDim.x) {
    uint64_t t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (ld_acquire_sys_u64(mine + 2 + par * xp.world + q) != seq) {
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > timeout_ns) {
        atomicOr(err, VT_ERR_EXCHANGE);
        s_ok = 0;
        break;
      }
      __nanosleep(100);
    }
  }
  __syncthreads();
  if (!s_ok) return;
  const uint4* src = reinterpret_cast<const uint4*>(mine + 2 + 2 * xp.world + (int64_t)par * xp.n_total * 4);
  uint4* dst = reinterpret_cast<uint4*>(out);
  for (int64_t i = threadIdx.x; i < 2 * xp.n_total; i += blockDim.x) dst[i] = __ldcg(src + i);
}

extern "C" size_t vt_digest_exchange_words(int world, int64_t n_total) {
  return (world > 0 && n_total >= 0) ? (size_t)(2 + 2 * world + 8 * n_total) : 0;
}

static bool dx_ok(uint64_t* const* xpeers, int world, int rank, int64_t dst, int64_t n, int64_t n_total) {
  return xpeers && world > 0 && rank >= 0 && rank < world && dst >= 0 && n >= 0 && n_total >= 0 &&
         dst + n <= n_total;
}

extern "C" int vt_merkle_level_exchange(const uint8_t* in, int64_t n_in, uint8_t* out, uint64_t* const* xpeers,
                                        int world, int rank, int64_t dst, int64_t n_total, vt_stream_t stream) {
  const int64_t n_out = (n_in + 1) / 2;
  if (n_in <= 0 || !in || !out || (reinterpret_cast<uintptr_t>(in) & 15) || (reinterpret_cast<uintptr_t>(out) & 15) ||
      !dx_ok(xpeers, world, rank, dst, n_out, n_total)) {
    vt_set_error("vt_merkle_level_exchange: bad argument");
    return VT_EINVAL;
  }
  NodeArgs a;
  a.in = in;
  a.n_in = n_in;
  a.out = out;
  a.pad = make_pad(64);
  a.one = 1u;
  const DXPeers xp{xpeers, world, rank, dst, n_total};
  const unsigned grid = (unsigned)((n_out + 127) / 128);
  if (sha_fma_adds())
    merkle_level_xchg_kernel<true><<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(a, xp);
  else
    merkle_level_xchg_kernel<false><<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(a, xp);
  return vt_check_launch("merkle_level_xchg_kernel");
}

extern "C" int vt_digests_publish(const uint8_t* digests, int64_t n, uint64_t* const* xpeers, int world, int rank,
                                  int64_t dst, int64_t n_total, vt_stream_t stream) {
  if ((n > 0 && (!digests || (reinterpret_cast<uintptr_t>(digests) & 15))) ||
      !dx_ok(xpeers, world, rank, dst, n, n_total)) {
    vt_set_error("vt_digests_publish: bad argument");
    return VT_EINVAL;
  }
  const DXPeers xp{xpeers, world, rank, dst, n_total};
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 127) / 128, 148));
  digests_publish_kernel<<<grid, 128, 0, static_cast<cudaStream_t>(stream)>>>(digests, n, xp);
  return vt_check_launch("digests_publish_kernel");
}

extern "C" int vt_digests_wait(uint64_t* const* xpeers, int world, int rank, int64_t n_total, uint8_t* out,
                               int32_t* err, vt_stream_t stream) {
  if (!dx_ok(xpeers, world, rank, 0, 0, n_total) || !err || (n_total > 0 && (!out || (reinterpret_cast<uintptr_t>(out) & 15)))) {
    vt_set_error("vt_digests_wait: bad argument");
    return VT_EINVAL;
  }
  const DXPeers xp{xpeers, world, rank, 0, n_total};
  digests_wait_kernel<<<1, 256, 0, static_cast<cudaStream_t>(stream)>>>(xp, out, err, 10ull * 1000 * 1000 * 1000);
  return vt_check_launch("digests_wait_kernel");
}

extern "C" int64_t vt_merkle_node_count(int64_t n_leaves) {
  if (n_leaves <= 0) return 0;
  int64_t total = n_leaves, m = n_leaves;
  while (m > 1) {
    m = (m + 1) / 2;
    total += m;
  }
  return total;
}

extern "C" int vt_merkle_build(const uint8_t* data, int64_t nbytes, int64_t leaf_bytes, uint8_t* nodes,
                               int64_t nodes_cap, vt_stream_t stream) {
  if (nbytes <= 0 || leaf_bytes <= 0) {
    vt_set_error("vt_merkle_build: bad argument");
    return VT_EINVAL;
  }
  const int64_t leaves = (nbytes + leaf_bytes - 1) / leaf_bytes;
  if (nodes_cap < vt_merkle_node_count(leaves)) {
    vt_set_error("vt_merkle_build: nodes buffer too small");
    return VT_EINVAL;
  }
  int rc = vt_sha256_leaves(data, nbytes, leaf_bytes, nodes, stream);
  if (rc) return rc;
  int64_t m = leaves;
  uint8_t* cur = nodes;
  while (m > 1) {
    uint8_t* nxt = cur + 32 * m;
    if ((rc = vt_merkle_level(cur, m, nxt, stream))) return rc;
    cur = nxt;
    m = (m + 1) / 2;
  }
  return VT_OK;
}

// ---------------------------------------------------------------------------
// Compute-only ceiling of this SHA-256 compression on the running chip:
// the same compress() over register-resident messages, no memory traffic.
// The Merkle kernels' compressions/s divided by this rate is the
// "fraction of SHA-256 integer-pipe peak" reported by bench.py.
// ---------------------------------------------------------------------------

namespace vt {
template <bool FMA>
__global__ void __launch_bounds__(128) sha256_peak_kernel(uint32_t* sink, int reps, uint32_t one) {
  uint32_t s[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) s[k] = kIV[k] ^ (threadIdx.x * 0x9e3779b9u + blockIdx.x);
  uint32_t m[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) m[k] = (blockIdx.x * 131u) ^ (threadIdx.x << k);
  for (int r = 0; r < reps; ++r) {
    uint32_t w[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) w[k] = m[k] ^ s[k & 7];
    compress<FMA>(s, w, one);
  }
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) acc ^= s[k];
  if (acc == 0x9e3779b9u) sink[0] = acc;  // keeps the work alive
}
}  // namespace vt

extern "C" int vt_sha256_peak_bench(uint32_t* sink, int64_t blocks, int reps, vt_stream_t stream) {
  if (blocks <= 0 || reps <= 0 || !sink) {
    vt_set_error("vt_sha256_peak_bench: bad argument");
    return VT_EINVAL;
  }
  if (vt::sha_fma_adds())
    vt::sha256_peak_kernel<true><<<(unsigned)blocks, 128, 0, static_cast<cudaStream_t>(stream)>>>(sink, reps, 1u);
  else
    vt::sha256_peak_kernel<false><<<(unsigned)blocks, 128, 0, static_cast<cudaStream_t>(stream)>>>(sink, reps, 1u);
  return vt_check_launch("sha256_peak_kernel");
}

// ---------------------------------------------------------------------------
// Integer-pipe peak, independent of compress(): register-only chains of the
// SHA-256 op MIX (per unit: 6 SHF funnel-shift rotates, 4 LOP3, 4 IADD3 --
// SURVEY.md §8(d) OPS) with no message schedule, no constants table, no
// memory traffic and 8 independent chains per thread for ILP.  The bench
// divides the Merkle kernel's analytic op rate (1,400 ops per compression)
// by this rate.  Ops per launch = blocks * 256 * reps *
// kMixChains * 14 (the SASS is checked by tests/test_abi.py).
// ---------------------------------------------------------------------------
namespace vt {
constexpr int kMixChains = 8;
// FMA_ADDS: every 3-input add as two IMADs by a runtime 1 on the FMA pipe
// (how ptxas balances adds off the ALU pipe in compress()); otherwise IADD3
// on the ALU pipe.  The bench takes the faster of the two as the peak of
// the mix.
template <bool FMA_ADDS>
__device__ __forceinline__ uint32_t add3(uint32_t x, uint32_t y, uint32_t z, uint32_t one) {
  if (FMA_ADDS) return x * one + (y * one + z);
  return x + y + z;
}

template <bool FMA_ADDS>
__global__ void __launch_bounds__(256) int_mix_peak_kernel(uint32_t* sink, int reps, uint32_t seed, uint32_t one) {
  uint32_t a[kMixChains], b[kMixChains], c[kMixChains], d[kMixChains];
#pragma unroll
  for (int k = 0; k < kMixChains; ++k) {
    a[k] = seed ^ (threadIdx.x * 0x9e3779b9u) ^ (k * 0x85ebca6bu);
    b[k] = a[k] * 3u + blockIdx.x;
    c[k] = b[k] ^ 0xc2b2ae35u;
    d[k] = c[k] + 0x27d4eb2fu;
  }
  // each update overwrites one state word; per chain and iteration the SHA-256
  // round's op mix: 6 SHF + 4 LOP3 + 4 three-input adds
#pragma unroll 1
  for (int r = 0; r < reps; ++r) {
#pragma unroll
    for (int k = 0; k < kMixChains; ++k) {
      a[k] = add3<FMA_ADDS>(a[k],
                            __funnelshift_r(b[k], b[k], 6) ^ __funnelshift_r(b[k], b[k], 11) ^
                                __funnelshift_r(b[k], b[k], 25),
                            (b[k] & c[k]) ^ (~b[k] & d[k]), one);
      b[k] = add3<FMA_ADDS>(b[k],
                            __funnelshift_r(c[k], c[k], 2) ^ __funnelshift_r(c[k], c[k], 13) ^
                                __funnelshift_r(c[k], c[k], 22),
                            (c[k] & d[k]) ^ (c[k] & a[k]) ^ (d[k] & a[k]), one);
      c[k] = add3<FMA_ADDS>(c[k], d[k], a[k], one);
      d[k] = add3<FMA_ADDS>(d[k], b[k], (uint32_t)r, one);
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int k = 0; k < kMixChains; ++k) acc ^= a[k] ^ b[k] ^ c[k] ^ d[k];
  if (acc == 0x9e3779b9u) sink[0] = acc;  // keeps the work alive
}
}  // namespace vt

extern "C" int vt_int_mix_peak_bench(uint32_t* sink, int64_t blocks, int reps, int fma_adds, vt_stream_t stream) {
  if (blocks <= 0 || reps <= 0 || !sink) {
    vt_set_error("vt_int_mix_peak_bench: bad argument");
    return VT_EINVAL;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (fma_adds)
    vt::int_mix_peak_kernel<true><<<(unsigned)blocks, 256, 0, s>>>(sink, reps, 0x1234567u, 1u);
  else
    vt::int_mix_peak_kernel<false><<<(unsigned)blocks, 256, 0, s>>>(sink, reps, 0x1234567u, 1u);
  return vt_check_launch("int_mix_peak_kernel");
}

extern "C" int64_t vt_int_mix_ops_per_thread_rep(void) { return (int64_t)vt::kMixChains * 14; }

// ---------------------------------------------------------------------------
// Canonical checkpoint serialization (merkle.hash_weights, merkle.py:155-166):
// FP64 -> FP32 round-to-nearest-even, little-endian (the device's own byte
// order), overflow to +-inf exactly like numpy's astype('<f4'); the first
// non-finite FP64 element is reported (the reference checks finiteness on
// the FP64 values before casting).  Streaming: 256-bit loads, 128-bit stores.
// ---------------------------------------------------------------------------
namespace vt {
__global__ void __launch_bounds__(256) serialize_f32_kernel(const double* __restrict__ x, int64_t n,
                                                            float* __restrict__ out, int64_t index_base,
                                                            unsigned long long* first_bad) {
  unsigned long long bad = ~0ull;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
    if (i + 3 < n) {
      const D4 v = ldg_stream4(x + i);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (!isfinite(v.v[k]) && bad == ~0ull) bad = (unsigned long long)(i + k);
      *reinterpret_cast<float4*>(out + i) = make_float4(__double2float_rn(v.v[0]), __double2float_rn(v.v[1]),
                                                        __double2float_rn(v.v[2]), __double2float_rn(v.v[3]));
    } else {
      for (int64_t k = i; k < n; ++k) {
        const double e = x[k];
        if (!isfinite(e) && bad == ~0ull) bad = (unsigned long long)k;
        out[k] = __double2float_rn(e);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, bad, o);
    bad = b < bad ? b : bad;
  }
  if ((threadIdx.x & 31) == 0 && bad != ~0ull) atomicMin(first_bad, bad + (unsigned long long)index_base);
}
}  // namespace vt

extern "C" int vt_serialize_f32(const double* x, int64_t n, float* out, int64_t index_base, int64_t* first_bad,
                                vt_stream_t stream) {
  if (n < 0 || index_base < 0 || !first_bad || (n > 0 && (!x || !out)) || (reinterpret_cast<uintptr_t>(x) & 31) ||
      (reinterpret_cast<uintptr_t>(out) & 15)) {
    vt_set_error("vt_serialize_f32: bad argument (x 32-byte, out 16-byte aligned)");
    return VT_EINVAL;
  }
  if (n == 0) return VT_OK;
  const int64_t blocks = std::min<int64_t>((n + 1023) / 1024, 148 * 8);
  vt::serialize_f32_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      x, n, out, index_base, reinterpret_cast<unsigned long long*>(first_bad));
  return vt_check_launch("serialize_f32_kernel");
}
