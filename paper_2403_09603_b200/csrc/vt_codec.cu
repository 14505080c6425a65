// .vtrl payload codec on the device: 5 ternary codes per byte, little-endian
// base 3 (reference roundlog.py:1-17, _pack_block :67-70, _unpack_block :73-82).
// The 15-byte header and optional DEFLATE stay on the host
// (paper_2403_09603_b200/roundlog.py).
#include <algorithm>

#include "vt_common.cuh"

namespace vt {

__global__ void pack5_kernel(const uint8_t* __restrict__ codes, int64_t n_groups,
                             uint8_t* __restrict__ out, int32_t* errp) {
  uint32_t err = 0;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_groups;
       g += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t* c = codes + 5 * g;
    uint32_t b = 0, w = 1;
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const uint32_t d = c[k];
      err |= (d > 2u) ? (uint32_t)VT_ERR_BAD_CODE : 0u;
      b += d * w;
      w *= 3u;
    }
    out[g] = (uint8_t)b;
  }
  report_err(errp, err);
}

// codes[i] = digit (pos + i) of the payload stream
__global__ void unpack5_kernel(const uint8_t* __restrict__ payload, int64_t pos, int64_t n,
                               uint8_t* __restrict__ codes, int32_t* errp) {
  uint32_t err = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = pos + i;
    const int64_t bi = p / 5;
    const int d = (int)(p - 5 * bi);
    const uint32_t b = __ldg(payload + bi);
    err |= (b > 242u) ? (uint32_t)VT_ERR_BAD_LOG_BYTE : 0u;
    const uint32_t p3 = d == 0 ? 1u : d == 1 ? 3u : d == 2 ? 9u : d == 3 ? 27u : 81u;
    codes[i] = (uint8_t)((b / p3) % 3u);
  }
  report_err(errp, err);
}

__global__ void validate_kernel(const uint8_t* __restrict__ payload, int64_t nbytes, int32_t* errp) {
  uint32_t bad = 0;
  const int64_t n16 = nbytes / 16;
  const uint4* p4 = reinterpret_cast<const uint4*>(payload);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) {
    const uint4 v = __ldg(p4 + i);
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // any byte > 242 (0xF2): per-byte unsigned max via __vmaxu4 against 242
      bad |= (__vcmpgtu4(w[k], 0xF2F2F2F2u) != 0u) ? 1u : 0u;
    }
  }
  for (int64_t i = n16 * 16 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nbytes; i += stride)
    bad |= (payload[i] > 242) ? 1u : 0u;
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(reinterpret_cast<int*>(errp), VT_ERR_BAD_LOG_BYTE);
}

__global__ void histogram_kernel(const uint8_t* __restrict__ payload, int64_t n_entries,
                                 unsigned long long* counts, int32_t* errp) {
  uint32_t c[3] = {0, 0, 0};
  uint32_t err = 0;
  const int64_t full = n_entries / 5;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b <= full;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int lim = (b < full) ? 5 : (int)(n_entries - 5 * full);
    if (lim == 0) continue;
    uint32_t v = payload[b];
    err |= (v > 242u) ? (uint32_t)VT_ERR_BAD_LOG_BYTE : 0u;
    for (int k = 0; k < lim; ++k) {
      const uint32_t d = v % 3u;
      v /= 3u;
      c[0] += d == 0u;
      c[1] += d == 1u;
      c[2] += d == 2u;
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    uint32_t v = c[k];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(counts + k, (unsigned long long)v);
  }
  report_err(errp, err);
}

unsigned cblocks(int64_t work) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, 148 * 16));
}

}  // namespace vt

using namespace vt;

extern "C" int vt_pack5(const uint8_t* codes, int64_t n_groups, uint8_t* out, int32_t* err,
                        vt_stream_t stream) {
  if (n_groups < 0 || !err || (n_groups && (!codes || !out))) {
    vt_set_error("vt_pack5: bad argument");
    return VT_EINVAL;
  }
  if (!n_groups) return VT_OK;
  pack5_kernel<<<cblocks(n_groups), 256, 0, static_cast<cudaStream_t>(stream)>>>(codes, n_groups, out, err);
  return vt_check_launch("pack5_kernel");
}

extern "C" int vt_unpack5(const uint8_t* payload, int64_t pos, int64_t n, uint8_t* codes,
                          int32_t* err, vt_stream_t stream) {
  if (n < 0 || pos < 0 || !err || (n && (!payload || !codes))) {
    vt_set_error("vt_unpack5: bad argument");
    return VT_EINVAL;
  }
  if (!n) return VT_OK;
  unpack5_kernel<<<cblocks(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(payload, pos, n, codes, err);
  return vt_check_launch("unpack5_kernel");
}

extern "C" int vt_log_validate(const uint8_t* payload, int64_t nbytes, int32_t* err, vt_stream_t stream) {
  if (nbytes < 0 || !err || (nbytes && !payload) || (reinterpret_cast<uintptr_t>(payload) & 15)) {
    vt_set_error("vt_log_validate: bad argument (payload must be 16-byte aligned)");
    return VT_EINVAL;
  }
  if (!nbytes) return VT_OK;
  validate_kernel<<<cblocks(std::max<int64_t>(nbytes / 16, 1)), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      payload, nbytes, err);
  return vt_check_launch("validate_kernel");
}

extern "C" int vt_log_histogram(const uint8_t* payload, int64_t n_entries, int64_t* counts3,
                                int32_t* err, vt_stream_t stream) {
  if (n_entries < 0 || !err || !counts3 || (n_entries && !payload)) {
    vt_set_error("vt_log_histogram: bad argument");
    return VT_EINVAL;
  }
  if (!n_entries) return VT_OK;
  histogram_kernel<<<cblocks(n_entries / 5 + 1), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      payload, n_entries, reinterpret_cast<unsigned long long*>(counts3), err);
  return vt_check_launch("histogram_kernel");
}
