/*
 * The drop-in boundary from plain C: no Python, no torch -- only the C ABI in
 * include/vtrain_b200.h and the CUDA runtime for device memory and a stream.
 * A trainer round-and-log (vt_round_log: protocol._TrainerChannel.process,
 * pkg/src/vtrain/protocol.py:198-202) and an auditor replay of a perturbed
 * copy (vt_replay: protocol._AuditorChannel.process, :212-216) of one FP64
 * tensor, then host checks: the FP32 outputs equal (float)x, the auditor
 * lands on the trainer's grid, the log is strictly ascending with global
 * indices, and its length matches the count the library reports.  Then the
 * checkpoint commitment of the trainer's FP32 output: vt_merkle_build (SHA-256
 * of 4 KiB chunks + merkle.build's levels, merkle.py:24-25,55-72) prints the
 * root; with a second argument the FP32 bytes are written to that file so a
 * caller can recompute the root independently (tests/test_abi_c.py, hashlib).
 *
 *   cc -O2 -I include -I /usr/local/cuda/include examples/abi_roundtrip.c \
 *      -L paper_2403_09603_b200 -lvtrain_b200 -L /usr/local/cuda/lib64 -lcudart \
 *      -Wl,-rpath,paper_2403_09603_b200 -o abi_roundtrip && ./abi_roundtrip [n [y.bin]]
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "vtrain_b200.h"

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess) {                                                       \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
      return 2;                                                                    \
    }                                                                              \
  } while (0)
#define VT(call)                                                                   \
  do {                                                                             \
    int r_ = (call);                                                               \
    if (r_ != VT_OK) {                                                             \
      fprintf(stderr, "%s:%d %s (%d)\n", __FILE__, __LINE__, vt_last_error(), r_); \
      return 3;                                                                    \
    }                                                                              \
  } while (0)

static uint64_t rng_state = 0x9e3779b97f4a7c15ull;
static uint64_t next_u64(void) {  /* splitmix64 */
  uint64_t z = (rng_state += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : (1 << 22) + 12345;
  const int64_t base = 1000;                       /* global index of element 0 */
  const double tau = ldexp(1.0 - 1e-3, -24);       /* configs[0] tau_ref */
  double* hx = (double*)malloc((size_t)n * 8);
  double* hxa = (double*)malloc((size_t)n * 8);
  float* hy = (float*)malloc((size_t)n * 4);
  float* hya = (float*)malloc((size_t)n * 4);
  for (int64_t i = 0; i < n; ++i) {
    /* ~10% exactly at an FP32 rounding midpoint (then perturbed), else random */
    const double u = (double)(next_u64() >> 11) * 0x1p-53 - 0.5;
    double v = u * 8.0;
    if (next_u64() % 10 == 0) {
      const float f = (float)v;
      const double up = (double)nextafterf(f, INFINITY), dn = (double)nextafterf(f, -INFINITY);
      const double lo = (double)f <= v ? (double)f : dn, hi = (double)f <= v ? up : (double)f;
      v = 0.5 * (lo + hi) * (1.0 + ((double)(next_u64() >> 11) * 0x1p-53 - 0.5) * 0x1p-39);
    }
    hx[i] = v;
    hxa[i] = (next_u64() % 20 == 0) ? nextafter(v, (next_u64() & 1) ? INFINITY : -INFINITY) : v;
  }
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  double *dx, *dxa;
  float *dy, *dya;
  uint64_t* dlog;
  int64_t* dflags;
  void *ws, *wsr;
  const int64_t cap = n / 4 + 1024;
  const size_t wsb = vt_round_log_workspace(n), wsrb = vt_replay_workspace(n);
  CK(cudaMalloc((void**)&dx, (size_t)n * 8));
  CK(cudaMalloc((void**)&dxa, (size_t)n * 8));
  CK(cudaMalloc((void**)&dy, (size_t)n * 4));
  CK(cudaMalloc((void**)&dya, (size_t)n * 4));
  CK(cudaMalloc((void**)&dlog, (size_t)cap * 8));
  CK(cudaMalloc((void**)&dflags, 16 * 8));
  CK(cudaMalloc(&ws, wsb));
  CK(cudaMalloc(&wsr, wsrb));
  CK(cudaMemsetAsync(ws, 0, wsb, st));   /* workspaces: zero-filled once */
  CK(cudaMemsetAsync(wsr, 0, wsrb, st));
  CK(cudaMemsetAsync(dflags, 0, 16 * 8, st));
  CK(cudaMemcpyAsync(dx, hx, (size_t)n * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dxa, hxa, (size_t)n * 8, cudaMemcpyHostToDevice, st));
  /* flags: [0] error bits (int32), [2..] counters; replay's at [8] / [10..] */
  VT(vt_round_log(dx, n, 32, tau, VT_OUT_F32, dy, dlog, cap, base, NULL, NULL, NULL, NULL, 0, NULL, dflags + 2,
                  (int32_t*)dflags, ws, wsb, st));
  int64_t hf[16];
  CK(cudaMemcpyAsync(hf, dflags, sizeof hf, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const int64_t count = hf[2];
  if ((int32_t)hf[0] != 0 || count < 0 || count > cap) {
    fprintf(stderr, "round-and-log: err %d, %lld entries\n", (int)(int32_t)hf[0], (long long)count);
    return 4;
  }
  VT(vt_replay(dxa, n, 32, VT_LOG_SPARSE, dlog, count, base, VT_OUT_F32, dya, dflags + 10, (int32_t*)(dflags + 8),
               wsr, wsrb, st));
  uint64_t* hlog = (uint64_t*)malloc((size_t)(count ? count : 1) * 8);
  CK(cudaMemcpyAsync(hy, dy, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hya, dya, (size_t)n * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hlog, dlog, (size_t)count * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hf, dflags, sizeof hf, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  int64_t bad_y = 0, bad_a = 0, bad_log = 0;
  for (int64_t i = 0; i < n; ++i) {
    const float f = (float)hx[i];  /* b_r = 32: rnd == round-to-nearest-even FP32 */
    if (memcmp(&f, &hy[i], 4)) ++bad_y;
    if (memcmp(&hy[i], &hya[i], 4)) ++bad_a;
  }
  for (int64_t k = 0; k < count; ++k) {
    const int64_t idx = (int64_t)(hlog[k] >> 1);
    if (idx < base || idx >= base + n || (k && (hlog[k] >> 1) <= (hlog[k - 1] >> 1))) ++bad_log;
  }
  printf("n=%lld logged=%lld (%.2f%%) corrections=%lld replay_err=%d bad_y=%lld bad_auditor=%lld bad_log=%lld\n",
         (long long)n, (long long)count, 100.0 * (double)count / (double)n, (long long)hf[10], (int)(int32_t)hf[8],
         (long long)bad_y, (long long)bad_a, (long long)bad_log);
  /* Merkle commitment of the FP32 output (little-endian bytes, 4 KiB leaves) */
  const int64_t nbytes = n * 4, leaf = 4096, leaves = (nbytes + leaf - 1) / leaf;
  const int64_t nodes = vt_merkle_node_count(leaves);
  uint8_t* dnodes;
  uint8_t root[32];
  CK(cudaMalloc((void**)&dnodes, (size_t)nodes * 32));
  VT(vt_merkle_build((const uint8_t*)dy, nbytes, leaf, dnodes, nodes, st));
  CK(cudaMemcpyAsync(root, dnodes + (nodes - 1) * 32, 32, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  printf("merkle leaves=%lld nodes=%lld root=", (long long)leaves, (long long)nodes);
  for (int k = 0; k < 32; ++k) printf("%02x", root[k]);
  printf("\n");
  if (argc > 2) {
    FILE* f = fopen(argv[2], "wb");
    if (!f || fwrite(hy, 4, (size_t)n, f) != (size_t)n) return 5;
    fclose(f);
  }
  return (bad_y || bad_a || bad_log || (int32_t)hf[8]) ? 1 : 0;
}
