// Library-wide C ABI plumbing: version string and a thread-local last-error
// message.  Entry points live next to their kernels (vt_round.cu,
// vt_codec.cu, vt_tau.cu, vt_sha256.cu); see include/vtrain_b200.h.
#include <cstdio>
#include <cstring>

#include "vt_common.cuh"

namespace {
thread_local char g_err[512] = "";
}

void vt_set_error(const char* what) {
  std::snprintf(g_err, sizeof(g_err), "%s", what);
}

int vt_check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return VT_OK;
  std::snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
  return VT_ECUDA;
}

extern "C" const char* vt_version(void) { return "vtrain_b200 0.1.0 sm_100a"; }

extern "C" const char* vt_last_error(void) { return g_err; }

// Host wait for a stream (the reference-API channels' one wait per call,
// without a round trip through torch's stream objects).
extern "C" int vt_stream_synchronize(vt_stream_t stream) {
  const cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e == cudaSuccess) return VT_OK;
  std::snprintf(g_err, sizeof(g_err), "vt_stream_synchronize: %s", cudaGetErrorString(e));
  return VT_ECUDA;
}
