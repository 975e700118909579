// capi.cu -- status strings and CUDA error plumbing for the C ABI (include/gsx.h).
#include <stdio.h>

#include "gsx_common.cuh"

static thread_local char g_last_err[256] = "";

void gsx_set_cuda_error(cudaError_t e) {
  snprintf(g_last_err, sizeof g_last_err, "%s: %s", cudaGetErrorName(e), cudaGetErrorString(e));
}

int gsx_check_launch() {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    gsx_set_cuda_error(e);
    return GSX_ERR_CUDA;
  }
  return GSX_OK;
}

extern "C" const char* gsx_last_cuda_error(void) { return g_last_err; }

extern "C" int gsx_abi_version(void) { return GSX_ABI_VERSION; }

extern "C" const char* gsx_status_string(int status) {
  switch (status) {
    case GSX_OK: return "ok";
    case GSX_ERR_EMPTY: return "empty scene";
    case GSX_ERR_VALIDATION: return "invalid primitive record";
    case GSX_ERR_OVERFLOW: return "hit buffer overflow";
    case GSX_ERR_ARG: return "invalid argument";
    case GSX_ERR_CUDA: return "CUDA error";
    case GSX_ERR_STACK: return "traversal stack exhausted";
    default: return "unknown status";
  }
}

// Tile order of camera launches (gsx_tile_at, gsx_common.cuh) for hosts that
// shard or assemble frames: the host never keeps its own copy of the order.
extern "C" int64_t gsx_tile_id(int64_t s, int64_t tiles_x, int64_t tiles_y, int64_t stride) {
  if (tiles_x < 1 || tiles_y < 1 || s < 0 || s >= tiles_x * tiles_y || stride < 1) return -1;
  return gsx_tile_at(s, tiles_x, tiles_y, stride);
}
