// Library-level C ABI: version, last error, device info.
#include <stdio.h>
#include <string.h>

#include "common.cuh"

namespace dc {
static thread_local char g_err[512] = "";
void set_error(const char* what, cudaError_t e) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
}
void set_error_msg(const char* msg) { snprintf(g_err, sizeof(g_err), "%s", msg); }
}  // namespace dc

extern "C" int dc_version(void) { return 1; }

extern "C" const char* dc_last_error(void) { return dc::g_err; }

extern "C" int dc_device_sm_count(int device) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return DC_ERR_CUDA;
    return n;
}
