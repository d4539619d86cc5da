// Shared device helpers for the dcomp B200 library (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dcomp_b200.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "dcomp_b200 is written for sm_100a (B200) only"
#endif

namespace dc {

// rANS constants: reference ans.py:32-40.
constexpr uint32_t kProbBits = 12;
constexpr uint32_t kProbScale = 1u << kProbBits;
constexpr uint32_t kStateLower = 1u << 20;
constexpr uint32_t kStateUpper = 1u << 28;
constexpr uint32_t kTableBytes = 384;
constexpr uint32_t kHeaderBytes = 388;
constexpr uint32_t kCheckBlock = 4096;  // ans.py:39 _BLOCK (over-read check cadence)

// Every device buffer the library reads stream bytes from is allocated with
// this many readable bytes past its logical end (Python side guarantees it),
// so per-lane byte fetches on corrupt streams stay in bounds.
constexpr uint32_t kReadSlack = 16384;

void set_error(const char* what, cudaError_t e);
void set_error_msg(const char* msg);

#define DC_CHECK_LAUNCH(name)                         \
    do {                                              \
        cudaError_t _e = cudaGetLastError();          \
        if (_e != cudaSuccess) {                      \
            ::dc::set_error(name, _e);                \
            return DC_ERR_CUDA;                       \
        }                                             \
    } while (0)

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t warp_id() { return threadIdx.x >> 5; }

// Unpack the 384-byte u12 table of blob `b` into freq[256] (ans.py:256-262,
// :284-299).  Called by 128 threads of a CTA; returns via smem.
__device__ __forceinline__ void unpack_pair(const uint8_t* t, int i, uint32_t& a, uint32_t& b) {
    uint32_t b0 = t[3 * i], b1 = t[3 * i + 1], b2 = t[3 * i + 2];
    a = b0 | ((b1 & 0x0F) << 8);
    b = (b1 >> 4) | (b2 << 4);
}

__device__ __forceinline__ uint32_t ld_u32_le_unaligned(const uint8_t* p) {
    return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

}  // namespace dc
