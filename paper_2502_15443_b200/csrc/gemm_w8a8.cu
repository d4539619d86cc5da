// Decode-shaped W8A8 GEMM on the 5th-gen tensor cores (sm_100a):
//     acc[t, n] = sum_k Xq[t, k] * Wq[n, k]      int8 x int8 -> exact int32
// This is the integer core of the reference's W8A8 numerics
// (scaling.py:127-152, simulate_layer: (qx*sx)(qw*sw)^T); the caller applies
// sx*sw.  Swap-AB: weight rows are UMMA M (128 per CTA), tokens are UMMA N
// (16..64, zero-padded by TMA), so a GEMV-like decode step still fills the
// tensor core.  Pipeline per CTA (128 threads):
//   warp 0 / lane 0  TMA producer: W tile 128 x 128 B + X tile N x 128 B per
//                    stage, SWIZZLE_128B, mbarrier expect_tx
//   warp 1 / lane 0  MMA issuer: 4 x tcgen05.mma.kind::i8 (K = 32) per stage,
//                    tcgen05.commit frees the stage
//   warps 0-3        epilogue: tcgen05.ld of the int32 accumulator (TMEM
//                    lanes = weight rows) -> exact int32 atomics (split-K)
#include "common.cuh"
#include "tc.cuh"

namespace dc {

constexpr int kGThreads = 128;
constexpr int kBM = 128;     // weight rows per tile
constexpr int kBK = 128;     // K bytes per stage (one 128-byte swizzle row)
constexpr int kStages = 6;

template <int NT>
struct GemmSmem {
    alignas(1024) uint8_t a[kStages][kBM * kBK];
    alignas(1024) uint8_t b[kStages][NT * kBK < 1024 ? 1024 : NT * kBK];
    uint64_t full[kStages];
    uint64_t empty[kStages];
    uint64_t done;
    uint32_t tmem;
};

template <int NT>
__global__ void __launch_bounds__(kGThreads, 1)
    k_w8a8_gemm(const __grid_constant__ CUtensorMap tm_w, const __grid_constant__ CUtensorMap tm_x, int n_rows,
                int kslice, int ntok, int32_t* __restrict__ yacc, int atomic_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    GemmSmem<NT>& S = *reinterpret_cast<GemmSmem<NT>*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * kBM;
    const int k0 = blockIdx.y * kslice;
    const int nkb = kslice / kBK;
    constexpr uint32_t kBytesA = kBM * kBK, kBytesB = NT * kBK;

    if (threadIdx.x == 0) {
        prefetch_tmap(&tm_w);
        prefetch_tmap(&tm_x);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], 1);
        }
        mbar_init(&S.done, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(&S.tmem, 32);  // N <= 32 columns of int32
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem;

    if (warp == 0 && lane == 0) {
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % kStages;
            const uint32_t ph = (kb / kStages) & 1;
            mbar_wait(&S.empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&S.full[s], kBytesA + kBytesB);
            tma_load_2d(S.a[s], &tm_w, k0 + kb * kBK, m0, &S.full[s]);
            tma_load_2d(S.b[s], &tm_x, k0 + kb * kBK, 0, &S.full[s]);
        }
    } else if (warp == 1 && lane == 0) {
        constexpr uint32_t idesc = idesc_i8(kBM, NT);
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % kStages;
            const uint32_t ph = (kb / kStages) & 1;
            mbar_wait(&S.full[s], ph);
            tc_fence_after();
            const uint32_t a0 = smem_u32(S.a[s]), b0 = smem_u32(S.b[s]);
#pragma unroll
            for (int k = 0; k < kBK / 32; ++k)
                mma_i8(tmem, sw128_kmajor_desc(a0 + 32 * k), sw128_kmajor_desc(b0 + 32 * k), idesc, (kb | k) != 0);
            mma_commit(&S.empty[s]);
        }
        mma_commit(&S.done);
    }
    __syncwarp();

    // epilogue: TMEM lane (32*warp + lane) = weight row m0 + 32*warp + lane
    mbar_wait(&S.done, 0);
    tc_fence_after();
    const int row = m0 + warp * 32 + lane;
#pragma unroll
    for (int c0 = 0; c0 < NT; c0 += 16) {
        uint32_t v[16];
        tmem_ld_32x32b_x16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
        if (row < n_rows) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int t = c0 + j;
                if (t < ntok) {
                    if (atomic_out)
                        atomicAdd(&yacc[(int64_t)t * n_rows + row], (int32_t)v[j]);
                    else
                        yacc[(int64_t)t * n_rows + row] = (int32_t)v[j];
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, 32);
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    }
    return fn;
}

// row-major [rows][k] int8, box {128 bytes of K, box_rows}, SWIZZLE_128B
int make_tmap_i8(CUtensorMap* m, const void* base, uint64_t rows, uint64_t k, uint32_t box_rows) {
    EncodeFn fn = encode_fn();
    if (!fn) return DC_ERR_CUDA;
    cuuint64_t dims[2] = {k, rows};
    cuuint64_t strides[1] = {k};
    cuuint32_t box[2] = {(cuuint32_t)kBK, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? DC_OK : DC_ERR_CUDA;
}

template <int NT>
static int launch_gemm(const int8_t* w, int64_t n_rows, int64_t k, const int8_t* x, int64_t ntok, int32_t* yacc,
                       int64_t kslice, cudaStream_t st) {
    CUtensorMap tw, tx;
    if (make_tmap_i8(&tw, w, n_rows, k, kBM) || make_tmap_i8(&tx, x, ntok, k, NT)) {
        set_error_msg("cuTensorMapEncodeTiled failed");
        return DC_ERR_CUDA;
    }
    const size_t smem = sizeof(GemmSmem<NT>) + 1024;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_w8a8_gemm<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    dim3 grid((unsigned)((n_rows + kBM - 1) / kBM), (unsigned)(k / kslice));
    k_w8a8_gemm<NT><<<grid, kGThreads, smem, st>>>(tw, tx, (int)n_rows, (int)kslice, (int)ntok, yacc,
                                                   grid.y > 1 ? 1 : 0);
    DC_CHECK_LAUNCH("k_w8a8_gemm");
    return DC_OK;
}

}  // namespace dc

using namespace dc;

// acc[t, n] (+)= sum_k x[t, k] * w[n, k].  w: [n_rows][k], x: [ntok][k] int8,
// row-major, k a multiple of 128, ntok <= 32.  kslice (multiple of 128,
// dividing k) splits K across CTAs; with kslice < k the int32 results are
// atomically accumulated into yacc (caller zeroes it), else stored.
extern "C" int dc_w8a8_gemm(const int8_t* w, int64_t n_rows, int64_t k, const int8_t* x, int64_t ntok,
                            int32_t* yacc, int64_t kslice, void* stream) {
    if (n_rows <= 0 || k <= 0 || k % kBK || ntok <= 0 || ntok > 32 || kslice <= 0 || kslice % kBK ||
        k % kslice)
        return DC_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    return ntok <= 16 ? launch_gemm<16>(w, n_rows, k, x, ntok, yacc, kslice, st)
                      : launch_gemm<32>(w, n_rows, k, x, ntok, yacc, kslice, st);
}
