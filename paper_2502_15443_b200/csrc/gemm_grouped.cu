// Grouped W8A8 GEMM and the fused decompress -> W8A8 GEMM (north-star kernel 3).
//
// Both run one "unit" = 128 weight rows x a K-slice of one linear layer per
// CTA step and accumulate exact int32 partial products into that layer's
// [ntok][n_rows] accumulator with atomics (split-K).  All linears of a model
// go in ONE launch (a unit table), so a decode step is not launch-bound.
//
// k_w8a8_grouped   uncompressed INT8 weights: TMA (SWIZZLE_128B) -> smem ->
//                  tcgen05.mma.kind::i8 (A, B from smem) -> TMEM accumulator.
// k_fused_decode   compressed weights (DCC1 chunks + split-point index):
//                  every thread decodes one 256-symbol segment of one weight
//                  row (the row's TMEM lane) straight from the rANS stream,
//                  16 bytes at a time into registers, and writes them to TMEM
//                  with tcgen05.st; tcgen05.mma then takes A from TMEM and X
//                  from smem.  Decoded weights never touch HBM (or smem).
//                  Segment chains are checked like k_decode_segments; a
//                  mismatch flags the chunk (DC_CHUNK_CHAIN) so the host falls
//                  back to the exact path.
#include "common.cuh"
#include "rans_common.cuh"
#include "tc.cuh"

namespace dc {

struct GemmTensor {  // 32 bytes, device array
    const int8_t* x;     // [ntok][k] quantized activations
    int32_t* acc;        // [ntok][n_rows] int32 accumulator (zeroed by caller)
    int64_t t_off;       // byte offset of the weight matrix in the payload
    int32_t n_rows;
    int32_t k;
};

__device__ __forceinline__ void tmem_st_32x32b_x4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(a), "r"(b),
                 "r"(c), "r"(d)
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// D[tmem] (+)= A[tmem] * B[smem]^T (int8 -> int32), one thread.
__device__ __forceinline__ void mma_i8_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// Load X[:, k0:k0+bytes) (ntok rows, zero padded to NT) into SWIZZLE_128B
// K-major atoms: stage s (128 B of K) at xs + s*NT*128, row r at r*128,
// 16-B chunk j at ((j ^ (r & 7)) << 4).  Generic-proxy stores: the caller
// issues fence.proxy.async before the MMA reads them.
template <int NT>
__device__ __forceinline__ void load_x_sw128(uint8_t* xs, const int8_t* __restrict__ x, int ntok, int k, int k0,
                                             int bytes) {
    const int chunks = NT * (bytes >> 4);  // 16-B pieces
    for (int i = threadIdx.x; i < chunks; i += blockDim.x) {
        const int r = i % NT, cj = i / NT;  // cj = 16-B chunk index along K
        const int s = cj >> 3, j = cj & 7;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (r < ntok) v = *reinterpret_cast<const uint4*>(x + (int64_t)r * k + k0 + (cj << 4));
        *reinterpret_cast<uint4*>(xs + s * NT * 128 + r * 128 + ((j ^ (r & 7)) << 4)) = v;
    }
}

// ================================================================ grouped
constexpr int kGrThreads = 128;
constexpr int kGrBK = 128;
constexpr int kGrStages = 6;
constexpr int kGrNT = 16;

struct GroupedSmem {
    alignas(1024) uint8_t a[kGrStages][128 * kGrBK];
    alignas(1024) uint8_t b[kGrStages][kGrNT * kGrBK];  // 16 rows x 128 B (two 1 KB swizzle atoms)
    uint64_t full[kGrStages];
    uint64_t empty[kGrStages];
    uint64_t done;
    uint32_t tmem;
};

// units: (tensor, m0, k0, kslice); maps: 2 CUtensorMaps per tensor (W, X)
__global__ void __launch_bounds__(kGrThreads, 1) k_w8a8_grouped(const CUtensorMap* __restrict__ maps,
                                                                 const GemmTensor* __restrict__ tens,
                                                                 const int4* __restrict__ units, int ntok) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    GroupedSmem& S = *reinterpret_cast<GroupedSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int4 u = units[blockIdx.x];
    const GemmTensor T = tens[u.x];
    const CUtensorMap* tw = maps + 2 * u.x;
    const CUtensorMap* tx = maps + 2 * u.x + 1;
    const int m0 = u.y, k0 = u.z, nkb = u.w / kGrBK;
    constexpr uint32_t kBytes = 128 * kGrBK + kGrNT * kGrBK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kGrStages; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], 1);
        }
        mbar_init(&S.done, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(&S.tmem, 32);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem;
    if (warp == 0 && lane == 0) {
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % kGrStages;
            mbar_wait(&S.empty[s], ((kb / kGrStages) & 1) ^ 1);
            mbar_arrive_expect_tx(&S.full[s], kBytes);
            tma_load_2d(S.a[s], tw, k0 + kb * kGrBK, m0, &S.full[s]);
            tma_load_2d(S.b[s], tx, k0 + kb * kGrBK, 0, &S.full[s]);
        }
    } else if (warp == 1 && lane == 0) {
        constexpr uint32_t idesc = idesc_i8(128, kGrNT);
        for (int kb = 0; kb < nkb; ++kb) {
            const int s = kb % kGrStages;
            mbar_wait(&S.full[s], (kb / kGrStages) & 1);
            tc_fence_after();
            const uint32_t a0 = smem_u32(S.a[s]), b0 = smem_u32(S.b[s]);
#pragma unroll
            for (int k = 0; k < kGrBK / 32; ++k)
                mma_i8(tmem, sw128_kmajor_desc(a0 + 32 * k), sw128_kmajor_desc(b0 + 32 * k), idesc, (kb | k) != 0);
            mma_commit(&S.empty[s]);
        }
        mma_commit(&S.done);
    }
    __syncwarp();
    mbar_wait(&S.done, 0);
    tc_fence_after();
    const int row = m0 + warp * 32 + lane;
    uint32_t v[16];
    tmem_ld_32x32b_x16(tmem + ((uint32_t)(warp * 32) << 16), v);
    if (row < T.n_rows) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (j < ntok) atomicAdd(&T.acc[(int64_t)j * T.n_rows + row], (int32_t)v[j]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, 32);
}

// ====================================================== grouped, persistent
// One CTA per SM (221 KB of smem: 12 TMA stages of W + X), looping over the
// unit table with stride gridDim.x.  Warp 0 streams W/X tiles with TMA
// continuously across units, warp 1 issues the MMAs into one of two TMEM
// accumulators (double-buffered per unit), warps 2-5 drain the other one
// (tcgen05.ld -> int32 atomics) while the next unit streams.  Because one CTA
// fills an SM, a capped grid occupies exactly that many SMs: the rest are
// left to a concurrent fused decode kernel (MixedStep).
constexpr int kPThreads = 192;
constexpr int kPStages = 12;

struct PersistSmem {
    alignas(1024) uint8_t a[kPStages][128 * kGrBK];
    alignas(1024) uint8_t b[kPStages][kGrNT * kGrBK];
    uint64_t full[kPStages];
    uint64_t empty[kPStages];
    uint64_t accf[2];  // accumulator ub ready (MMA commit)
    uint64_t acce[2];  // accumulator ub drained (4 epilogue warps)
    uint32_t tmem;
};

__global__ void __launch_bounds__(kPThreads, 1) k_w8a8_persist(const CUtensorMap* __restrict__ maps,
                                                                const GemmTensor* __restrict__ tens,
                                                                const int4* __restrict__ units, int n_units,
                                                                int ntok) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    PersistSmem& S = *reinterpret_cast<PersistSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t kBytes = 128 * kGrBK + kGrNT * kGrBK;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kPStages; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&S.accf[b], 1);
            mbar_init(&S.acce[b], 4);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(&S.tmem, 32);  // two 16-column int32 accumulators
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem;

    if (warp == 0) {
        if (lane == 0) {
            uint32_t it = 0;
            for (int ui = blockIdx.x; ui < n_units; ui += gridDim.x) {
                const int4 u = units[ui];
                const CUtensorMap* tw = maps + 2 * u.x;
                const CUtensorMap* tx = maps + 2 * u.x + 1;
                const int nkb = u.w / kGrBK;
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const uint32_t s = it % kPStages;
                    mbar_wait(&S.empty[s], ((it / kPStages) & 1) ^ 1);
                    mbar_arrive_expect_tx(&S.full[s], kBytes);
                    tma_load_2d(S.a[s], tw, u.z + kb * kGrBK, u.y, &S.full[s]);
                    tma_load_2d(S.b[s], tx, u.z + kb * kGrBK, 0, &S.full[s]);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_i8(128, kGrNT);
            uint32_t it = 0, j = 0;
            for (int ui = blockIdx.x; ui < n_units; ui += gridDim.x, ++j) {
                const int nkb = units[ui].w / kGrBK;
                const uint32_t ub = j & 1;
                mbar_wait(&S.acce[ub], ((j >> 1) & 1) ^ 1);  // epilogue drained this accumulator
                tc_fence_after();
                for (int kb = 0; kb < nkb; ++kb, ++it) {
                    const uint32_t s = it % kPStages;
                    mbar_wait(&S.full[s], (it / kPStages) & 1);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(S.a[s]), b0 = smem_u32(S.b[s]);
#pragma unroll
                    for (int k = 0; k < kGrBK / 32; ++k)
                        mma_i8(tmem + ub * kGrNT, sw128_kmajor_desc(a0 + 32 * k), sw128_kmajor_desc(b0 + 32 * k),
                               idesc, (kb | k) != 0);
                    mma_commit(&S.empty[s]);
                }
                mma_commit(&S.accf[ub]);
            }
        }
    } else {
        const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31 (warps 2,3,4,5 -> 2,3,0,1)
        uint32_t j = 0;
        for (int ui = blockIdx.x; ui < n_units; ui += gridDim.x, ++j) {
            const int4 u = units[ui];
            const uint32_t ub = j & 1;
            mbar_wait(&S.accf[ub], (j >> 1) & 1);
            tc_fence_after();
            uint32_t v[16];
            tmem_ld_32x32b_x16(tmem + ((uint32_t)(quarter * 32) << 16) + ub * kGrNT, v);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&S.acce[ub]);
            const GemmTensor T = tens[u.x];
            const int row = u.y + quarter * 32 + lane;
            if (row < T.n_rows) {
#pragma unroll
                for (int t = 0; t < kGrNT; ++t)
                    if (t < ntok) atomicAdd(&T.acc[(int64_t)t * T.n_rows + row], (int32_t)v[t]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 32);
}

int make_tmap_i8(CUtensorMap* m, const void* base, uint64_t rows, uint64_t k, uint32_t box_rows);  // gemm_w8a8.cu

static int make_maps(CUtensorMap* maps_host, const int8_t* const* w, const int8_t* const* x, const int64_t* rows,
                     const int64_t* k, int n, int ntok) {
    for (int i = 0; i < n; ++i) {
        if (make_tmap_i8(&maps_host[2 * i], w[i], rows[i], k[i], 128)) return DC_ERR_CUDA;
        if (make_tmap_i8(&maps_host[2 * i + 1], x[i], ntok, k[i], kGrNT)) return DC_ERR_CUDA;
    }
    return DC_OK;
}

}  // namespace dc

using namespace dc;

extern "C" int dc_gemm_tensor_bytes(void) { return (int)sizeof(GemmTensor); }
extern "C" int dc_tmap_bytes(void) { return (int)sizeof(CUtensorMap); }

// Build the 2 tensor maps per layer (host memory, 64-B aligned, n*2 maps).
extern "C" int dc_w8a8_grouped_maps(const int8_t* const* w_host, const int8_t* const* x_host,
                                    const int64_t* rows_host, const int64_t* k_host, int n, int ntok,
                                    void* maps_host) {
    if (n <= 0 || ntok <= 0 || ntok > kGrNT) return DC_ERR_ARG;
    return make_maps(reinterpret_cast<CUtensorMap*>(maps_host), w_host, x_host, rows_host, k_host, n, ntok);
}

// Grouped uncompressed W8A8: maps (device, 2 per layer), tens (device
// GemmTensor[n_layers]), units (device int4 (layer, m0, k0, kslice)).
extern "C" int dc_w8a8_grouped(const void* maps, const void* tens, const int32_t* units, int64_t n_units, int ntok,
                               void* stream) {
    if (n_units <= 0 || ntok <= 0 || ntok > kGrNT) return DC_ERR_ARG;
    const size_t smem = sizeof(GroupedSmem) + 1024;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_w8a8_grouped, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    k_w8a8_grouped<<<(unsigned)n_units, kGrThreads, smem, (cudaStream_t)stream>>>(
        reinterpret_cast<const CUtensorMap*>(maps), reinterpret_cast<const GemmTensor*>(tens),
        reinterpret_cast<const int4*>(units), ntok);
    DC_CHECK_LAUNCH("k_w8a8_grouped");
    return DC_OK;
}

// Persistent variant of dc_w8a8_grouped: min(n_units, SMs, max_ctas > 0 ?
// max_ctas : SMs) CTAs, one per SM.
extern "C" int dc_w8a8_grouped_persist(const void* maps, const void* tens, const int32_t* units, int64_t n_units,
                                       int ntok, int max_ctas, void* stream) {
    if (n_units <= 0 || ntok <= 0 || ntok > kGrNT) return DC_ERR_ARG;
    const size_t smem = sizeof(PersistSmem) + 1024;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_w8a8_persist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (max_ctas > 0 && max_ctas < sms) sms = max_ctas;
    const int64_t grid = n_units < sms ? n_units : sms;
    k_w8a8_persist<<<(unsigned)grid, kPThreads, smem, (cudaStream_t)stream>>>(
        reinterpret_cast<const CUtensorMap*>(maps), reinterpret_cast<const GemmTensor*>(tens),
        reinterpret_cast<const int4*>(units), (int)n_units, ntok);
    DC_CHECK_LAUNCH("k_w8a8_persist");
    return DC_OK;
}
