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

// ================================================================== fused
constexpr int kFThreads = 256;   // 8 warps: TMEM lane quarter = warp & 3, segment = warp >> 2
constexpr int kFSlice = 512;     // K bytes per unit (2 segments of 256 per row)
constexpr int kFSeg = 256;       // symbols per chain; index seg_shift must be 8
constexpr int kFSlot = 256;      // staged stream bytes per chain (larger -> read from global)
constexpr int kFNT = 16;
constexpr uint32_t kFCols = 256; // TMEM: A in cols [0,128), accumulator at col 128

struct FusedSmem {
    TableSmem tab[2];
    alignas(1024) uint8_t x[kFSlice / 128][kFNT * 128];  // X slice, SW128 atoms (2 KB per 128 B of K)
    alignas(16) uint8_t slot[kFThreads][kFSlot + 16];
    uint64_t sbar;
    uint64_t done;
    uint32_t tmem;
    int32_t cur[2];
};

// one 16-symbol group of a chain read from a generic (global) stream pointer
__device__ __forceinline__ uint32_t gen_step(uint32_t& x, const uint8_t*& p, const uint8_t* pend, uint32_t tab) {
    const uint32_t e = lds_u32(tab + ((x & (kProbScale - 1)) << 2));
    x = (e >> 20) * ((x >> 12) - kProbScale) + (e >> 8);
    for (int k = 0; k < 2; ++k)
        if (x < kStateLower) {
            x = (x << 8) | (p < pend ? (uint32_t)*p : 0u);
            ++p;
        }
    return e;
}

__global__ void __launch_bounds__(kFThreads, 2) k_fused_decode(
    const uint8_t* __restrict__ base, const uint64_t* __restrict__ blob_off, const uint64_t* __restrict__ blob_len,
    const uint64_t* __restrict__ out_len, const uint8_t* __restrict__ codec, uint64_t chunk_size,
    const int64_t* __restrict__ seg_base, const uint32_t* __restrict__ seg_state,
    const uint32_t* __restrict__ seg_off, const GemmTensor* __restrict__ tens, const int4* __restrict__ units,
    int n_units, int ntok, int32_t* __restrict__ status) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    FusedSmem& S = *reinterpret_cast<FusedSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, part = warp >> 2;
    if (threadIdx.x == 0) {
        mbar_init(&S.sbar, kFThreads);
        mbar_init(&S.done, 1);
        fence_mbar_init();
        S.cur[0] = S.cur[1] = -1;
    }
    if (warp == 0) tmem_alloc(&S.tmem, kFCols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem;
    const uint32_t tlane = tmem + ((uint32_t)(q * 32) << 16);
    uint32_t sphase = 0, dphase = 0;

    for (int ui = blockIdx.x; ui < n_units; ui += gridDim.x) {
        const int4 u = units[ui];
        const GemmTensor T = tens[u.x];
        const int m0 = u.y, k0 = u.z;
        const int row = m0 + q * 32 + lane;
        const bool valid = row < T.n_rows;
        const int last_row = min(m0 + 127, T.n_rows - 1);
        const uint64_t g0 = (uint64_t)T.t_off + (uint64_t)m0 * T.k + k0;
        const uint64_t g1 = (uint64_t)T.t_off + (uint64_t)last_row * T.k + k0 + kFSlice - 1;
        const int c_lo = (int)(g0 / chunk_size), c_hi = (int)(g1 / chunk_size);
        if (c_hi - c_lo > 1) {  // the host never builds such units; refuse rather than mis-decode
            if (threadIdx.x == 0) atomicExch(&status[c_lo], DC_CHUNK_CHAIN);
            continue;
        }
        const uint64_t g =(uint64_t)T.t_off + (uint64_t)(valid ? row : m0) * T.k + k0 + part * kFSeg;
        const int c = (int)(g / chunk_size);
        const uint32_t o = (uint32_t)(g - (uint64_t)c * chunk_size);
        const bool ans = codec[c] == 1;
        const uint8_t* blob = base + blob_off[c];

        // ---- chain setup and stream staging (one bulk copy per chain)
        uint32_t x0 = kStateLower, xe = kStateLower, s_lo = 0, s_hi = 0;
        const uint8_t* src;
        if (ans) {
            const uint64_t nseg = (out_len[c] + kFSeg - 1) / kFSeg;
            const int64_t j = seg_base[c] + (o / kFSeg);
            x0 = seg_state[j];
            s_lo = seg_off[j];
            const bool lastseg = (o / kFSeg) + 1 >= nseg;
            s_hi = lastseg ? (uint32_t)(blob_len[c] - kHeaderBytes) : seg_off[j + 1];
            xe = lastseg ? kStateLower : seg_state[j + 1];
            src = blob + kHeaderBytes + s_lo;
        } else {
            s_hi = kFSeg;
            src = blob + o;  // stored chunk: raw bytes
        }
        const uintptr_t a16 = reinterpret_cast<uintptr_t>(src) & ~(uintptr_t)15;
        const uint32_t delta = (uint32_t)(reinterpret_cast<uintptr_t>(src) - a16);
        const uint32_t span = (s_hi >= s_lo) ? s_hi - s_lo : 0xFFFFFFFFu;
        const uint32_t nbytes = (span + delta + 15u) & ~15u;
        const bool staged = valid && span != 0xFFFFFFFFu && nbytes <= kFSlot + 16 && nbytes > 0;
        __syncthreads();  // previous unit done with slots, tables and X
        fence_proxy_async_smem();
        mbar_arrive_expect_tx(&S.sbar, staged ? nbytes : 0u);
        if (staged) bulk_g2s(S.slot[threadIdx.x], reinterpret_cast<const void*>(a16), nbytes, &S.sbar);
        // ---- decode tables for the (at most two) chunks of this unit
        const bool two = c_hi > c_lo;
        for (int t = 0; t < 1 + (int)two; ++t) {
            const int ct = c_lo + t;
            if (S.cur[t] != ct) {  // uniform: every thread reads the same S.cur
                __syncthreads();
                if (codec[ct] == 1) build_decode_table(base + blob_off[ct], S.tab[t]);
                __syncthreads();
                if (threadIdx.x == 0) S.cur[t] = ct;
            }
        }
        load_x_sw128<kFNT>(&S.x[0][0], T.x, ntok, T.k, k0, kFSlice);
        mbar_wait(&S.sbar, sphase);
        sphase ^= 1u;
        __syncthreads();  // S.cur / tables visible

        // ---- decode 256 symbols of this row into TMEM columns [part*64, part*64+64)
        const TableSmem& TB = S.tab[c - c_lo];
        const uint32_t tab = smem_u32(TB.tab);
        const int mode = !valid ? 3 : (!ans ? 1 : (TB.single >= 0 ? 2 : (staged ? 0 : 4)));
        const bool fast = __all_sync(0xffffffffu, mode == 0);
        uint32_t x = x0;
        uint32_t p = smem_u32(S.slot[threadIdx.x]) + delta;
        const uint32_t pbase = p;
        uint32_t nb = staged ? lds_u8(p) : 0u;
        const uint8_t* gp = src;
        const uint8_t* gend = blob + kHeaderBytes + s_hi;
        const uint32_t col0 = tlane + (uint32_t)part * (kFSeg / 4);
        for (int grp = 0; grp < kFSeg / 16; ++grp) {
            uint32_t w[4];
            if (fast) {
#pragma unroll
                for (int v = 0; v < 16; ++v) w[v >> 2] = put_byte(w[v >> 2], dec_step<true>(x, p, nb, tab), v & 3);
            } else {
#pragma unroll 1
                for (int v = 0; v < 16; ++v) {
                    uint32_t e;
                    if (mode == 0) e = dec_step<false>(x, p, nb, tab);
                    else if (mode == 4) e = gen_step(x, gp, gend, tab);
                    else if (mode == 1) e = lds_u8(p + grp * 16 + v);
                    else if (mode == 2) e = (uint32_t)TB.single;
                    else e = 0u;
                    w[v >> 2] = put_byte(w[v >> 2], e, v & 3);
                }
            }
            tmem_st_32x32b_x4(col0 + grp * 4, w[0], w[1], w[2], w[3]);
        }
        // chain check: the segment must end on the next split point
        if (mode == 0 || mode == 4) {
            const uint32_t pend = (mode == 0) ? (p - pbase) : (uint32_t)(gp - src);
            if (x != xe || pend != span) atomicExch(&status[c], DC_CHUNK_CHAIN);
        } else if (mode == 2 && (x0 != kStateLower || s_hi != s_lo)) {
            atomicExch(&status[c], DC_CHUNK_CORRUPT);
        }
        tmem_wait_st();
        fence_proxy_async_smem();  // X tile written with generic stores
        tc_fence_before();
        __syncthreads();

        // ---- MMA: 16 x (128 x 16 x 32), A from TMEM, X from smem
        if (threadIdx.x == 0) {
            tc_fence_after();
            constexpr uint32_t idesc = idesc_i8(128, kFNT);
#pragma unroll
            for (int ks = 0; ks < kFSlice / 32; ++ks)
                mma_i8_ts(tmem + 128, tmem + ks * 8, sw128_kmajor_desc(smem_u32(S.x[ks >> 2]) + 32 * (ks & 3)), idesc,
                          ks > 0);
            mma_commit(&S.done);
        }
        __syncwarp();
        mbar_wait(&S.done, dphase);
        dphase ^= 1u;
        tc_fence_after();
        if (part == 0) {  // warps 0-3 read the accumulator quarter they own
            uint32_t acc[16];
            tmem_ld_32x32b_x16(tlane + 128, acc);
            if (valid) {
#pragma unroll
                for (int t = 0; t < kFNT; ++t)
                    if (t < ntok) atomicAdd(&T.acc[(int64_t)t * T.n_rows + row], (int32_t)acc[t]);
            }
        }
        tc_fence_before();
    }
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, kFCols);
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

extern "C" int dc_fused_slice_bytes(void) { return kFSlice; }

// Fused decompress -> W8A8 over DCC1 chunks.  units: int4 (layer, m0, k0, 0)
// with k0 % 512 == 0; the index must use 256-symbol segments (seg_shift 8);
// chunk_size, every layer's t_off and k must be multiples of 512 and a unit's
// 128 rows must span at most two chunks.
extern "C" int dc_fused_decode_gemm(const uint8_t* base, const uint64_t* blob_off, const uint64_t* blob_len,
                                    const uint64_t* out_len, const uint8_t* codec, uint64_t chunk_size,
                                    const int64_t* seg_base, const uint32_t* seg_state, const uint32_t* seg_off,
                                    const void* tens, const int32_t* units, int64_t n_units, int ntok,
                                    int32_t* status, void* stream) {
    if (n_units <= 0 || ntok <= 0 || ntok > kFNT || chunk_size % kFSlice) return DC_ERR_ARG;
    const size_t smem = sizeof(FusedSmem) + 1024;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_fused_decode, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = n_units < 2LL * sms ? n_units : 2LL * sms;
    k_fused_decode<<<(unsigned)grid, kFThreads, smem, (cudaStream_t)stream>>>(
        base, blob_off, blob_len, out_len, codec, chunk_size, seg_base, seg_state, seg_off,
        reinterpret_cast<const GemmTensor*>(tens), reinterpret_cast<const int4*>(units), (int)n_units, ntok, status);
    DC_CHECK_LAUNCH("k_fused_decode");
    return DC_OK;
}
