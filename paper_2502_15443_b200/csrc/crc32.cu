// Parallel CRC-32/ISO-HDLC (zlib.crc32) of many byte ranges on B200.
//
// The reference checks every chunk with zlib.crc32 (container.py:169, :329),
// a byte-serial recurrence.  CRC is affine over GF(2), so a range D split into
// pieces D_j of P bytes (counted from the END of the range) satisfies
//     crc(D) = XOR_j  L(D_j) * x^(8*P*j)  mod G   ^  (~0 * x^(8|D|) mod G) ^ ~0
// where L is the zero-init, no-final-xor ("linear") CRC of a piece.  Every
// thread computes L of one piece with slicing-by-8 tables in shared memory,
// multiplies by the precomputed power for its distance from the range end,
// and the products are XOR-reduced (order-independent, deterministic).  A
// partial first piece is zero-padded on the left, which L ignores.
//
// Two kernels share that decomposition:
//   k_crc_lanes   the bulk: ranges whose end is 16-B aligned, in whole 4 KB
//                 lane pieces counted from the end.  One persistent CTA per
//                 SM; every lane streams its own piece through a 3-slot shared
//                 ring with TMA bulk copies (no L1 wavefronts for the data)
//                 and runs slicing-by-4 over tables replicated 32 times so
//                 that lane l always reads bank l: conflict-free lookups.
//   k_crc_pieces  everything else (the < 4 KB head of those ranges, and
//                 ranges with an unaligned end) in 256-byte pieces.
#include "common.cuh"
#include "ptx.cuh"
#include "tc.cuh"

namespace dc {

int sm_count();  // rans_decode.cu
int make_tmap_i8(CUtensorMap* m, const void* base, uint64_t rows, uint64_t k, uint32_t box_rows);  // gemm_w8a8.cu

constexpr uint32_t kPoly = 0xEDB88320u;
constexpr uint32_t kPiece = 256;          // bytes per thread
constexpr int kCrcThreads = 256;
constexpr uint32_t kPowLo = 1u << 16;     // M_lo[j] = x^(8*P*j),          j < 2^16
                                          // M_hi[k] = x^(8*P*2^16*k),     k < 2^16

__constant__ uint32_t c_x2n[64];  // x^(2^k) mod G, k = 0..63
__device__ uint32_t g_pow_lo[kPowLo];
__device__ uint32_t g_pow_hi[kPowLo];

__host__ __device__ inline uint32_t multmodp(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
    }
    return p;
}

// x^(n * 2^k) mod G from the x^(2^k) table (zlib's x2nmodp).
__device__ inline uint32_t x2nmodp_dev(uint64_t n, unsigned k) {
    uint32_t p = 1u << 31;
    while (n) {
        if (n & 1) p = multmodp(c_x2n[k & 63], p);
        n >>= 1;
        ++k;
    }
    return p;
}

__global__ void k_init_pows() {
    const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= kPowLo) return;
    g_pow_lo[j] = x2nmodp_dev((uint64_t)j * kPiece, 3);
    g_pow_hi[j] = x2nmodp_dev((uint64_t)j * kPiece * kPowLo, 3);
}

__device__ __forceinline__ uint32_t pow_for(uint64_t j) {
    const uint32_t lo = g_pow_lo[j & (kPowLo - 1)];
    const uint64_t hi = j >> 16;
    return hi ? multmodp(g_pow_hi[hi & (kPowLo - 1)], lo) : lo;
}

// ------------------------------------------------------------ k_crc_lanes
// Task = one 64 KB span of a range (spans counted from the range end), 32
// rounds of 2 KB.  A round is ONE 2-D TMA copy (16 rows x 128 B, SWIZZLE_128B)
// into a ring slot; lane l owns the 64-byte block [64 l, 64 l + 64) of every
// round, so its chain runs over blocks 2 KB apart: before each block the
// state is advanced over the 1984-byte gap (c <- c * x^(8*1984) mod G, four
// lookups in small shift tables), then the block's 16 words go through
// slicing-by-4 (tables replicated 32x so lane l always reads bank l).  The
// swizzle makes each lane's four 16-byte loads bank-conflict-free.
#ifndef DC_CRC_SLOTS
#define DC_CRC_SLOTS 1  // measured: warps, not prefetch depth, hide the latency (1 slot x 32 warps: 4.46 TB/s; 3 x 14: 3.41)
#endif
#ifndef DC_CRC_L2PF
#define DC_CRC_L2PF 1  // L2 prefetch of the next round: +3 % (tools/ab_crc.sh)
#endif
#ifndef DC_CRC_WARPS
#define DC_CRC_WARPS 32
#endif
constexpr uint32_t kSpanBytes = 65536;
constexpr uint32_t kRoundBytes = 2048;
constexpr uint32_t kRounds = kSpanBytes / kRoundBytes;  // 32
constexpr uint32_t kRingSlots = DC_CRC_SLOTS;
constexpr int kLaneWarps = DC_CRC_WARPS;
constexpr uint32_t kTabBytes = 4 * 256 * 32 * 4;        // 4 tables x 256 entries x 32 lane copies
constexpr uint32_t kShiftBytes = 4 * 256 * 4;           // gap-shift tables
constexpr size_t kLaneSmem = kTabBytes + kShiftBytes + (size_t)kLaneWarps * kRingSlots * kRoundBytes +
                             kLaneWarps * kRingSlots * 8 + 1024;

__device__ uint32_t g_crc_t4[4][256];     // slicing-by-4 tables
__device__ uint32_t g_crc_gap[4][256];    // S_k[i] = (i << 8k) * x^(8*1984) mod G
__device__ uint32_t g_crc_lanepow[32];    // x^(8*64*(31-l)) mod G

// The lane kernel takes a range iff its end is 128-B aligned against the map
// base (whole rows of the 2-D view) and it holds at least one span.
__device__ __forceinline__ uint64_t fast_spans(uint64_t map_base, const uint8_t* data, uint64_t off, uint64_t len) {
    if (!map_base) return 0;
    return ((reinterpret_cast<uint64_t>(data) + off + len - map_base) & 127) == 0 ? len / kSpanBytes : 0;
}

__global__ void __launch_bounds__(kCrcThreads) k_crc_pieces(uint64_t map_base, const uint8_t* __restrict__ data,
                                                             const uint64_t* __restrict__ off,
                                                             const uint64_t* __restrict__ len, int64_t n,
                                                             uint32_t* __restrict__ acc) {
    __shared__ uint32_t T[8][256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
        T[0][i] = c;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = T[0][i];
        for (int t = 1; t < 8; ++t) {
            c = (c >> 8) ^ T[0][c & 0xFF];
            T[t][i] = c;
        }
    }
    __syncthreads();
    for (int64_t r = blockIdx.y; r < n; r += gridDim.y) {
        const uint64_t L = len[r];
        const uint64_t j = (uint64_t)blockIdx.x * kCrcThreads + threadIdx.x;  // piece index from the end
        const uint64_t npieces = (L + kPiece - 1) / kPiece;
        // pieces [0, j0) (from the end) belong to k_crc_lanes
        const uint64_t j0 = fast_spans(map_base, data, off[r], L) * (kSpanBytes / kPiece);
        uint32_t contrib = 0;
        if ((uint64_t)blockIdx.x * kCrcThreads >= npieces) continue;                 // uniform per block
        if ((uint64_t)blockIdx.x * kCrcThreads + kCrcThreads <= j0) continue;        // uniform per block
        if (j < npieces && j >= j0) {
            const uint8_t* rbeg = data + off[r];
            const uint8_t* pend = rbeg + L - j * kPiece;  // one past the piece
            const uint8_t* pbeg = pend - kPiece;          // may precede rbeg (first piece)
            // 4-byte aligned word stream, funnel-shifted by the byte offset
            const uintptr_t a0 = reinterpret_cast<uintptr_t>(pbeg) & ~(uintptr_t)3;
            const uint32_t sh = 8u * (uint32_t)(reinterpret_cast<uintptr_t>(pbeg) & 3);
            const uintptr_t lo_ok = reinterpret_cast<uintptr_t>(rbeg);
            const uintptr_t hi_ok = lo_ok + L;
            auto ldw = [&](uintptr_t a) -> uint32_t {  // bytes before the range read as zero
                if (a >= lo_ok && a + 4 <= hi_ok) return *reinterpret_cast<const uint32_t*>(a);
                if (a >= hi_ok) return 0u;  // past the range: never read (buffers may lack slack)
                if (a + 4 <= lo_ok) return 0u;
                uint32_t v = 0;
                for (int k = 0; k < 4; ++k)
                    if (a + k >= lo_ok && a + k < hi_ok)
                        v |= (uint32_t)(*reinterpret_cast<const uint8_t*>(a + k)) << (8 * k);
                return v;
            };
            uint32_t c = 0;
            uint32_t prev = ldw(a0);
            for (int q = 0; q < (int)(kPiece / 16); ++q) {
                const uintptr_t a = a0 + 16u * q;
                const uint32_t n0 = ldw(a + 4), n1 = ldw(a + 8), n2 = ldw(a + 12), n3 = ldw(a + 16);
                const uint32_t w0 = __funnelshift_r(prev, n0, sh), w1 = __funnelshift_r(n0, n1, sh);
                const uint32_t w2 = __funnelshift_r(n1, n2, sh), w3 = __funnelshift_r(n2, n3, sh);
                prev = n3;
                {
                    uint32_t lo = c ^ w0, hi = w1;
                    c = T[7][lo & 0xFF] ^ T[6][(lo >> 8) & 0xFF] ^ T[5][(lo >> 16) & 0xFF] ^ T[4][lo >> 24] ^
                        T[3][hi & 0xFF] ^ T[2][(hi >> 8) & 0xFF] ^ T[1][(hi >> 16) & 0xFF] ^ T[0][hi >> 24];
                }
                {
                    uint32_t lo = c ^ w2, hi = w3;
                    c = T[7][lo & 0xFF] ^ T[6][(lo >> 8) & 0xFF] ^ T[5][(lo >> 16) & 0xFF] ^ T[4][lo >> 24] ^
                        T[3][hi & 0xFF] ^ T[2][(hi >> 8) & 0xFF] ^ T[1][(hi >> 16) & 0xFF] ^ T[0][hi >> 24];
                }
            }
            contrib = c ? multmodp(pow_for(j), c) : 0u;
        }
#pragma unroll
        for (int d = 16; d; d >>= 1) contrib ^= __shfl_xor_sync(0xffffffffu, contrib, d);
        if ((threadIdx.x & 31) == 0 && contrib) atomicXor(&acc[r], contrib);
    }
}

__global__ void __launch_bounds__(kLaneWarps * 32, 1) k_crc_lanes(const __grid_constant__ CUtensorMap tmap,
                                                                   uint64_t map_base, const uint8_t* __restrict__ data,
                                                                   const uint64_t* __restrict__ off,
                                                                   const uint64_t* __restrict__ len, int64_t n,
                                                                   int64_t spans_max, uint32_t* __restrict__ acc) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);  // SW128 atoms: 1 KB aligned
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint8_t* ring = smem + kTabBytes + kShiftBytes + (size_t)warp * kRingSlots * kRoundBytes;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + kTabBytes + kShiftBytes +
                                                (size_t)kLaneWarps * kRingSlots * kRoundBytes) + warp * kRingSlots;
    // tables: entry i of table k, lane copy l at word (k * 256 + i) * 32 + l
    uint32_t* tab = reinterpret_cast<uint32_t*>(smem);
    for (uint32_t w = threadIdx.x; w < 4 * 256 * 32; w += blockDim.x) tab[w] = (&g_crc_t4[0][0])[w >> 5];
    uint32_t* gap = reinterpret_cast<uint32_t*>(smem + kTabBytes);
    for (uint32_t w = threadIdx.x; w < 4 * 256; w += blockDim.x) gap[w] = (&g_crc_gap[0][0])[w];
    if (lane == 0)
        for (uint32_t k = 0; k < kRingSlots; ++k) mbar_init(&bar[k], 1);
    fence_mbar_init();
    __syncthreads();
    const uint32_t tbase = smem_u32(tab) + 4u * lane;
    const uint32_t gbase = smem_u32(gap);
    // lane l: row l >> 1 of the round, 16-B units (l & 1) * 4 + v, stored at unit ^ (row & 7)
    const uint32_t row = (uint32_t)lane >> 1;
    uint32_t uoff[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) uoff[v] = row * 128u + ((((uint32_t)(lane & 1) * 4u + v) ^ (row & 7u)) << 4);
    const uint32_t lpow = g_crc_lanepow[lane];

    const int64_t total = n * spans_max;
    const int64_t wstride = (int64_t)gridDim.x * kLaneWarps;
    auto span_row = [&](int64_t t, int32_t& r0) -> bool {  // first map row of task t's span
        const int64_t r = t / spans_max, sp = t - r * spans_max;
        const uint64_t L = len[r];
        if ((uint64_t)sp >= fast_spans(map_base, data, off[r], L)) return false;
        const uint64_t start = reinterpret_cast<uint64_t>(data) + off[r] + L - (uint64_t)(sp + 1) * kSpanBytes;
        r0 = (int32_t)((start - map_base) >> 7);
        return true;
    };
    // issue cursor (task it, round iq) runs kRingSlots - 1 rounds ahead of the consumer
    int64_t it = (int64_t)blockIdx.x * kLaneWarps + warp;
    int32_t i_row = 0;
    while (it < total && !span_row(it, i_row)) it += wstride;
    uint32_t iq = 0;
    uint64_t gq_issue = 0, gq = 0;
    auto issue = [&]() {
        if (it >= total) return;
        const uint32_t slot = (uint32_t)(gq_issue % kRingSlots);
        if (lane == 0) {
            fence_proxy_async_smem();
            mbar_arrive_expect_tx(&bar[slot], kRoundBytes);
            tma_load_2d(ring + slot * kRoundBytes, &tmap, 0, i_row + (int32_t)(iq * (kRoundBytes / 128)), &bar[slot]);
#if DC_CRC_L2PF
            // pull the next DC_CRC_L2PF rounds of this span into L2 so their
            // (serialised, one-slot) TMA loads hit L2 instead of HBM
            if (iq + DC_CRC_L2PF < kRounds) {
                const uint64_t nxt = map_base + ((uint64_t)(i_row + (int32_t)((iq + DC_CRC_L2PF) * (kRoundBytes / 128))) << 7);
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nxt), "r"(kRoundBytes) : "memory");
            }
#endif
        }
        ++gq_issue;
        if (++iq == kRounds) {
            iq = 0;
            do it += wstride;
            while (it < total && !span_row(it, i_row));
        }
    };
    for (uint32_t k = 0; k + 1 < kRingSlots; ++k) issue();
    int64_t t = (int64_t)blockIdx.x * kLaneWarps + warp;
    int32_t dummy;
    while (t < total && !span_row(t, dummy)) t += wstride;
    for (; t < total;) {
        uint32_t c = 0;
        for (uint32_t q = 0; q < kRounds; ++q, ++gq) {
            __syncwarp();  // every lane is done with the slot the next copy overwrites
            issue();
            const uint32_t slot = (uint32_t)(gq % kRingSlots);
            mbar_wait(&bar[slot], (uint32_t)(gq / kRingSlots) & 1u);
            const uint32_t sb = smem_u32(ring + slot * kRoundBytes);
            if (q) {  // skip the 1984 bytes between this lane's blocks
                uint32_t s0, s1, s2, s3;
                asm volatile(
                    "{\n\t.reg .u32 b0, b1, b2, b3;\n\t"
                    "prmt.b32 b0, %4, 0, 0x4440;\n\t"
                    "prmt.b32 b1, %4, 0, 0x4441;\n\t"
                    "prmt.b32 b2, %4, 0, 0x4442;\n\t"
                    "shr.u32 b3, %4, 24;\n\t"
                    "mad.lo.u32 b0, b0, 4, %5;\n\t"
                    "mad.lo.u32 b1, b1, 4, %5;\n\t"
                    "mad.lo.u32 b2, b2, 4, %5;\n\t"
                    "mad.lo.u32 b3, b3, 4, %5;\n\t"
                    "ld.shared.u32 %0, [b0];\n\t"
                    "ld.shared.u32 %1, [b1+1024];\n\t"
                    "ld.shared.u32 %2, [b2+2048];\n\t"
                    "ld.shared.u32 %3, [b3+3072];\n\t}"
                    : "=r"(s0), "=r"(s1), "=r"(s2), "=r"(s3)
                    : "r"(c), "r"(gbase));
                c = s0 ^ s1 ^ s2 ^ s3;
            }
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                uint32_t wv[4];
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(wv[0]), "=r"(wv[1]), "=r"(wv[2]), "=r"(wv[3])
                             : "r"(sb + uoff[v]));
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    // byte b of x (PRMT, zero-extended) * 128 + lane base (IMAD, FMA pipe)
                    const uint32_t x = c ^ wv[k];
                    uint32_t t0, t1, t2, t3;
                    asm volatile(
                        "{\n\t.reg .u32 b0, b1, b2, b3;\n\t"
                        "prmt.b32 b0, %4, 0, 0x4440;\n\t"
                        "prmt.b32 b1, %4, 0, 0x4441;\n\t"
                        "prmt.b32 b2, %4, 0, 0x4442;\n\t"
                        "shr.u32 b3, %4, 24;\n\t"
                        "mad.lo.u32 b0, b0, 128, %5;\n\t"
                        "mad.lo.u32 b1, b1, 128, %5;\n\t"
                        "mad.lo.u32 b2, b2, 128, %5;\n\t"
                        "mad.lo.u32 b3, b3, 128, %5;\n\t"
                        "ld.shared.u32 %0, [b0+98304];\n\t"
                        "ld.shared.u32 %1, [b1+65536];\n\t"
                        "ld.shared.u32 %2, [b2+32768];\n\t"
                        "ld.shared.u32 %3, [b3];\n\t}"
                        : "=r"(t0), "=r"(t1), "=r"(t2), "=r"(t3)
                        : "r"(x), "r"(tbase));
                    c = t0 ^ t1 ^ t2 ^ t3;
                }
            }
        }
        const int64_t r = t / spans_max, sp = t - r * spans_max;
        // distance from this lane's last block end to the range end: 64 (31 - l) + 64 KB * sp
        uint32_t contrib = c ? multmodp(pow_for((uint64_t)sp * (kSpanBytes / kPiece)), multmodp(lpow, c)) : 0u;
#pragma unroll
        for (int d = 16; d; d >>= 1) contrib ^= __shfl_xor_sync(0xffffffffu, contrib, d);
        if (lane == 0 && contrib) atomicXor(&acc[r], contrib);
        do t += wstride;
        while (t < total && !span_row(t, dummy));
    }
}

__global__ void k_crc_finalize(const uint64_t* __restrict__ len, int64_t n, uint32_t* __restrict__ acc,
                               uint32_t* __restrict__ crc_out) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint32_t aff = multmodp(x2nmodp_dev(len[r], 3), 0xFFFFFFFFu) ^ 0xFFFFFFFFu;
    crc_out[r] = acc[r] ^ aff;
}

static bool g_crc_ready = false;

static int crc_init(cudaStream_t st) {
    if (g_crc_ready) return DC_OK;
    uint32_t x2n[64];
    uint32_t p = 1u << 30;  // x^1
    for (int k = 0; k < 64; ++k) {
        x2n[k] = p;
        p = multmodp(p, p);
    }
    cudaError_t e = cudaMemcpyToSymbolAsync(c_x2n, x2n, sizeof(x2n), 0, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) {
        set_error("crc init", e);
        return DC_ERR_CUDA;
    }
    uint32_t t4[4][256];
    for (uint32_t i = 0; i < 256; ++i) {
        uint32_t c = i;
        for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
        t4[0][i] = c;
    }
    for (uint32_t i = 0; i < 256; ++i)
        for (int t = 1; t < 4; ++t) t4[t][i] = (t4[t - 1][i] >> 8) ^ t4[0][t4[t - 1][i] & 0xFF];
    e = cudaMemcpyToSymbolAsync(g_crc_t4, t4, sizeof(t4), 0, cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) {
        set_error("crc init", e);
        return DC_ERR_CUDA;
    }
    auto x2nmodp_host = [&](uint64_t nn, unsigned k) {  // x^(nn * 2^k) mod G
        uint32_t q = 1u << 31;
        while (nn) {
            if (nn & 1) q = multmodp(x2n[k & 63], q);
            nn >>= 1;
            ++k;
        }
        return q;
    };
    static uint32_t gap[4][256], lanepow[32];
    const uint32_t pg = x2nmodp_host(kRoundBytes - 64, 3);
    for (int k = 0; k < 4; ++k)
        for (uint32_t i = 0; i < 256; ++i) gap[k][i] = multmodp(pg, i << (8 * k));
    for (int l = 0; l < 32; ++l) lanepow[l] = x2nmodp_host(64ull * (31 - l), 3);
    if ((e = cudaMemcpyToSymbolAsync(g_crc_gap, gap, sizeof(gap), 0, cudaMemcpyHostToDevice, st)) != cudaSuccess ||
        (e = cudaMemcpyToSymbolAsync(g_crc_lanepow, lanepow, sizeof(lanepow), 0, cudaMemcpyHostToDevice, st)) !=
            cudaSuccess) {
        set_error("crc init", e);
        return DC_ERR_CUDA;
    }
    if ((e = cudaFuncSetAttribute(k_crc_lanes, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLaneSmem)) !=
        cudaSuccess) {
        set_error("crc lanes smem", e);
        return DC_ERR_CUDA;
    }
    k_init_pows<<<kPowLo / 256, 256, 0, st>>>();
    DC_CHECK_LAUNCH("k_init_pows");
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
        set_error("crc init sync", e);
        return DC_ERR_CUDA;
    }
    g_crc_ready = true;
    return DC_OK;
}

}  // namespace dc

using namespace dc;

// crc_out doubles as the XOR accumulator until finalize.
extern "C" int dc_crc32_ranges(const uint8_t* data, uint64_t data_bytes, const uint64_t* off, const uint64_t* len,
                               int64_t n, uint64_t max_len, uint32_t* crc_out, void* stream) {
    if (n < 0) return DC_ERR_ARG;
    if (n == 0) return DC_OK;
    cudaStream_t st = (cudaStream_t)stream;
    int rc = crc_init(st);
    if (rc) return rc;
    cudaError_t e = cudaMemsetAsync(crc_out, 0, (size_t)n * sizeof(uint32_t), st);
    if (e != cudaSuccess) {
        set_error("crc memset", e);
        return DC_ERR_CUDA;
    }
    // the bulk: whole 64 KB spans of ranges with a row-aligned end, through a
    // 2-D (rows of 128 B) view of the buffer
    uint64_t map_base = 0;
    const int64_t spans_max = (int64_t)(max_len / kSpanBytes);
    CUtensorMap tmap;
    if (data_bytes && spans_max > 0) {
        const uint64_t b = reinterpret_cast<uint64_t>(data) & ~(uint64_t)127;
        const uint64_t rows = (reinterpret_cast<uint64_t>(data) + data_bytes - b + 127) / 128;
        if (make_tmap_i8(&tmap, reinterpret_cast<const void*>(b), rows, 128, kRoundBytes / 128) == DC_OK) map_base = b;
    }
    if (map_base) {
        const int64_t tasks = n * spans_max;
        const int64_t per = (int64_t)sm_count() * kLaneWarps;
        const int64_t grid = tasks < per ? (tasks + kLaneWarps - 1) / kLaneWarps : sm_count();
        k_crc_lanes<<<(unsigned)grid, kLaneWarps * 32, kLaneSmem, st>>>(tmap, map_base, data, off, len, n, spans_max,
                                                                        crc_out);
        DC_CHECK_LAUNCH("k_crc_lanes");
    }
    const uint64_t pieces = (max_len + kPiece - 1) / kPiece;
    const uint64_t gx = pieces ? (pieces + kCrcThreads - 1) / kCrcThreads : 1;
    dim3 grid((unsigned)gx, (unsigned)(n < 65535 ? n : 65535));
    k_crc_pieces<<<grid, kCrcThreads, 0, st>>>(map_base, data, off, len, n, crc_out);
    DC_CHECK_LAUNCH("k_crc_pieces");
    k_crc_finalize<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(len, n, crc_out, crc_out);
    DC_CHECK_LAUNCH("k_crc_finalize");
    return DC_OK;
}
