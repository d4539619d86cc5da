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
#include "common.cuh"

namespace dc {

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

__global__ void __launch_bounds__(kCrcThreads) k_crc_pieces(const uint8_t* __restrict__ data,
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
        uint32_t contrib = 0;
        if ((uint64_t)blockIdx.x * kCrcThreads >= npieces) continue;  // uniform per block
        if (j < npieces) {
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
extern "C" int dc_crc32_ranges(const uint8_t* data, const uint64_t* off, const uint64_t* len, int64_t n,
                                       uint64_t max_len, uint32_t* crc_out, void* stream) {
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
    const uint64_t pieces = (max_len + kPiece - 1) / kPiece;
    const uint64_t gx = pieces ? (pieces + kCrcThreads - 1) / kCrcThreads : 1;
    dim3 grid((unsigned)gx, (unsigned)(n < 65535 ? n : 65535));
    k_crc_pieces<<<grid, kCrcThreads, 0, st>>>(data, off, len, n, crc_out);
    DC_CHECK_LAUNCH("k_crc_pieces");
    k_crc_finalize<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(len, n, crc_out, crc_out);
    DC_CHECK_LAUNCH("k_crc_finalize");
    return DC_OK;
}
