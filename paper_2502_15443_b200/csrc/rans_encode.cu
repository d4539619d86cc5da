// rANS encoding of DCC1 chunks on B200 (sm_100a): bit-exact with the
// reference's container.pack -> ans.compress_blob (ans.py:213-330).
//
//   k_hist       per-chunk 256-bin histograms (warp-private smem bins)
//   k_normalize  one warp per chunk replays _normalize (ans.py:213-243)
//                exactly: floor allocation, largest-remainder top-up in
//                (remainder desc, symbol asc) order, argmax repayment; then
//                packs the 384-byte u12 wire table (ans.py:246-253)
//   k_encode     one lane per chunk runs the reverse encoder (ans.py:55-68)
//                with exact reciprocal division; per-lane symbol tables live
//                in bank-private shared memory (lane l only touches bank l)
//   k_assemble   scatters table | state | stream (or raw) into the file image
#include "common.cuh"

namespace dc {

// ------------------------------------------------------------------ hist
constexpr int kHistThreads = 256;
constexpr uint32_t kHistSlice = 64 * 1024;

__global__ void __launch_bounds__(kHistThreads) k_hist(const uint8_t* __restrict__ data, uint64_t total,
                                                        uint64_t chunk_size, int64_t n_chunks,
                                                        uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[kHistThreads / 32][256];
    const int warp = threadIdx.x >> 5;
    for (int64_t c = blockIdx.y; c < n_chunks; c += gridDim.y) {
    __syncthreads();
    for (int i = threadIdx.x; i < (kHistThreads / 32) * 256; i += blockDim.x) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint64_t cbeg = c * chunk_size;
    uint64_t cend = cbeg + chunk_size;
    if (cend > total) cend = total;
    const uint64_t beg = cbeg + (uint64_t)blockIdx.x * kHistSlice;
    if (beg < cend) {
        uint64_t end = beg + kHistSlice;
        if (end > cend) end = cend;
        const uint64_t abeg = (beg + 15) & ~(uint64_t)15;
        const uint64_t aend = end & ~(uint64_t)15;
        uint32_t* hw = h[warp];
        if (abeg >= aend) {
            for (uint64_t i = beg + threadIdx.x; i < end; i += blockDim.x) atomicAdd(&hw[data[i]], 1u);
        } else {
            for (uint64_t i = beg + threadIdx.x; i < abeg; i += blockDim.x) atomicAdd(&hw[data[i]], 1u);
            for (uint64_t i = aend + threadIdx.x; i < end; i += blockDim.x) atomicAdd(&hw[data[i]], 1u);
            for (uint64_t v = abeg + (uint64_t)threadIdx.x * 16; v < aend; v += (uint64_t)blockDim.x * 16) {
                const uint4 q = *reinterpret_cast<const uint4*>(data + v);
                const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    atomicAdd(&hw[w[k] & 0xFF], 1u);
                    atomicAdd(&hw[(w[k] >> 8) & 0xFF], 1u);
                    atomicAdd(&hw[(w[k] >> 16) & 0xFF], 1u);
                    atomicAdd(&hw[w[k] >> 24], 1u);
                }
            }
        }
    }
    __syncthreads();
    for (int s = threadIdx.x; s < 256; s += blockDim.x) {
        uint32_t t = 0;
#pragma unroll
        for (int w = 0; w < kHistThreads / 32; ++w) t += h[w][s];
        if (t) atomicAdd(&hist[c * 256 + s], t);
    }
    }
}

// ------------------------------------------------------------- normalize
__global__ void k_normalize(const uint32_t* __restrict__ hist, int64_t n_chunks, uint32_t* __restrict__ freq_out,
                            uint8_t* __restrict__ tbytes) {
    __shared__ int64_t s_rem[8][256];
    const int wib = threadIdx.x >> 5;
    const int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
    const int lane = threadIdx.x & 31;
    if (c >= n_chunks) return;
    const uint32_t* h = hist + c * 256;
    // lane owns symbols lane*8 .. lane*8+7
    uint64_t hv[8];
    uint64_t n = 0;
    int present = 0, last = -1;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        hv[k] = h[lane * 8 + k];
        n += hv[k];
        if (hv[k]) {
            ++present;
            last = lane * 8 + k;
        }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        n += __shfl_xor_sync(0xffffffffu, n, d);
        present += __shfl_xor_sync(0xffffffffu, present, d);
        last = max(last, __shfl_xor_sync(0xffffffffu, last, d));
    }
    int64_t alloc[8];
    if (present <= 1) {  // ans.py:222-224 (present == 0 cannot come from a chunk)
#pragma unroll
        for (int k = 0; k < 8; ++k) alloc[k] = (lane * 8 + k == last) ? (int64_t)kProbScale : 0;
    } else {
        int64_t sum = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint64_t scaled = hv[k] * kProbScale;  // ans.py:225
            const int64_t a = (int64_t)(scaled / n);
            alloc[k] = hv[k] ? (a < 1 ? 1 : a) : 0;   // ans.py:226
            s_rem[wib][lane * 8 + k] = hv[k] ? (int64_t)(scaled % n) : -1;
            sum += alloc[k];
        }
#pragma unroll
        for (int d = 16; d; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
        int64_t deficit = (int64_t)kProbScale - sum;  // ans.py:227
        __syncwarp();
        if (deficit > 0) {
            // ans.py:228-235: present symbols in (remainder desc, symbol asc)
            // order receive +1 until the deficit is paid: rank < deficit.
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int s = lane * 8 + k;
                if (!hv[k]) continue;
                const int64_t r = s_rem[wib][s];
                int rank = 0;
                for (int t = 0; t < 256; ++t) {
                    const int64_t rt = s_rem[wib][t];
                    rank += (rt > r) || (rt == r && t < s);  // absent symbols carry -1: never ahead
                }
                if (rank < deficit) alloc[k] += 1;
            }
        }
        while (deficit < 0) {  // ans.py:236-240: decrement the first argmax
            int64_t best = -1;
            int bs = 256;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (alloc[k] > best) {
                    best = alloc[k];
                    bs = lane * 8 + k;
                }
#pragma unroll
            for (int d = 16; d; d >>= 1) {
                const int64_t ob = __shfl_xor_sync(0xffffffffu, best, d);
                const int os = __shfl_xor_sync(0xffffffffu, bs, d);
                if (ob > best || (ob == best && os < bs)) {
                    best = ob;
                    bs = os;
                }
            }
            if ((bs >> 3) == lane) {
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    if ((bs & 7) == k) alloc[k] -= 1;
            }
            ++deficit;
        }
    }
    uint32_t* f = freq_out + c * 256;
#pragma unroll
    for (int k = 0; k < 8; ++k) f[lane * 8 + k] = (uint32_t)alloc[k];
    // u12 wire table: lane packs pairs 4*lane .. 4*lane+3 (12 bytes)
    uint8_t* tb = tbytes + c * kTableBytes;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        uint32_t a = (uint32_t)alloc[2 * k], b = (uint32_t)alloc[2 * k + 1];
        a = a > 4095 ? 4095 : a;
        b = b > 4095 ? 4095 : b;
        const int i = lane * 4 + k;
        tb[3 * i + 0] = (uint8_t)(a & 0xFF);
        tb[3 * i + 1] = (uint8_t)(((a >> 8) & 0x0F) | ((b & 0x0F) << 4));
        tb[3 * i + 2] = (uint8_t)((b >> 4) & 0xFF);
    }
}

// ----------------------------------------------------------------- encode
// Per-lane symbol table in bank-private layout: word (s*2 + w)*32 + lane.
//   w0 = reciprocal (ryg_rans style exact division for x < 2^31)
//   w1 = f (13 bits) | cum << 13 (12 bits) | shift << 25 (4 bits)
constexpr int kEncLanes = 32;

__global__ void __launch_bounds__(kEncLanes) k_encode(const uint8_t* __restrict__ data, uint64_t total,
                                                       uint64_t chunk_size, int64_t n_chunks,
                                                       const uint8_t* __restrict__ todo,
                                                       const uint32_t* __restrict__ freq, uint8_t* __restrict__ scratch,
                                                       uint32_t* __restrict__ final_state,
                                                       uint64_t* __restrict__ stream_len, uint32_t seg_shift,
                                                       const int64_t* __restrict__ seg_base,
                                                       uint32_t* __restrict__ seg_state,
                                                       uint32_t* __restrict__ seg_emitted, uint32_t flags) {
    extern __shared__ uint32_t etab[];  // 256 * 2 * 32 words = 64 KB
    const int lane = threadIdx.x;
    const int64_t c = (int64_t)blockIdx.x * kEncLanes + lane;
    const bool active = c < n_chunks && todo[c];
    uint64_t beg = 0, len = 0;
    if (active) {
        beg = (uint64_t)c * chunk_size;
        len = total - beg < chunk_size ? total - beg : chunk_size;
        const uint32_t* f = freq + c * 256;
        uint32_t cum = 0;
        for (int s = 0; s < 256; ++s) {
            const uint32_t fs = f[s];
            uint32_t rcp = 0, shift = 0;
            if (fs >= 2) {
                while (fs > (1u << shift)) ++shift;
                rcp = (uint32_t)(((1ull << (shift + 31)) + fs - 1) / fs);
                shift -= 1;
            } else {
                rcp = 0xFFFFFFFFu;  // f == 1: q = x - 1 via mulhi
            }
            etab[(s * 2 + 0) * 32 + lane] = rcp;
            etab[(s * 2 + 1) * 32 + lane] = fs | (cum << 13) | (shift << 25);
            cum += fs;
        }
    }
    if (!active) return;  // no block-level sync below
    const uint8_t* src = data + beg;
    uint8_t* slot_end = scratch + beg + len;  // bytes go backwards from here
    // emitted >= limit -> the chunk will be stored (container.py:165); a
    // standalone blob (flags & 1) is always completed (ans.py:316-330)
    const uint64_t limit = (flags & 1) ? ~0ull : (len > kHeaderBytes ? len - kHeaderBytes : 0);
    const uint32_t K = 1u << seg_shift;
    const int64_t sb = seg_state ? seg_base[c] : 0;
    uint32_t x = kStateLower;
    uint64_t pos = 0;
    bool stored = (limit == 0);
    // walk the chunk backwards in aligned 16-byte blocks
    const uintptr_t a_beg = reinterpret_cast<uintptr_t>(src);
    const uintptr_t a_end = a_beg + len;
    const uintptr_t data_end = reinterpret_cast<uintptr_t>(data) + total;
    uintptr_t blk = (a_end - 1) & ~(uintptr_t)15;
    for (; !stored && blk + 16 > a_beg; blk -= 16) {
        uint4 q;
        if (blk + 16 <= data_end) {
            q = *reinterpret_cast<const uint4*>(blk);
        } else {  // last block of the buffer: never read past its end
            uint8_t b[16];
            for (int k = 0; k < 16; ++k) b[k] = (blk + k < data_end) ? *reinterpret_cast<const uint8_t*>(blk + k) : 0;
            q.x = b[0] | b[1] << 8 | b[2] << 16 | (uint32_t)b[3] << 24;
            q.y = b[4] | b[5] << 8 | b[6] << 16 | (uint32_t)b[7] << 24;
            q.z = b[8] | b[9] << 8 | b[10] << 16 | (uint32_t)b[11] << 24;
            q.w = b[12] | b[13] << 8 | b[14] << 16 | (uint32_t)b[15] << 24;
        }
        const uint32_t wv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int k = 15; k >= 0; --k) {
            const uintptr_t a = blk + k;
            if (a < a_beg || a >= a_end) continue;
            const uint32_t s = (wv[k >> 2] >> (8 * (k & 3))) & 0xFF;
            const uint32_t rcp = etab[(s * 2 + 0) * 32 + lane];
            const uint32_t meta = etab[(s * 2 + 1) * 32 + lane];
            const uint32_t f = meta & 0x1FFF;
            const uint32_t cum = (meta >> 13) & 0xFFF;
            const uint32_t sh = meta >> 25;
            const uint32_t x_max = f << 16;  // ans.py:62
            while (x >= x_max) {             // ans.py:63-66
                *(slot_end - 1 - pos) = (uint8_t)(x & 0xFF);
                ++pos;
                x >>= 8;
            }
            // ans.py:67: x = (x // f) * 4096 + cum + x % f, exact via reciprocal
            const uint32_t qd = __umulhi(x, rcp) >> sh;
            x = x + (f >= 2 ? cum : cum + (kProbScale - 1)) + qd * (f >= 2 ? kProbScale - f : kProbScale - 1);
            const uint64_t i = (uint64_t)(a - a_beg);
            if (seg_state && (i & (K - 1)) == 0) {
                seg_state[sb + (i >> seg_shift)] = x;
                seg_emitted[sb + (i >> seg_shift)] = (uint32_t)pos;
            }
            if (pos >= limit) {  // could not beat raw storage (container.py:165)
                stored = true;
                break;
            }
        }
        if (blk < 16) break;
    }
    final_state[c] = x;
    stream_len[c] = stored ? ~0ull : pos;
}

// --------------------------------------------------------------- assemble
__global__ void k_assemble(const uint8_t* __restrict__ data, uint64_t total, uint64_t chunk_size, int64_t n_chunks,
                           const uint8_t* __restrict__ codec, const uint8_t* __restrict__ tbytes,
                           const uint32_t* __restrict__ final_state, const uint64_t* __restrict__ stream_len,
                           const uint8_t* __restrict__ scratch, const uint64_t* __restrict__ file_off,
                           uint8_t* __restrict__ dst) {
    for (int64_t c = blockIdx.y; c < n_chunks; c += gridDim.y) {
        const uint64_t beg = (uint64_t)c * chunk_size;
        const uint64_t len = total - beg < chunk_size ? total - beg : chunk_size;
        uint8_t* d = dst + file_off[c];
        const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
        const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
        if (codec[c] == 0) {
            for (uint64_t i = tid; i < len; i += stride) d[i] = data[beg + i];
        } else {
            const uint64_t sl = stream_len[c];
            const uint8_t* s = scratch + beg + len - sl;
            const uint32_t x = final_state[c];
            for (uint64_t i = tid; i < kHeaderBytes + sl; i += stride) {
                uint8_t v;
                if (i < kTableBytes)
                    v = tbytes[c * kTableBytes + i];
                else if (i < kHeaderBytes)
                    v = (uint8_t)(x >> (8 * (i - kTableBytes)));
                else
                    v = s[i - kHeaderBytes];
                d[i] = v;
            }
        }
    }
}

}  // namespace dc

using namespace dc;

extern "C" int dc_hist_chunks(const uint8_t* data, uint64_t total, uint64_t chunk_size, int64_t n_chunks,
                              uint32_t* hist, void* stream) {
    if (n_chunks < 0 || chunk_size == 0) return DC_ERR_ARG;
    if (n_chunks == 0) return DC_OK;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemsetAsync(hist, 0, (size_t)n_chunks * 256 * sizeof(uint32_t), st);
    if (e != cudaSuccess) {
        set_error("hist memset", e);
        return DC_ERR_CUDA;
    }
    dim3 grid((unsigned)((chunk_size + kHistSlice - 1) / kHistSlice), (unsigned)(n_chunks < 65535 ? n_chunks : 65535));
    k_hist<<<grid, kHistThreads, 0, st>>>(data, total, chunk_size, n_chunks, hist);
    DC_CHECK_LAUNCH("k_hist");
    return DC_OK;
}

extern "C" int dc_normalize_tables(const uint32_t* hist, int64_t n_chunks, uint32_t* freq, uint8_t* table_bytes,
                                   void* stream) {
    if (n_chunks < 0) return DC_ERR_ARG;
    if (n_chunks == 0) return DC_OK;
    const int warps = 8;
    k_normalize<<<(unsigned)((n_chunks + warps - 1) / warps), warps * 32, 0, (cudaStream_t)stream>>>(
        hist, n_chunks, freq, table_bytes);
    DC_CHECK_LAUNCH("k_normalize");
    return DC_OK;
}

extern "C" int dc_ans_encode_chunks(const uint8_t* data, uint64_t total, uint64_t chunk_size, int64_t n_chunks,
                                    const uint8_t* todo, const uint32_t* freq, uint8_t* scratch,
                                    uint32_t* final_state, uint64_t* stream_len, uint32_t seg_shift,
                                    const int64_t* seg_base, uint32_t* seg_state, uint32_t* seg_emitted,
                                    uint32_t flags, void* stream) {
    if (n_chunks < 0 || chunk_size == 0 || (seg_state && (seg_shift < 4 || seg_shift > 20))) return DC_ERR_ARG;
    if (n_chunks == 0) return DC_OK;
    const int smem = 256 * 2 * 32 * 4;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_encode, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    k_encode<<<(unsigned)((n_chunks + kEncLanes - 1) / kEncLanes), kEncLanes, smem, (cudaStream_t)stream>>>(
        data, total, chunk_size, n_chunks, todo, freq, scratch, final_state, stream_len, seg_shift, seg_base,
        seg_state, seg_emitted, flags);
    DC_CHECK_LAUNCH("k_encode");
    return DC_OK;
}

extern "C" int dc_assemble_payloads(const uint8_t* data, uint64_t total, uint64_t chunk_size, int64_t n_chunks,
                                    const uint8_t* codec, const uint8_t* table_bytes, const uint32_t* final_state,
                                    const uint64_t* stream_len, const uint8_t* scratch, const uint64_t* file_off,
                                    uint8_t* dst, void* stream) {
    if (n_chunks < 0 || chunk_size == 0) return DC_ERR_ARG;
    if (n_chunks == 0) return DC_OK;
    const uint64_t per = chunk_size < 4096 * 64 ? 4 : 64;
    dim3 grid((unsigned)per, (unsigned)(n_chunks < 65535 ? n_chunks : 65535));
    k_assemble<<<grid, 256, 0, (cudaStream_t)stream>>>(data, total, chunk_size, n_chunks, codec, table_bytes,
                                                       final_state, stream_len, scratch, file_off, dst);
    DC_CHECK_LAUNCH("k_assemble");
    return DC_OK;
}
