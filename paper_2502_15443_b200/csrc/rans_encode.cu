// rANS encoding of DCC1 chunks on B200 (sm_100a): bit-exact with the
// reference's container.pack -> ans.compress_blob (ans.py:213-330).
//
//   k_hist       per-chunk 256-bin histograms (warp-private smem bins)
//   k_normalize  one warp per chunk replays _normalize (ans.py:213-243)
//                exactly: floor allocation, largest-remainder top-up in
//                (remainder desc, symbol asc) order, argmax repayment; then
//                packs the 384-byte u12 wire table (ans.py:246-253)
//   k_encode     one warp per chunk, one lane runs the reverse encoder
//                (ans.py:55-68) as a branch-free recurrence with exact
//                reciprocal division; the warp builds the chunk's table
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
// Two passes.  The reverse encoder (ans.py:55-68) is a serial recurrence per
// chunk, so pass 1 runs ONLY the state chain -- one chunk per warp, four warps
// per CTA (one per SM sub-partition), every lane running the same branch-free
// step so there is no divergence:
//   p1 = x >= f<<16, p2 = x >= f<<24  (at most two renorm bytes: x < 2^28)
//   xr = x >> 8*(p1+p2)
//   x  = xr + bias + (umulhi(xr, rcp) >> sh) * (4096 - f)
// with ryg_rans-style exact reciprocals (f == 1: rcp = 2^32-1 gives q = xr-1,
// folded into bias = cum + 4095).  It stores each symbol's input state (16-B
// stores per 4 symbols) and the running byte count every 256 symbols.
// Pass 2 (k_encode_emit, fully parallel, one thread per 256 symbols) turns the
// recorded states back into the renormalization bytes at their final stream
// positions: the byte count at each 256-symbol boundary is known from pass 1.
constexpr int kEncWarps = 4;
constexpr int kEmitSeg = 256;  // symbols per pass-2 thread (= pass-1 record cadence)

struct __align__(16) EncEnt {
    uint32_t rcp, xm1, xm2, sh;  // xm1 = f << 16; xm2 = f << 24 or 2^32-1 when f >= 16
    uint32_t bias, gmul, sh8, sh16;  // gmul = 4096 - f; sh8 = sh + 8, sh16 = sh + 16
};


// One reverse-encode step.  q = floor(x / (f << 8n)) = mulhi(x, rcp) >> (sh + 8n)
// -- the same reciprocal for every renorm count n (nested floor division), so
// the IMAD.HI starts from x itself in parallel with the renorm test -- and
// x' = (x >> 8n) + cum + q * (4096 - f).  The shift sh + 8n is picked from
// per-symbol copies (sh, sh + 8, sh + 16) by the renorm predicates (two SELs,
// no add on the path): critical path max(IMAD.HI, ISETP -> SEL -> SEL) -> SHF
// -> IMAD (595 -> 538 ms for the OPT-1.3B chains vs forming n8 then sh + n8).
// f == 1: x >= 2^20 > xm1 = 2^16 always renormalizes (8n >= 8), so rcp = 2^31
// with sh = -1 gives q = (x >> 1) >> (8n - 1) = x >> 8n exactly.
__device__ __forceinline__ void enc_step(uint32_t& x, uint32_t& pos, const uint4& a, const uint4& b) {
    asm volatile(
        "{\n\t.reg .pred p1, p2;\n\t.reg .u32 q, n8, s, xr, n1;\n\t"
        "mul.hi.u32 q, %0, %2;\n\t"
        "setp.ge.u32 p1, %0, %3;\n\t"
        "setp.ge.u32 p2, %0, %4;\n\t"
        "selp.u32 s, %8, %5, p1;\n\t"
        "selp.u32 s, %9, s, p2;\n\t"
        "selp.u32 n8, 8, 0, p1;\n\t"
        "selp.u32 n8, 16, n8, p2;\n\t"
        "shr.u32 q, q, s;\n\t"
        "shr.u32 xr, %0, n8;\n\t"
        "add.u32 xr, xr, %6;\n\t"
        "shr.u32 n1, n8, 3;\n\t"
        "add.u32 %1, %1, n1;\n\t"
        "mad.lo.u32 %0, q, %7, xr;\n\t}"
        : "+r"(x), "+r"(pos)
        : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w));
}

// the encoder's per-symbol table for chunk c (called by one warp)
__device__ __forceinline__ void build_enc_table(const uint32_t* __restrict__ freq, int64_t c, EncEnt* T, int lane) {
    uint32_t fs[8], loc = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        fs[k] = freq[c * 256 + lane * 8 + k];
        loc += fs[k];
    }
    uint32_t inc = loc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    uint32_t cum = inc - loc;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t f = fs[k];
        EncEnt e;
        e.sh = 0;
        if (f >= 2) {
            uint32_t shift = 0;
            while (f > (1u << shift)) ++shift;
            e.rcp = (uint32_t)(((1ull << (shift + 31)) + f - 1) / f);
            e.sh = shift - 1;
        } else {  // f == 1 (see enc_step)
            e.rcp = 0x80000000u;
            e.sh = 0xFFFFFFFFu;
        }
        e.xm1 = f << 16;
        e.xm2 = f < 16 ? f << 24 : 0xFFFFFFFFu;
        e.bias = cum;
        e.gmul = kProbScale - f;
        e.sh8 = e.sh + 8u;  // shift amounts for one / two renorm bytes (enc_step)
        e.sh16 = e.sh + 16u;
        T[lane * 8 + k] = e;
        cum += f;
    }
}

__global__ void __launch_bounds__(kEncWarps * 32) k_encode(const uint8_t* __restrict__ data, uint64_t total,
                                                            uint64_t chunk_size, int64_t n_chunks,
                                                            const uint8_t* __restrict__ todo,
                                                            const uint32_t* __restrict__ freq,
                                                            uint32_t* __restrict__ final_state,
                                                            uint64_t* __restrict__ stream_len, uint32_t seg_shift,
                                                            const int64_t* __restrict__ seg_base,
                                                            uint32_t* __restrict__ seg_state,
                                                            uint32_t* __restrict__ seg_emitted, uint32_t flags,
                                                            uint32_t* __restrict__ xs, uint32_t* __restrict__ rec,
                                                            int64_t rec_per_chunk) {
    __shared__ EncEnt tabs[kEncWarps][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c = (int64_t)blockIdx.x * kEncWarps + warp;
    if (c >= n_chunks || !todo[c]) return;  // whole warp; no block-level sync below
    const uint64_t beg = (uint64_t)c * chunk_size;
    const uint64_t len = total - beg < chunk_size ? total - beg : chunk_size;
    EncEnt* T = tabs[warp];
    build_enc_table(freq, c, T, lane);
    __syncwarp();

    const uint8_t* src = data + beg;
    uint32_t* xsc = xs + beg;             // input state of every symbol
    uint32_t* rc = rec + c * rec_per_chunk;  // bytes emitted after symbol 256*k
    // emitted >= limit -> the chunk will be stored (container.py:165); a
    // standalone blob (flags & 1) is always completed (ans.py:316-330)
    const uint64_t limit = (flags & 1) ? ~0ull : (len > kHeaderBytes ? len - kHeaderBytes : 0);
    const uint32_t K = 1u << seg_shift;
    const int64_t sb = seg_state ? seg_base[c] : 0;
    const bool lead = lane == 0;
    uint32_t x = kStateLower, pos = 0;
    bool stored = (limit == 0);
    auto record = [&](uint64_t i) {  // after encoding symbol i
        if (!lead) return;
        if ((i & (kEmitSeg - 1)) == 0) rc[i / kEmitSeg] = pos;
        if (seg_state && (i & (K - 1)) == 0) {
            seg_state[sb + (i >> seg_shift)] = x;
            seg_emitted[sb + (i >> seg_shift)] = pos;
        }
    };
    const uint64_t nblk = len >> 4;  // whole 16-symbol blocks [0, 16*nblk)
    // tail symbols [16*nblk, len), last to first
    for (uint64_t i = len; !stored && i > nblk * 16;) {
        --i;
        const uint32_t sy = src[i];
        const uint4 ea = *reinterpret_cast<const uint4*>(&T[sy].rcp);
        const uint4 eb = *reinterpret_cast<const uint4*>(&T[sy].bias);
        if (lead) xsc[i] = x;
        enc_step(x, pos, ea, eb);
        record(i);
        if (pos >= limit) stored = true;
    }
    const bool al16 = (reinterpret_cast<uintptr_t>(src) & 15) == 0;
    const bool xal = (reinterpret_cast<uintptr_t>(xsc) & 15) == 0;
    auto load_blk = [&](uint64_t b) -> uint4 {
        if (al16) return __ldg(reinterpret_cast<const uint4*>(src + 16 * b));
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            w[k] = src[16 * b + 4 * k] | (uint32_t)src[16 * b + 4 * k + 1] << 8 |
                   (uint32_t)src[16 * b + 4 * k + 2] << 16 | (uint32_t)src[16 * b + 4 * k + 3] << 24;
        return make_uint4(w[0], w[1], w[2], w[3]);
    };
    uint4 nxt = (!stored && nblk) ? load_blk(nblk - 1) : make_uint4(0, 0, 0, 0);
    for (uint64_t b = nblk; !stored && b > 0;) {
        --b;
        const uint4 cur = nxt;
        if (b) nxt = load_blk(b - 1);  // prefetch the next (lower) block
        const uint32_t wv[4] = {cur.x, cur.y, cur.z, cur.w};
        // table entries of the whole block first (they do not depend on x), then the chain
        uint4 ea[16];
        uint4 eb[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const uint32_t sy = (wv[k >> 2] >> (8 * (k & 3))) & 0xFF;
            ea[k] = *reinterpret_cast<const uint4*>(&T[sy].rcp);
            eb[k] = *reinterpret_cast<const uint4*>(&T[sy].bias);
        }
        uint32_t xin[16];
#pragma unroll
        for (int k = 15; k >= 0; --k) {
            xin[k] = x;
            enc_step(x, pos, ea[k], eb[k]);
        }
        if (lead) {
            uint32_t* dst = xsc + 16 * b;
            if (xal) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    reinterpret_cast<uint4*>(dst)[k] = make_uint4(xin[4 * k], xin[4 * k + 1], xin[4 * k + 2], xin[4 * k + 3]);
            } else {
#pragma unroll
                for (int k = 0; k < 16; ++k) dst[k] = xin[k];
            }
        }
        record(16 * b);  // split points sit at multiples of K >= 16: only at k == 0
        if (pos >= limit) stored = true;  // could not beat raw storage (container.py:165)
    }
    if (lead) {
        final_state[c] = x;
        stream_len[c] = stored ? ~0ull : pos;
    }
}

// Pass 2: one thread per 256 symbols of an encoded chunk.  Replays the
// renormalization test on the recorded input states and writes the bytes
// backwards from the chunk's slot end (stream order reversed at assembly).
__global__ void __launch_bounds__(256) k_encode_emit(const uint8_t* __restrict__ data, uint64_t total,
                                                     uint64_t chunk_size, int64_t n_chunks,
                                                     const uint8_t* __restrict__ todo,
                                                     const uint32_t* __restrict__ freq,
                                                     const uint64_t* __restrict__ stream_len,
                                                     const uint32_t* __restrict__ xs, const uint32_t* __restrict__ rec,
                                                     int64_t rec_per_chunk, uint8_t* __restrict__ scratch) {
    __shared__ uint32_t xm[256][2];
    for (int64_t c = blockIdx.y; c < n_chunks; c += gridDim.y) {
        if (!todo[c] || stream_len[c] == ~0ull) continue;  // uniform per CTA
        __syncthreads();  // previous chunk's table readers are done
        for (int s = threadIdx.x; s < 256; s += blockDim.x) {
            const uint32_t f = freq[c * 256 + s];
            xm[s][0] = f << 16;
            xm[s][1] = f < 16 ? f << 24 : 0xFFFFFFFFu;
        }
        __syncthreads();
        const uint64_t beg = (uint64_t)c * chunk_size;
        const uint64_t len = total - beg < chunk_size ? total - beg : chunk_size;
        const uint64_t nseg = (len + kEmitSeg - 1) / kEmitSeg;
        const uint8_t* src = data + beg;
        const uint32_t* xsc = xs + beg;
        uint8_t* out_end = scratch + beg + len;
        for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < nseg;
             g += (uint64_t)gridDim.x * blockDim.x) {
            const uint64_t lo = g * kEmitSeg, hi = (g + 1) * kEmitSeg < len ? (g + 1) * kEmitSeg : len;
            uint32_t pos = hi < len ? rec[c * rec_per_chunk + hi / kEmitSeg] : 0u;  // bytes emitted before symbol hi-1
            for (uint64_t i = hi; i > lo;) {
                --i;
                const uint32_t x = xsc[i];
                const uint32_t sy = src[i];
                if (x >= xm[sy][0]) {
                    *(out_end - 1 - pos) = (uint8_t)x;
                    ++pos;
                    if (x >= xm[sy][1]) {
                        *(out_end - 1 - pos) = (uint8_t)(x >> 8);
                        ++pos;
                    }
                }
            }
        }
    }
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

extern "C" int dc_ans_encode_work_bytes(uint64_t total, uint64_t chunk_size, int64_t n_chunks, uint64_t* out) {
    if (!out || chunk_size == 0 || n_chunks < 0) return DC_ERR_ARG;
    const uint64_t per = (chunk_size + kEmitSeg - 1) / kEmitSeg + 1;
    *out = 4 * total + 16 + 4 * per * (uint64_t)n_chunks + 256;
    return DC_OK;
}

extern "C" int dc_ans_encode_chunks(const uint8_t* data, uint64_t total, uint64_t chunk_size, int64_t n_chunks,
                                    const uint8_t* todo, const uint32_t* freq, uint8_t* scratch,
                                    uint32_t* final_state, uint64_t* stream_len, uint32_t seg_shift,
                                    const int64_t* seg_base, uint32_t* seg_state, uint32_t* seg_emitted,
                                    uint32_t flags, void* work, uint64_t work_bytes, void* stream) {
    if (n_chunks < 0 || chunk_size == 0 || (seg_state && (seg_shift < 4 || seg_shift > 20))) return DC_ERR_ARG;
    if (n_chunks == 0) return DC_OK;
    uint64_t need = 0;
    dc_ans_encode_work_bytes(total, chunk_size, n_chunks, &need);
    if (!work || work_bytes < need) return DC_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    uintptr_t w = (reinterpret_cast<uintptr_t>(work) + 15) & ~(uintptr_t)15;
    uint32_t* xs = reinterpret_cast<uint32_t*>(w);
    uint32_t* rec = reinterpret_cast<uint32_t*>(w + ((4 * total + 15) & ~(uint64_t)15));
    const int64_t rec_per = (int64_t)((chunk_size + kEmitSeg - 1) / kEmitSeg + 1);
    k_encode<<<(unsigned)((n_chunks + kEncWarps - 1) / kEncWarps), kEncWarps * 32, 0, st>>>(
        data, total, chunk_size, n_chunks, todo, freq, final_state, stream_len, seg_shift, seg_base, seg_state,
        seg_emitted, flags, xs, rec, rec_per);
    DC_CHECK_LAUNCH("k_encode");
    if (flags & 2) return DC_OK;  // lengths only: no stream bytes needed
    const uint64_t nseg = (chunk_size + kEmitSeg - 1) / kEmitSeg;
    const unsigned gx = (unsigned)((nseg + 255) / 256 < 64 ? (nseg + 255) / 256 : 64);
    dim3 grid(gx, (unsigned)(n_chunks < 65535 ? n_chunks : 65535));
    k_encode_emit<<<grid, 256, 0, st>>>(data, total, chunk_size, n_chunks, todo, freq, stream_len, xs, rec, rec_per,
                                        scratch);
    DC_CHECK_LAUNCH("k_encode_emit");
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
