// Activation-aware magnitude pruning on B200, exact with the reference
// (pruning.py:37-64): zero the k = floor(sparsity * n) entries with the
// lowest score cm[c] * |q[r,c]| (f64), ties broken by flat row-major index
// (np.argsort kind="stable").  No sort is needed:
//   per tensor: scores take at most cols * 129 distinct values, so one pass
//     builds the (column, |q|) histogram; a 4 x 16-bit radix select over
//     those weighted keys finds the k-th smallest score T and how many of
//     the ties r must go; a final ordered pass zeroes score < T and the
//     first r entries with score == T (block counts + exclusive scan).
//   per row: one CTA per row, 8 x 8-bit radix select in shared memory and
//     the same ordered tie pass.
// Non-negative doubles order like their u64 bit patterns, so keys are bits.
#include "common.cuh"

namespace dc {

constexpr int kPrThreads = 256;
constexpr int kBins = 129;  // |q| in 0..128
constexpr int kEqBlock = 4096;

struct SelectState {
    unsigned long long prefix;  // key bits selected so far
    unsigned long long k;       // 1-based rank still to find within the prefix bucket
    unsigned long long below;   // elements with key < current bucket
};

__device__ __forceinline__ unsigned long long key_of(double cm, int a) {
    return (unsigned long long)__double_as_longlong(__dmul_rn(cm, (double)a));
}

__device__ __forceinline__ int absq(int8_t v) { return v < 0 ? -(int)v : (int)v; }

// counts[c * 129 + |q|]; CTA = 256 columns x a row range, u16 private bins.
__global__ void __launch_bounds__(kPrThreads) k_colhist(const int8_t* __restrict__ q, int64_t rows, int64_t cols,
                                                         int64_t rows_per_cta, uint32_t* __restrict__ counts) {
    extern __shared__ uint16_t bins[];  // [256][130]
    const int t = threadIdx.x;
    for (int i = t; i < kPrThreads * 130; i += blockDim.x) bins[i] = 0;
    __syncthreads();
    const int64_t c = (int64_t)blockIdx.y * kPrThreads + t;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
    const int64_t r1 = min(rows, r0 + rows_per_cta);
    if (c < cols) {
        uint16_t* b = bins + t * 130;
        for (int64_t r = r0; r < r1; ++r) b[absq(q[r * cols + c])]++;
        for (int a = 0; a < kBins; ++a)
            if (b[a]) atomicAdd(&counts[c * kBins + a], (uint32_t)b[a]);
    }
}

// one radix pass over the (column, |q|) entries
__global__ void k_select_hist(const uint32_t* __restrict__ counts, const double* __restrict__ cm, int64_t cols,
                              int shift, const SelectState* __restrict__ st, unsigned long long* __restrict__ hist) {
    const int64_t n = cols * kBins;
    const unsigned long long prefix = st->prefix;
    const int top = shift + 16;  // bits above this pass's digit
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t cnt = counts[i];
        if (!cnt) continue;
        const unsigned long long key = key_of(cm[i / kBins], (int)(i % kBins));
        if (top < 64 && (key >> top) != prefix) continue;
        atomicAdd(&hist[(key >> shift) & 0xFFFF], (unsigned long long)cnt);
    }
}

// single CTA: find the digit bucket holding rank st->k
__global__ void __launch_bounds__(1024) k_select_pick(const unsigned long long* __restrict__ hist,
                                                      SelectState* __restrict__ st) {
    __shared__ unsigned long long part[1024];
    const int t = threadIdx.x;
    unsigned long long s = 0;
    for (int i = 0; i < 64; ++i) s += hist[t * 64 + i];
    part[t] = s;
    __syncthreads();
    if (t == 0) {
        unsigned long long k = st->k, acc = 0;
        int blk = 0;
        while (blk < 1023 && acc + part[blk] < k) acc += part[blk++];
        int b = blk * 64;
        while (b < blk * 64 + 63 && acc + hist[b] < k) acc += hist[b++];
        st->prefix = (st->prefix << 16) | (unsigned long long)b;
        st->k = k - acc;
        st->below += acc;
    }
}

// per 4096-element block: how many entries have key == T
__global__ void k_eq_count(const int8_t* __restrict__ q, const double* __restrict__ cm, int64_t n, int64_t cols,
                           const SelectState* __restrict__ st, uint32_t* __restrict__ blk_cnt) {
    const unsigned long long T = st->prefix;
    const int64_t b = blockIdx.x;
    uint32_t cnt = 0;
    for (int64_t i = b * kEqBlock + threadIdx.x; i < min(n, (b + 1) * kEqBlock); i += blockDim.x)
        cnt += key_of(cm[i % cols], absq(q[i])) == T;
    __shared__ uint32_t red[kPrThreads / 32];
#pragma unroll
    for (int d = 16; d; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int w = 0; w < kPrThreads / 32; ++w) s += red[w];
        blk_cnt[b] = s;
    }
}

__global__ void __launch_bounds__(1024) k_excl_scan(uint32_t* __restrict__ v, int64_t n) {
    __shared__ unsigned long long part[1024];
    const int t = threadIdx.x;
    const int64_t per = (n + 1023) / 1024;
    unsigned long long s = 0;
    for (int64_t i = t * per; i < min(n, (t + 1) * per); ++i) s += v[i];
    part[t] = s;
    __syncthreads();
    if (t == 0) {
        unsigned long long acc = 0;
        for (int i = 0; i < 1024; ++i) {
            const unsigned long long x = part[i];
            part[i] = acc;
            acc += x;
        }
    }
    __syncthreads();
    unsigned long long acc = part[t];
    for (int64_t i = t * per; i < min(n, (t + 1) * per); ++i) {
        const uint32_t x = v[i];
        v[i] = (uint32_t)acc;
        acc += x;
    }
}

// zero key < T, and key == T while the ordered tie rank < r
__global__ void __launch_bounds__(kPrThreads) k_apply(const int8_t* __restrict__ q, const double* __restrict__ cm,
                                                       int64_t n, int64_t cols, const SelectState* __restrict__ st,
                                                       const uint32_t* __restrict__ blk_prefix,
                                                       int8_t* __restrict__ out) {
    const unsigned long long T = st->prefix, r = st->k;
    const int64_t b = blockIdx.x;
    __shared__ uint32_t wc[kPrThreads / 32];
    unsigned long long run = blk_prefix[b];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t base = b * kEqBlock; base < min(n, (b + 1) * kEqBlock); base += kPrThreads) {
        const int64_t i = base + threadIdx.x;
        int8_t v = 0;
        bool eq = false, lt = false;
        if (i < n) {
            v = q[i];
            const unsigned long long key = key_of(cm[i % cols], absq(v));
            eq = key == T;
            lt = key < T;
        }
        const unsigned m = __ballot_sync(0xffffffffu, eq);
        if (lane == 0) wc[warp] = __popc(m);
        __syncthreads();
        uint32_t before = 0, total = 0;
        for (int w = 0; w < kPrThreads / 32; ++w) {
            before += (w < warp) ? wc[w] : 0;
            total += wc[w];
        }
        const unsigned long long rank = run + before + __popc(m & ((1u << lane) - 1));
        if (i < n) out[i] = (lt || (eq && rank < r)) ? (int8_t)0 : v;
        run += total;
        __syncthreads();
    }
}

// ---------------------------------------------------------------- per row
__global__ void __launch_bounds__(kPrThreads) k_prune_rows(const int8_t* __restrict__ q, const double* __restrict__ cm,
                                                            int64_t cols, int64_t k, int8_t* __restrict__ out) {
    __shared__ uint32_t hist[256];
    __shared__ unsigned long long s_prefix, s_k;
    __shared__ uint32_t wc[kPrThreads / 32];
    const int64_t row = blockIdx.x;
    const int8_t* qr = q + row * cols;
    int8_t* orow = out + row * cols;
    const int t = threadIdx.x;
    if (k <= 0) {
        for (int64_t c = t; c < cols; c += blockDim.x) orow[c] = qr[c];
        return;
    }
    if (t == 0) {
        s_prefix = 0;
        s_k = (unsigned long long)k;
    }
    for (int pass = 0; pass < 8; ++pass) {
        const int shift = 56 - 8 * pass;
        __syncthreads();
        hist[t] = 0;
        __syncthreads();
        const unsigned long long prefix = s_prefix;
        for (int64_t c = t; c < cols; c += blockDim.x) {
            const unsigned long long key = key_of(cm[c], absq(qr[c]));
            if (pass > 0 && (key >> (shift + 8)) != prefix) continue;
            atomicAdd(&hist[(key >> shift) & 0xFF], 1u);
        }
        __syncthreads();
        if (t == 0) {
            unsigned long long acc = 0, kk = s_k;
            int b = 0;
            while (b < 255 && acc + hist[b] < kk) acc += hist[b++];
            s_prefix = (prefix << 8) | (unsigned long long)b;
            s_k = kk - acc;
        }
    }
    __syncthreads();
    const unsigned long long T = s_prefix, r = s_k;
    const int warp = t >> 5, lane = t & 31;
    unsigned long long run = 0;
    for (int64_t base = 0; base < cols; base += kPrThreads) {
        const int64_t c = base + t;
        int8_t v = 0;
        bool eq = false, lt = false;
        if (c < cols) {
            v = qr[c];
            const unsigned long long key = key_of(cm[c], absq(v));
            eq = key == T;
            lt = key < T;
        }
        const unsigned m = __ballot_sync(0xffffffffu, eq);
        if (lane == 0) wc[warp] = __popc(m);
        __syncthreads();
        uint32_t before = 0, total = 0;
        for (int w = 0; w < kPrThreads / 32; ++w) {
            before += (w < warp) ? wc[w] : 0;
            total += wc[w];
        }
        const unsigned long long rank = run + before + __popc(m & ((1u << lane) - 1));
        if (c < cols) orow[c] = (lt || (eq && rank < r)) ? (int8_t)0 : v;
        run += total;
        __syncthreads();
    }
}

}  // namespace dc

using namespace dc;

// Per-tensor prune.  scratch: >= 8*65536 + 64 + 4*ceil(n/4096) + 4*cols*129 bytes.
extern "C" int dc_prune_scratch_bytes(int64_t rows, int64_t cols, uint64_t* out) {
    const int64_t n = rows * cols;
    *out = 8ull * 65536 + 64 + 4ull * (uint64_t)((n + kEqBlock - 1) / kEqBlock) + 4ull * (uint64_t)cols * kBins + 256;
    return DC_OK;
}

extern "C" int dc_prune_tensor(const int8_t* q, const double* cm, int64_t rows, int64_t cols, int64_t k,
                               int8_t* out, uint8_t* scratch, void* stream) {
    if (rows < 0 || cols < 0 || k < 0 || k > rows * cols) return DC_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = rows * cols;
    if (n == 0) return DC_OK;
    if (k == 0) {
        cudaError_t e = cudaMemcpyAsync(out, q, (size_t)n, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) {
            set_error("prune copy", e);
            return DC_ERR_CUDA;
        }
        return DC_OK;
    }
    uint8_t* p = scratch;
    auto* hist = reinterpret_cast<unsigned long long*>(p);
    p += 8ull * 65536;
    auto* sel = reinterpret_cast<SelectState*>(p);
    p += 64;
    const int64_t nblk = (n + kEqBlock - 1) / kEqBlock;
    auto* blk = reinterpret_cast<uint32_t*>(p);
    p += 4ull * nblk;
    p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 255) & ~(uintptr_t)255);
    auto* counts = reinterpret_cast<uint32_t*>(p);

    cudaMemsetAsync(counts, 0, 4ull * cols * kBins, st);
    SelectState init{0ull, (unsigned long long)k, 0ull};
    cudaMemcpyAsync(sel, &init, sizeof(init), cudaMemcpyHostToDevice, st);
    const int64_t rp = rows < 4096 ? rows : 4096;  // u16 private bins
    dim3 g1((unsigned)((rows + rp - 1) / rp), (unsigned)((cols + kPrThreads - 1) / kPrThreads));
    const int smem = kPrThreads * 130 * 2;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_colhist, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    k_colhist<<<g1, kPrThreads, smem, st>>>(q, rows, cols, rp, counts);
    DC_CHECK_LAUNCH("k_colhist");
    for (int pass = 0; pass < 4; ++pass) {
        cudaMemsetAsync(hist, 0, 8ull * 65536, st);
        k_select_hist<<<592, 256, 0, st>>>(counts, cm, cols, 48 - 16 * pass, sel, hist);
        DC_CHECK_LAUNCH("k_select_hist");
        k_select_pick<<<1, 1024, 0, st>>>(hist, sel);
        DC_CHECK_LAUNCH("k_select_pick");
    }
    k_eq_count<<<(unsigned)nblk, kPrThreads, 0, st>>>(q, cm, n, cols, sel, blk);
    DC_CHECK_LAUNCH("k_eq_count");
    k_excl_scan<<<1, 1024, 0, st>>>(blk, nblk);
    DC_CHECK_LAUNCH("k_excl_scan");
    k_apply<<<(unsigned)nblk, kPrThreads, 0, st>>>(q, cm, n, cols, sel, blk, out);
    DC_CHECK_LAUNCH("k_apply");
    return DC_OK;
}

extern "C" int dc_prune_rows(const int8_t* q, const double* cm, int64_t rows, int64_t cols, int64_t k, int8_t* out,
                             void* stream) {
    if (rows < 0 || cols < 0 || k < 0 || k > cols) return DC_ERR_ARG;
    if (rows == 0 || cols == 0) return DC_OK;
    k_prune_rows<<<(unsigned)rows, kPrThreads, 0, (cudaStream_t)stream>>>(q, cm, cols, k, out);
    DC_CHECK_LAUNCH("k_prune_rows");
    return DC_OK;
}
