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
    // whole warps iterate together so equal digits can be combined: the first
    // pass (top 16 key bits) sends nearly every entry to a handful of bins
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
        const int64_t i = base + threadIdx.x;
        uint32_t cnt = 0, bin = 0xFFFFFFFFu;
        if (i < n) {
            cnt = counts[i];
            if (cnt) {
                const uint32_t col = (uint32_t)i / (uint32_t)kBins;  // n < 2^32: 32-bit magic division
                const unsigned long long key = key_of(cm[col], (int)((uint32_t)i - col * (uint32_t)kBins));
                if (top >= 64 || (key >> top) == prefix) bin = (uint32_t)((key >> shift) & 0xFFFF);
            }
        }
        const uint32_t peers = __match_any_sync(0xffffffffu, bin);
        const uint32_t sum = __reduce_add_sync(peers, bin == 0xFFFFFFFFu ? 0u : cnt);
        if (bin != 0xFFFFFFFFu && (threadIdx.x & 31) == __ffs(peers) - 1)
            atomicAdd(&hist[bin], (unsigned long long)sum);
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
#pragma unroll 8
    for (int64_t i = t * per; i < min(n, (t + 1) * per); ++i) s += v[i];
    // block-wide exclusive scan of the 1024 thread sums (warp scans + a scan of
    // the 32 warp totals; counts < 2^32, see dc_prune_tensor)
    const int lane = t & 31, w = t >> 5;
    uint32_t inc = (uint32_t)s;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    __shared__ uint32_t wtot[32];
    if (lane == 31) wtot[w] = inc;
    __syncthreads();
    if (w == 0) {
        const uint32_t x0 = wtot[lane];
        uint32_t x = x0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += o;
        }
        wtot[lane] = x - x0;
    }
    __syncthreads();
    part[t] = wtot[w] + inc - (uint32_t)s;
    __syncthreads();
    unsigned long long acc = part[t];
    const int64_t e = min(n, (t + 1) * per);
    for (int64_t i0 = t * per; i0 < e; i0 += 8) {  // 8 loads in flight, then the stores
        uint32_t x[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = i0 + j < e ? v[i0 + j] : 0u;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (i0 + j < e) {
                v[i0 + j] = (uint32_t)acc;
                acc += x[j];
            }
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

__global__ void k_sel_init(SelectState* st, unsigned long long k) {
    st->prefix = 0;
    st->k = k;
    st->below = 0;
}

// ------------------------------------------------- per tensor, fast path
// (column, |q|) histogram: CTA = 64 columns x a row range, u32 bins in
// shared memory (thread = column x row phase, coalesced byte loads), partial
// histograms written whole (no global atomics) and summed by k_colhist_sum.
constexpr int kHcCols = 64;

__global__ void __launch_bounds__(kPrThreads) k_colhist2(const int8_t* __restrict__ q, int64_t rows, int64_t cols,
                                                          int64_t rows_per, uint32_t* __restrict__ partial) {
    __shared__ uint32_t bins[kHcCols * kBins];
    for (int i = threadIdx.x; i < kHcCols * kBins; i += blockDim.x) bins[i] = 0;
    __syncthreads();
    const int cl = threadIdx.x % kHcCols, rph = threadIdx.x / kHcCols;  // 4 row phases
    const int64_t c = (int64_t)blockIdx.y * kHcCols + cl;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = min(rows, r0 + rows_per);
    if (c < cols)
        for (int64_t r = r0 + rph; r < r1; r += kPrThreads / kHcCols) atomicAdd(&bins[cl * kBins + absq(q[r * cols + c])], 1u);
    __syncthreads();
    uint32_t* out = partial + ((int64_t)blockIdx.x * gridDim.y + blockIdx.y) * (kHcCols * kBins);
    for (int i = threadIdx.x; i < kHcCols * kBins; i += blockDim.x) out[i] = bins[i];
}

// counts[c * 129 + a] = sum over row blocks of the partials
__global__ void k_colhist_sum(const uint32_t* __restrict__ partial, int64_t n_rb, int64_t n_cb, int64_t cols,
                              uint32_t* __restrict__ counts) {
    const int64_t per_rb = n_cb * kHcCols * kBins;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cols * kBins;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t s = 0;
        for (int64_t rb = 0; rb < n_rb; ++rb) s += partial[rb * per_rb + i];
        counts[i] = s;
    }
}

// single CTA: find the 16-bit digit bucket holding rank st->k.  Coalesced
// 1024-bin tiles -> 2048 partial sums of 32 bins -> block scan -> one warp
// resolves the bin inside its 32.
__global__ void __launch_bounds__(1024) k_select_pick2(const unsigned long long* __restrict__ hist,
                                                       SelectState* __restrict__ st) {
    __shared__ unsigned long long part[2048];
    __shared__ unsigned long long wsum[32];
    __shared__ int s_part;
    __shared__ unsigned long long s_base;
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    // partial p = bins [32p, 32p + 32): warp w, round i reduces partial 32i + w
    // from one coalesced 256-B load with one REDUX (the host caps a tensor at
    // 2^32 - 1 elements, so every partial fits 32 bits); 16 loads in flight
    for (int i0 = 0; i0 < 64; i0 += 16) {
        unsigned long long v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = hist[(i0 + j) * 1024 + t];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint32_t sum = __reduce_add_sync(0xffffffffu, (uint32_t)v[j]);
            if (lane == 0) part[(i0 + j) * 32 + w] = sum;
        }
    }
    __syncthreads();
    const unsigned long long a = part[2 * t], b = part[2 * t + 1], s = a + b;
    unsigned long long inc = s;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    if (w == 0) {
        unsigned long long v = wsum[lane], x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long o = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += o;
        }
        wsum[lane] = x - v;  // exclusive
    }
    __syncthreads();
    inc += wsum[w];
    const unsigned long long k = st->k, excl = inc - s;
    if (excl < k && k <= inc) {  // exactly one thread owns the rank
        const bool first = k <= excl + a;
        s_part = 2 * t + (first ? 0 : 1);
        s_base = first ? excl : excl + a;
    }
    __syncthreads();
    if (w == 0) {  // resolve inside the 32 bins of partial s_part
        const int bin0 = s_part * 32;
        const unsigned long long v = hist[bin0 + lane];
        unsigned long long x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned long long o = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += o;
        }
        const unsigned long long lo = s_base + x - v, hi = s_base + x;
        if (lo < k && k <= hi) {
            st->prefix = (st->prefix << 16) | (unsigned long long)(bin0 + lane);
            st->k = k - lo;
            st->below += lo;
        }
    }
}

// per column: |q| < lo -> score < T; lo <= |q| < hi -> score == T (cm >= 0, so
// the score is non-decreasing in |q|; strictly increasing when cm > 0)
__global__ void k_col_bounds(const double* __restrict__ cm, int64_t cols, const SelectState* __restrict__ st,
                             uint8_t* __restrict__ lo, uint8_t* __restrict__ hi) {
    const unsigned long long T = st->prefix;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += (int64_t)gridDim.x * blockDim.x) {
        int l = 0, h;
        while (l < kBins && key_of(cm[c], l) < T) ++l;
        h = l;
        while (h < kBins && key_of(cm[c], h) == T) ++h;
        lo[c] = (uint8_t)l;
        hi[c] = (uint8_t)h;
    }
}

// 16 consecutive elements per thread (one 4096-element block per CTA):
// lt / eq flags from the column bounds, no f64 work per element
__device__ __forceinline__ void flags16(const int8_t* __restrict__ q, const uint8_t* __restrict__ lo,
                                        const uint8_t* __restrict__ hi, int64_t n, int64_t cols, int64_t i0,
                                        bool vec, int8_t (&v)[16], uint32_t& ltm, uint32_t& eqm) {
    ltm = eqm = 0;
    if (vec && i0 + 16 <= n) {  // cols % 16 == 0: one row, 16-B aligned
        const int64_t c0 = (uint32_t)i0 % (uint32_t)cols;  // n < 2^32 (dc_prune_tensor): 32-bit division
        const uint4 qv = *reinterpret_cast<const uint4*>(q + i0);
        const uint4 lv = *reinterpret_cast<const uint4*>(lo + c0);
        const uint4 hv = *reinterpret_cast<const uint4*>(hi + c0);
        memcpy(v, &qv, 16);
        // four bytes per SIMD op: |q| (0x80 -> 128, unsigned), byte compares
        // against the column bounds, byte masks folded to 4 bits each
        const uint32_t qw[4] = {qv.x, qv.y, qv.z, qv.w}, lw[4] = {lv.x, lv.y, lv.z, lv.w},
                       hw[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t a = __vabs4(qw[k]);
            const uint32_t lt = __vcmpltu4(a, lw[k]);
            const uint32_t eq = __vcmpltu4(a, hw[k]) & ~lt;
            ltm |= (((lt & 0x01010101u) * 0x01020408u) >> 24) << (4 * k);
            eqm |= (((eq & 0x01010101u) * 0x01020408u) >> 24) << (4 * k);
        }
        return;
    }
    int64_t c = (uint32_t)i0 % (uint32_t)cols;
    for (int k = 0; k < 16; ++k) {
        const int64_t i = i0 + k;
        v[k] = 0;
        if (i < n) {
            v[k] = q[i];
            const int a = absq(v[k]);
            ltm |= (uint32_t)(a < lo[c]) << k;
            eqm |= (uint32_t)(a >= lo[c] && a < hi[c]) << k;
        }
        if (++c == cols) c = 0;
    }
}

// Fast per-element passes: a block covers kEqSub sub-tiles of kEqBlock
// elements (thread t: 16 elements at sub-tile r, offset 16t); all kEqSub
// 16-B loads are issued before any use, so each thread keeps 4 in flight.
constexpr int kEqSub = 4;
constexpr int64_t kEqBlock2 = (int64_t)kEqSub * kEqBlock;

__global__ void __launch_bounds__(kPrThreads) k_eq_count2(const int8_t* __restrict__ q, const uint8_t* __restrict__ lo,
                                                           const uint8_t* __restrict__ hi, int64_t n, int64_t cols,
                                                           bool vec, uint32_t* __restrict__ blk_cnt) {
    uint32_t cnt = 0;
#pragma unroll
    for (int r = 0; r < kEqSub; ++r) {
        int8_t v[16];
        uint32_t ltm, eqm;
        flags16(q, lo, hi, n, cols, (int64_t)blockIdx.x * kEqBlock2 + r * kEqBlock + threadIdx.x * 16, vec, v, ltm,
                eqm);
        cnt += __popc(eqm);
    }
    __shared__ uint32_t red[kPrThreads / 32];
#pragma unroll
    for (int d = 16; d; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t s = 0;
        for (int w = 0; w < kPrThreads / 32; ++w) s += red[w];
        blk_cnt[blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(kPrThreads) k_apply2(const int8_t* __restrict__ q, const uint8_t* __restrict__ lo,
                                                        const uint8_t* __restrict__ hi, int64_t n, int64_t cols,
                                                        bool vec, const SelectState* __restrict__ st,
                                                        const uint32_t* __restrict__ blk_prefix,
                                                        int8_t* __restrict__ out) {
    const unsigned long long r_keep = st->k;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int8_t v[kEqSub][16];
    uint32_t ltm[kEqSub], eqm[kEqSub];
#pragma unroll
    for (int r = 0; r < kEqSub; ++r)
        flags16(q, lo, hi, n, cols, (int64_t)blockIdx.x * kEqBlock2 + r * kEqBlock + threadIdx.x * 16, vec, v[r],
                ltm[r], eqm[r]);
    __shared__ uint32_t ws[kEqSub][kPrThreads / 32];
    // tie ranks in row-major order: sub-tile r before r + 1, thread t before t + 1
    uint32_t inc[kEqSub];
#pragma unroll
    for (int r = 0; r < kEqSub; ++r) {
        inc[r] = __popc(eqm[r]);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc[r], d);
            if (lane >= d) inc[r] += o;
        }
        if (lane == 31) ws[r][w] = inc[r];
    }
    __syncthreads();
    unsigned long long base = blk_prefix[blockIdx.x];
#pragma unroll
    for (int r = 0; r < kEqSub; ++r) {
        uint32_t before = 0, total = 0;
        for (int k = 0; k < kPrThreads / 32; ++k) {
            const uint32_t x = ws[r][k];
            before += k < w ? x : 0u;
            total += x;
        }
        unsigned long long rank = base + before + inc[r] - __popc(eqm[r]);
        base += total;
        uint32_t zero = ltm[r];
        for (uint32_t e = eqm[r]; e; e &= e - 1) {  // ties (few): the first r_keep in row-major order
            if (rank < r_keep) zero |= e & (0u - e);
            ++rank;
        }
        const int64_t i0 = (int64_t)blockIdx.x * kEqBlock2 + r * kEqBlock + threadIdx.x * 16;
        if (vec && i0 + 16 <= n) {
            uint32_t o[4];
            memcpy(o, v[r], 16);
#pragma unroll
            for (int k = 0; k < 4; ++k)  // 4 zero bits -> 4 byte masks
                o[k] &= ~((((zero >> (4 * k)) & 15u) * 0x00204081u & 0x01010101u) * 0xFFu);
            *reinterpret_cast<uint4*>(out + i0) = make_uint4(o[0], o[1], o[2], o[3]);
        } else {
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if ((zero >> k) & 1) v[r][k] = 0;
            for (int k = 0; k < 16; ++k)
                if (i0 + k < n) out[i0 + k] = v[r][k];
        }
    }
}

static int sm_count_pr() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// ---------------------------------------------------------------- per row
// Register path (cols <= 4096): a CTA per row, 16 columns per thread, keys
// computed once; 8 x 8-bit radix passes over a shared 256-bin histogram with a
// block-scan bucket pick; then the ordered tie pass.
constexpr int kRowMax = kPrThreads * 16;

__device__ __forceinline__ void block_pick256(const uint32_t* hist, unsigned long long& prefix, unsigned long long& kk,
                                              unsigned long long* s_prefix, unsigned long long* s_k,
                                              uint32_t* wsum) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const uint32_t v = hist[t];
    uint32_t inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    uint32_t before = 0;
    for (int i = 0; i < w; ++i) before += wsum[i];
    inc += before;
    const unsigned long long lo = inc - v;
    if (lo < kk && kk <= (unsigned long long)inc) {
        *s_prefix = (prefix << 8) | (unsigned long long)t;
        *s_k = kk - lo;
        s_k[1] = v;  // the chosen bucket's population
    }
    __syncthreads();
    prefix = *s_prefix;
    kk = *s_k;
}

__global__ void __launch_bounds__(kPrThreads) k_prune_rows2(const int8_t* __restrict__ q, const double* __restrict__ cm,
                                                             int64_t rows, int64_t cols, int64_t k,
                                                             int8_t* __restrict__ out) {
    // persistent over rows: thread t owns columns [16t, 16t + 16) of every row,
    // their channel maxima stay in registers (one load per CTA, not per row)
    __shared__ uint32_t hist[256];
    __shared__ uint32_t wsum[kPrThreads / 32];
    __shared__ unsigned long long s_prefix, s_k[2], s_min[kPrThreads / 32], s_max[kPrThreads / 32];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int c0 = t * 16;
    double cmr[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) cmr[j] = c0 + j < cols ? cm[c0 + j] : 0.0;
    const bool vec = (cols & 15) == 0 && ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        const int8_t* qr = q + row * cols;
        int8_t* orow = out + row * cols;
        int8_t v[16];
        if (vec) {
            uint4 qv = make_uint4(0, 0, 0, 0);
            if (c0 < cols) qv = *reinterpret_cast<const uint4*>(qr + c0);
            memcpy(v, &qv, 16);
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) v[j] = c0 + j < cols ? qr[c0 + j] : 0;
        }
        unsigned long long key[16];
        unsigned long long kmin = ~0ull, kmax = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            key[j] = c0 + j < cols ? key_of(cmr[j], absq(v[j])) : ~0ull;
            if (c0 + j < cols) {
                kmin = min(kmin, key[j]);
                kmax = max(kmax, key[j]);
            }
        }
        // the row's keys share their leading bytes (scores span a few binades):
        // start the radix passes at the first byte where min and max differ
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            kmin = min(kmin, __shfl_xor_sync(0xffffffffu, kmin, d));
            kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, d));
        }
        __syncthreads();  // previous row done with the shared scratch
        if (lane == 0) {
            s_min[w] = kmin;
            s_max[w] = kmax;
        }
        __syncthreads();
        for (int i = 0; i < kPrThreads / 32; ++i) {
            kmin = min(kmin, s_min[i]);
            kmax = max(kmax, s_max[i]);
        }
        const int p0 = kmin == kmax ? 8 : __clzll(kmin ^ kmax) / 8;
        unsigned long long prefix = p0 == 0 ? 0ull : p0 == 8 ? kmin : kmin >> (64 - 8 * p0);
        unsigned long long kk = (unsigned long long)k;
        for (int pass = p0; pass < 8; ++pass) {
            const int shift = 56 - 8 * pass;
            hist[t] = 0;
            __syncthreads();
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (c0 + j < cols && (pass == 0 || (key[j] >> (shift + 8)) == prefix))
                    atomicAdd(&hist[(key[j] >> shift) & 0xFF], 1u);
            __syncthreads();
            block_pick256(hist, prefix, kk, &s_prefix, s_k, wsum);
            if (s_k[1] == 1 && shift > 0) {  // one key in the bucket: it is the threshold
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < cols && (key[j] >> shift) == prefix) s_prefix = key[j];
                __syncthreads();
                prefix = s_prefix;
                break;
            }
        }
        // ordered ties: zero key < T, and the first kk entries with key == T
        const unsigned long long T = prefix;
        uint32_t eqm = 0, ltm = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            eqm |= (uint32_t)(c0 + j < cols && key[j] == T) << j;
            ltm |= (uint32_t)(key[j] < T) << j;
        }
        const uint32_t cnt = __popc(eqm);
        uint32_t inc = cnt;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += o;
        }
        __syncthreads();
        if (lane == 31) wsum[w] = inc;
        __syncthreads();
        uint32_t before = 0;
        for (int i = 0; i < w; ++i) before += wsum[i];
        unsigned long long rank = before + inc - cnt;
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if ((eqm >> j) & 1) {
                if (rank < kk) ltm |= 1u << j;
                ++rank;
            }
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if ((ltm >> j) & 1) v[j] = 0;
        if (vec) {
            if (c0 < cols) {
                uint4 o;
                memcpy(&o, v, 16);
                *reinterpret_cast<uint4*>(orow + c0) = o;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (c0 + j < cols) orow[c0 + j] = v[j];
        }
    }
}

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
namespace dc {
// Eq. 5 importance score (pruning.py:37-40): score[r, c] = cm[c] * |q[r, c]|,
// f64 (exact: |q| <= 127 is exact and one IEEE multiply, never -0.0 since
// cm >= 0 and |q| >= 0).  16 int8 per thread (one 16-B load), 8-B stores.
__global__ void k_prune_scores(const int8_t* __restrict__ q, const double* __restrict__ cm, int64_t rows,
                               int64_t cols, double* __restrict__ out) {
    const int64_t n = rows * cols;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 16;
    for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16; i0 < n; i0 += stride) {
        if (i0 + 16 <= n && (reinterpret_cast<uintptr_t>(q + i0) & 15) == 0) {
            const int4 v = *reinterpret_cast<const int4*>(q + i0);
            const int8_t* b = reinterpret_cast<const int8_t*>(&v);
            int64_t c = i0 % cols;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                out[i0 + k] = cm[c] * (double)abs((int)b[k]);
                if (++c == cols) c = 0;
            }
        } else {
            for (int64_t i = i0; i < n && i < i0 + 16; ++i) out[i] = cm[i % cols] * (double)abs((int)q[i]);
        }
    }
}
}  // namespace dc

extern "C" int dc_prune_scores(const int8_t* q, const double* cm, int64_t rows, int64_t cols, double* out,
                               void* stream) {
    if (rows < 0 || cols < 0) return DC_ERR_ARG;
    const int64_t n = rows * cols;
    if (n == 0) return DC_OK;
    const int64_t want = (n + 16 * 256 - 1) / (16 * 256);
    const int64_t grid = want < (int64_t)sm_count_pr() * 8 ? want : (int64_t)sm_count_pr() * 8;
    k_prune_scores<<<(unsigned)grid, 256, 0, (cudaStream_t)stream>>>(q, cm, rows, cols, out);
    DC_CHECK_LAUNCH("k_prune_scores");
    return DC_OK;
}

extern "C" int dc_prune_scratch_bytes(int64_t rows, int64_t cols, uint64_t* out) {
    const int64_t n = rows * cols;
    const uint64_t n_cb = (uint64_t)((cols + kHcCols - 1) / kHcCols);
    *out = 8ull * 65536 + 64 + 4ull * (uint64_t)((n + kEqBlock - 1) / kEqBlock) + 4ull * (uint64_t)cols * kBins + 256 +
           2ull * (uint64_t)cols + 256 + 4ull * kHcCols * kBins * n_cb * 16 + 256;
    return DC_OK;
}

extern "C" int dc_prune_tensor(const int8_t* q, const double* cm, int64_t rows, int64_t cols, int64_t k,
                               int8_t* out, uint8_t* scratch, void* stream) {
    if (rows < 0 || cols < 0 || k < 0 || k > rows * cols) return DC_ERR_ARG;
    if (rows * cols > 0xFFFFFFFFll) {  // selection partials are summed in 32 bits
        set_error_msg("dc_prune_tensor: at most 2^32 - 1 elements per tensor");
        return DC_ERR_ARG;
    }
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

    p += 4ull * cols * kBins;
    p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 255) & ~(uintptr_t)255);
    uint8_t* lo = p;
    uint8_t* hi = p + cols;
    p += 2ull * cols;
    p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 255) & ~(uintptr_t)255);
    auto* partial = reinterpret_cast<uint32_t*>(p);

    k_sel_init<<<1, 1, 0, st>>>(sel, (unsigned long long)k);  // (a pageable H2D copy would synchronize)
    DC_CHECK_LAUNCH("k_sel_init");
    // (column, |q|) histogram: <= 16 row blocks, ~4 CTAs per SM
    const int64_t n_cb = (cols + kHcCols - 1) / kHcCols;
    int64_t n_rb = (4 * 148 + n_cb - 1) / n_cb;
    n_rb = n_rb < 1 ? 1 : (n_rb > 16 ? 16 : n_rb);
    if (n_rb > rows) n_rb = rows;
    const int64_t rows_per = (rows + n_rb - 1) / n_rb;
    n_rb = (rows + rows_per - 1) / rows_per;
    k_colhist2<<<dim3((unsigned)n_rb, (unsigned)n_cb), kPrThreads, 0, st>>>(q, rows, cols, rows_per, partial);
    DC_CHECK_LAUNCH("k_colhist2");
    k_colhist_sum<<<(unsigned)((cols * kBins + 255) / 256 < 1184 ? (cols * kBins + 255) / 256 : 1184), 256, 0, st>>>(partial, n_rb, n_cb, cols,
                                                                                          counts);
    DC_CHECK_LAUNCH("k_colhist_sum");
    for (int pass = 0; pass < 4; ++pass) {
        cudaMemsetAsync(hist, 0, 8ull * 65536, st);
        k_select_hist<<<592, 256, 0, st>>>(counts, cm, cols, 48 - 16 * pass, sel, hist);
        DC_CHECK_LAUNCH("k_select_hist");
        k_select_pick2<<<1, 1024, 0, st>>>(hist, sel);
        DC_CHECK_LAUNCH("k_select_pick2");
    }
    k_col_bounds<<<(unsigned)((cols + 255) / 256 < 1184 ? (cols + 255) / 256 : 1184), 256, 0, st>>>(cm, cols, sel, lo, hi);
    DC_CHECK_LAUNCH("k_col_bounds");
    const bool vec = cols % 16 == 0 && (reinterpret_cast<uintptr_t>(q) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    const int64_t nblk2 = (n + kEqBlock2 - 1) / kEqBlock2;  // <= nblk: fits the scratch
    k_eq_count2<<<(unsigned)nblk2, kPrThreads, 0, st>>>(q, lo, hi, n, cols, vec, blk);
    DC_CHECK_LAUNCH("k_eq_count2");
    k_excl_scan<<<1, 1024, 0, st>>>(blk, nblk2);
    DC_CHECK_LAUNCH("k_excl_scan");
    k_apply2<<<(unsigned)nblk2, kPrThreads, 0, st>>>(q, lo, hi, n, cols, vec, sel, blk, out);
    DC_CHECK_LAUNCH("k_apply2");
    return DC_OK;
}

extern "C" int dc_prune_rows(const int8_t* q, const double* cm, int64_t rows, int64_t cols, int64_t k, int8_t* out,
                             void* stream) {
    if (rows < 0 || cols < 0 || k < 0 || k > cols) return DC_ERR_ARG;
    if (rows == 0 || cols == 0) return DC_OK;
    if (k > 0 && cols <= kRowMax) {
        const int64_t cap = (int64_t)sm_count_pr() * 2;  // resident CTAs (123 regs x 256 threads)
        k_prune_rows2<<<(unsigned)(rows < cap ? rows : cap), kPrThreads, 0, (cudaStream_t)stream>>>(q, cm, rows,
                                                                                                  cols, k, out);
        DC_CHECK_LAUNCH("k_prune_rows2");
        return DC_OK;
    }
    k_prune_rows<<<(unsigned)rows, kPrThreads, 0, (cudaStream_t)stream>>>(q, cm, cols, k, out);
    DC_CHECK_LAUNCH("k_prune_rows");
    return DC_OK;
}
