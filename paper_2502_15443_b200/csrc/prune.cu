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
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

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

// ------------------------------------------- per tensor, round-2 path
// (column, |q|) histogram with 16-byte loads: a CTA is 8 column groups of 16
// columns (one uint4 per row each) x 128 row phases, 4 rows in flight per
// thread; u32 bins for its 128 columns in shared memory; partial histograms
// per row block, summed by k_colhist3_sum.
constexpr int kH3Cols = 128;
constexpr int kH3Threads = 1024;

__global__ void __launch_bounds__(kH3Threads, 2) k_colhist3(const int8_t* __restrict__ q, int64_t rows, int64_t cols,
                                                             int64_t rows_per, bool vec, uint32_t* __restrict__ partial) {
    extern __shared__ uint32_t hb[];  // [kH3Cols][kBins]
    for (int i = threadIdx.x; i < kH3Cols * kBins; i += blockDim.x) hb[i] = 0;
    __syncthreads();
    const int cg8 = threadIdx.x & 7, rph = threadIdx.x >> 3;  // 8 column groups x 128 row phases
    const int64_t c0 = (int64_t)blockIdx.y * kH3Cols + cg8 * 16;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = min(rows, r0 + rows_per);
    uint32_t* b = hb + cg8 * 16 * kBins;
    if (vec && c0 + 16 <= cols) {
        for (int64_t r = r0 + rph; r < r1; r += 4 * (kH3Threads / 8)) {
            uint4 v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int64_t rr = r + j * (kH3Threads / 8);
                v[j] = rr < r1 ? __ldg(reinterpret_cast<const uint4*>(q + rr * cols + c0)) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (r + j * (kH3Threads / 8) >= r1) break;
                const uint32_t w[4] = {__vabs4(v[j].x), __vabs4(v[j].y), __vabs4(v[j].z), __vabs4(v[j].w)};
#pragma unroll
                for (int e = 0; e < 16; ++e) atomicAdd(&b[e * kBins + ((w[e >> 2] >> (8 * (e & 3))) & 0xFF)], 1u);
            }
        }
    } else {
        for (int64_t r = r0 + rph; r < r1; r += kH3Threads / 8)
            for (int e = 0; e < 16 && c0 + e < cols; ++e) atomicAdd(&b[e * kBins + absq(q[r * cols + c0 + e])], 1u);
    }
    __syncthreads();
    uint32_t* out = partial + ((int64_t)blockIdx.x * gridDim.y + blockIdx.y) * (kH3Cols * kBins);
    for (int i = threadIdx.x; i < kH3Cols * kBins; i += blockDim.x) out[i] = hb[i];
}

// counts[c * 129 + a] = sum over row blocks of the k_colhist3 partials
__global__ void k_colhist3_sum(const uint32_t* __restrict__ partial, int64_t n_rb, int64_t n_cb, int64_t cols,
                               uint32_t* __restrict__ counts) {
    const int64_t per_rb = n_cb * kH3Cols * kBins;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cols * kBins;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t s = 0;
        for (int64_t rb = 0; rb < n_rb; ++rb) s += partial[rb * per_rb + i];
        counts[i] = s;
    }
}

// Block-wide: find the entry of v[0..m) (m <= blockDim.x, u32 counts) holding
// rank k (1-based) given `base` = count before v[0]; returns index and the
// count before it through shared memory.  All threads participate.
__device__ __forceinline__ void block_find(const uint32_t* v, int m, unsigned long long k, unsigned long long base,
                                           int* s_idx, unsigned long long* s_before, unsigned long long* wsum) {
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const unsigned long long x = t < m ? __ldcg(v + t) : 0ull;  // written by other CTAs: bypass L1
    unsigned long long inc = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    unsigned long long before = base;
    for (int i = 0; i < w; ++i) before += wsum[i];
    inc += before;
    if (t < m && inc - x < k && k <= inc) {
        *s_idx = t;
        *s_before = inc - x;
    }
    __syncthreads();
}

// The whole k-th-score selection in ONE cooperative launch (grid = SMs):
// per 16-bit digit pass, a grid-strided (column, |q|) histogram with
// warp-aggregated atomics into u32 bins (n < 2^32), per-CTA slice sums, and
// CTA 0 picks the slice and then the bin with block scans; the two histogram
// buffers alternate so the next pass's zeroing overlaps the pick.  Then the
// per-column |q| bounds of score < T and score == T.  Replaces 4 x (memset,
// k_select_hist, k_select_pick2) + k_col_bounds (13 launches).
constexpr int kSelThreads = 512;

__global__ void __launch_bounds__(kSelThreads) k_select_coop(const uint32_t* __restrict__ counts,
                                                             const double* __restrict__ cm, int64_t cols,
                                                             SelectState* __restrict__ st, uint32_t* __restrict__ hist2,
                                                             uint32_t* __restrict__ psum2, uint8_t* __restrict__ lo,
                                                             uint8_t* __restrict__ hi) {
    // hist2 / psum2: two buffers each (pass parity), zeroed by the host before
    // the launch; the buffer of pass p + 2 is re-zeroed during pass p + 1's pick
    cg::grid_group grid = cg::this_grid();
    const int64_t n = cols * kBins;
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    const int slice = (65536 + gridDim.x - 1) / gridDim.x;
    __shared__ unsigned long long wsum[kSelThreads / 32], s_before;
    __shared__ int s_idx;
    for (int pass = 0; pass < 4; ++pass) {
        uint32_t* hist = hist2 + (pass & 1) * 65536;
        uint32_t* psum = psum2 + (pass & 1) * 4096;
        const int shift = 48 - 16 * pass, top = shift + 16;
        // st / hist / psum are written by other CTAs between grid barriers: every
        // read of them bypasses L1 (ld.cg), which is not coherent across SMs
        const unsigned long long prefix = __ldcg(&st->prefix);
        // histogram of this pass's digit; the slice totals accumulate alongside
        for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += gs) {
            const int64_t i = base + threadIdx.x;
            uint32_t cnt = 0, bin = 0xFFFFFFFFu;
            if (i < n) {
                cnt = counts[i];
                if (cnt) {
                    const uint32_t col = (uint32_t)i / (uint32_t)kBins;
                    const unsigned long long key = key_of(cm[col], (int)((uint32_t)i - col * (uint32_t)kBins));
                    if (top >= 64 || (key >> top) == prefix) bin = (uint32_t)((key >> shift) & 0xFFFF);
                }
            }
            const uint32_t peers = __match_any_sync(0xffffffffu, bin);
            const uint32_t sum = __reduce_add_sync(peers, bin == 0xFFFFFFFFu ? 0u : cnt);
            if (bin != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], sum);
        }
        grid.sync();
        {  // per-CTA slice sums (an atomic per slice would serialise: pass 0 sends
           // nearly every key to a handful of bins)
            __shared__ uint32_t red[kSelThreads / 32];
            uint32_t v = 0;
            const int b0 = blockIdx.x * slice;
            for (int b = b0 + threadIdx.x; b < min(65536, b0 + slice); b += blockDim.x) v += __ldcg(hist + b);
            v = __reduce_add_sync(0xffffffffu, v);
            if (lane == 0) red[threadIdx.x >> 5] = v;
            __syncthreads();
            if (threadIdx.x == 0) {
                uint32_t t = 0;
                for (int k = 0; k < kSelThreads / 32; ++k) t += red[k];
                psum[blockIdx.x] = t;
            }
        }
        grid.sync();
        if (blockIdx.x == 0) {
            const unsigned long long k = __ldcg(&st->k);
            // windows of kSelThreads entries: (index, count before) of the rank-k entry
            auto find = [&](const uint32_t* v, int m, unsigned long long& base) -> int {
                for (int c0 = 0; c0 < m; c0 += kSelThreads) {
                    if (threadIdx.x == 0) s_idx = -1;
                    __syncthreads();
                    block_find(v + c0, min(kSelThreads, m - c0), k, base, &s_idx, &s_before, wsum);
                    const int idx = s_idx;
                    if (idx >= 0) {
                        base = s_before;
                        __syncthreads();
                        return c0 + idx;
                    }
                    for (int i = 0; i < kSelThreads / 32; ++i) base += wsum[i];
                    __syncthreads();
                }
                return m - 1;  // unreachable for 1 <= k <= total
            };
            unsigned long long base = 0;
            const int sl = find(psum, (int)gridDim.x, base);  // slice holding rank k
            const int b0 = sl * slice;
            const int bin = b0 + find(hist + b0, min(65536, b0 + slice) - b0, base);  // bin inside it
            if (threadIdx.x == 0) {
                st->prefix = (__ldcg(&st->prefix) << 16) | (unsigned long long)bin;
                st->k = k - base;
                st->below = __ldcg(&st->below) + base;
            }
        }
        // the buffers of pass - 1 were consumed by its pick: zero them for pass + 1
        if (pass >= 1 && pass < 3 && (blockIdx.x != 0 || gridDim.x == 1)) {
            uint32_t* h = hist2 + ((pass - 1) & 1) * 65536;
            const bool solo = gridDim.x == 1;
            const int64_t zt = solo ? threadIdx.x : (int64_t)(blockIdx.x - 1) * blockDim.x + threadIdx.x;
            const int64_t zs = solo ? blockDim.x : (int64_t)(gridDim.x - 1) * blockDim.x;
            for (int64_t i = zt; i < 65536; i += zs) h[i] = 0;
        }
        grid.sync();
    }
    const unsigned long long T = __ldcg(&st->prefix);
    for (int64_t c = gt; c < cols; c += gs) {
        int l = 0, h;
        while (l < kBins && key_of(cm[c], l) < T) ++l;
        h = l;
        while (h < kBins && key_of(cm[c], h) == T) ++h;
        lo[c] = (uint8_t)l;
        hi[c] = (uint8_t)h;
    }
}

// Single-pass tie ranks (decoupled look-back): tiles of kEqBlock2 elements
// are claimed in order from a counter; a tile publishes its tie count (flag
// A), then warp 0 looks back 32 predecessors at a time, adding counts until
// a predecessor with an inclusive prefix (flag P), and publishes its own
// inclusive prefix -- eq_count + scan + apply as one pass over q.
constexpr unsigned long long kLbA = 1ull << 62, kLbP = 2ull << 62, kLbMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kPrThreads) k_apply3(const int8_t* __restrict__ q, const uint8_t* __restrict__ lo,
                                                        const uint8_t* __restrict__ hi, int64_t n, int64_t cols,
                                                        bool vec, const SelectState* __restrict__ st,
                                                        unsigned long long* __restrict__ look,
                                                        uint32_t* __restrict__ tile_ctr, int8_t* __restrict__ out) {
    __shared__ uint32_t s_tile;
    __shared__ unsigned long long s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    const unsigned long long r_keep = st->k;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int8_t v[kEqSub][16];
    uint32_t ltm[kEqSub], eqm[kEqSub];
#pragma unroll
    for (int r = 0; r < kEqSub; ++r)
        flags16(q, lo, hi, n, cols, tile * kEqBlock2 + r * kEqBlock + threadIdx.x * 16, vec, v[r], ltm[r], eqm[r]);
    __shared__ uint32_t ws[kEqSub][kPrThreads / 32];
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
    if (w == 0) {
        uint32_t tot = 0;
#pragma unroll
        for (int r = 0; r < kEqSub; ++r) tot += lane < kPrThreads / 32 ? ws[r][lane] : 0u;
        tot = __reduce_add_sync(0xffffffffu, tot);
        unsigned long long excl = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(&look[0], kLbP | tot);
        } else {
            if (lane == 0) atomicExch(&look[tile], kLbA | tot);
            int64_t j = tile - 1;  // window [j - 31, j], lane l reads j - l
            while (true) {
                unsigned long long f = kLbP;  // before tile 0: an empty inclusive prefix
                if (j - lane >= 0) {
                    do f = *((volatile unsigned long long*)&look[j - lane]);
                    while ((f & ~kLbMask) == 0);
                }
                const uint32_t pm = __ballot_sync(0xffffffffu, (f & ~kLbMask) == kLbP);
                const int stop = pm ? __ffs(pm) - 1 : 32;  // nearest predecessor with a prefix
                const unsigned long long add = lane <= stop ? (f & kLbMask) : 0ull;
                unsigned long long sum = add;
#pragma unroll
                for (int d = 16; d; d >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, d);
                excl += sum;
                if (pm) break;
                j -= 32;
            }
            if (lane == 0) atomicExch(&look[tile], kLbP | (excl + tot));
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    unsigned long long base = s_excl;
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
        const int64_t i0 = tile * kEqBlock2 + r * kEqBlock + threadIdx.x * 16;
        if (vec && i0 + 16 <= n) {
            uint32_t o[4];
            memcpy(o, v[r], 16);
#pragma unroll
            for (int k = 0; k < 4; ++k)
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

static int64_t colhist3_rb(int64_t rows, int64_t cols) {
    const int64_t n_cb = (cols + kH3Cols - 1) / kH3Cols;
    int64_t n_rb = (2 * (int64_t)sm_count_pr() + n_cb - 1) / n_cb;
    n_rb = n_rb < 1 ? 1 : (n_rb > 64 ? 64 : n_rb);
    return n_rb > rows ? (rows > 0 ? rows : 1) : n_rb;
}

extern "C" int dc_prune_scratch_bytes(int64_t rows, int64_t cols, uint64_t* out) {
    const int64_t n = rows * cols;
    const uint64_t n_cb = (uint64_t)((cols + kH3Cols - 1) / kH3Cols);
    const uint64_t tiles = (uint64_t)((n + kEqBlock2 - 1) / kEqBlock2);
    *out = 4ull * 2 * 65536 + 4ull * 2 * 4096 + 64 + 256 + 8ull * tiles + 256 + 4ull * (uint64_t)cols * kBins + 256 +
           2ull * (uint64_t)cols + 256 + 4ull * kH3Cols * kBins * n_cb * (uint64_t)colhist3_rb(rows, cols) + 256;
    return DC_OK;
}

// Per tensor: (column, |q|) histogram -> one cooperative selection launch ->
// one look-back apply pass (5 launches + 2 memsets, was 20).
extern "C" int dc_prune_tensor(const int8_t* q, const double* cm, int64_t rows, int64_t cols, int64_t k,
                               int8_t* out, uint8_t* scratch, void* stream) {
    if (rows < 0 || cols < 0 || k < 0 || k > rows * cols) return DC_ERR_ARG;
    if (rows * cols > 0xFFFFFFFFll) {  // selection bins are u32
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
    auto align = [](uint8_t* p) {
        return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 255) & ~(uintptr_t)255);
    };
    uint8_t* p = scratch;
    auto* hist2 = reinterpret_cast<uint32_t*>(p);
    p += 4ull * 2 * 65536;
    auto* psum = reinterpret_cast<uint32_t*>(p);
    p += 4ull * 2 * 4096;
    auto* sel = reinterpret_cast<SelectState*>(p);
    p += 64;
    auto* tile_ctr = reinterpret_cast<uint32_t*>(p);
    p = align(p + 4);
    const int64_t tiles = (n + kEqBlock2 - 1) / kEqBlock2;
    auto* look = reinterpret_cast<unsigned long long*>(p);
    p = align(p + 8ull * tiles);
    auto* counts = reinterpret_cast<uint32_t*>(p);
    p = align(p + 4ull * cols * kBins);
    uint8_t* lo = p;
    uint8_t* hi = p + cols;
    p = align(p + 2ull * cols);
    auto* partial = reinterpret_cast<uint32_t*>(p);
    const bool vec = cols % 16 == 0 && (reinterpret_cast<uintptr_t>(q) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(out) & 15) == 0;

    k_sel_init<<<1, 1, 0, st>>>(sel, (unsigned long long)k);  // (a pageable H2D copy would synchronize)
    DC_CHECK_LAUNCH("k_sel_init");
    const int64_t n_cb = (cols + kH3Cols - 1) / kH3Cols;
    int64_t n_rb = colhist3_rb(rows, cols);
    const int64_t rows_per = (rows + n_rb - 1) / n_rb;
    n_rb = (rows + rows_per - 1) / rows_per;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_colhist3, cudaFuncAttributeMaxDynamicSharedMemorySize, kH3Cols * kBins * 4);
        attr = true;
    }
    k_colhist3<<<dim3((unsigned)n_rb, (unsigned)n_cb), kH3Threads, kH3Cols * kBins * 4, st>>>(q, rows, cols, rows_per,
                                                                                           vec, partial);
    DC_CHECK_LAUNCH("k_colhist3");
    const int64_t sb = (cols * kBins + 255) / 256;
    k_colhist3_sum<<<(unsigned)(sb < 1184 ? sb : 1184), 256, 0, st>>>(partial, n_rb, n_cb, cols, counts);
    DC_CHECK_LAUNCH("k_colhist3_sum");
    {  // the k-th score and the per-column bounds: one cooperative launch
        cudaError_t ez = cudaMemsetAsync(hist2, 0, 4ull * 2 * 65536 + 4ull * 2 * 4096, st);  // hist2 + psum2
        if (ez != cudaSuccess) {
            set_error("prune memset", ez);
            return DC_ERR_CUDA;
        }
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_select_coop, kSelThreads, 0);
        if (per_sm < 1) {
            set_error_msg("k_select_coop: not resident");
            return DC_ERR_CUDA;
        }
        int grid = sm_count_pr();
        if (grid > 4096) grid = 4096;
        void* args[] = {(void*)&counts, (void*)&cm, (void*)&cols, (void*)&sel, (void*)&hist2, (void*)&psum,
                        (void*)&lo, (void*)&hi};
        cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_select_coop, dim3((unsigned)grid), dim3(kSelThreads),
                                                    args, 0, st);
        if (e != cudaSuccess) {
            set_error("k_select_coop", e);
            return DC_ERR_CUDA;
        }
    }
    cudaError_t e = cudaMemsetAsync(tile_ctr, 0, 4, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(look, 0, 8ull * tiles, st);
    if (e != cudaSuccess) {
        set_error("prune memset", e);
        return DC_ERR_CUDA;
    }
    k_apply3<<<(unsigned)tiles, kPrThreads, 0, st>>>(q, lo, hi, n, cols, vec, sel, look, tile_ctr, out);
    DC_CHECK_LAUNCH("k_apply3");
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
