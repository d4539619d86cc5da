// Activation-aware magnitude pruning on B200, exact with the reference
// (pruning.py:37-64): zero the k = floor(sparsity * n) entries with the
// lowest score cm[c] * |q[r,c]| (f64), ties broken by flat row-major index
// (np.argsort kind="stable").  No sort is needed:
//   per tensor: scores take at most cols * 129 distinct values, so one pass
//     builds the (column, |q|) histogram; a radix select over those weighted
//     keys (20 bits grid-wide, the rest over the few candidates left) finds
//     the k-th smallest score T and how many ties r must go; the ties live
//     only in the columns where some |q| scores exactly T, so the flat index
//     of the r-th tie (row-major) is found by scanning just those columns;
//     a streaming pass then zeroes score < T and the ties up to that index.
//   per row: one CTA per row, 8 x 8-bit radix select in shared memory and
//     the same ordered tie pass.
// Non-negative doubles order like their u64 bit patterns, so keys are bits.
#include <cooperative_groups.h>
#include <cstdio>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace dc {

constexpr int kPrThreads = 256;
constexpr int kBins = 129;  // |q| in 0..128

constexpr int kSelThreads = 512;
constexpr int kSelHBins = 4096;  // 12-bit digit passes (two), in shared memory

struct SelectOut {
    unsigned long long T;         // the k-th smallest score's bits
    unsigned long long kk;        // ties (score == T) to zero, the first kk in row-major order
    unsigned long long eq_total;  // elements with score == T
    unsigned long long cut;       // flat index of the last tie to zero (~0: every tie goes)
    uint32_t n_cand, n_eqc, bin, pad;
};

__device__ __forceinline__ unsigned long long key_of(double cm, int a) {
    return (unsigned long long)__double_as_longlong(__dmul_rn(cm, (double)a));
}

__device__ __forceinline__ int absq(int8_t v) { return v < 0 ? -(int)v : (int)v; }

// ------------------------------------------------------------ per tensor
// (column, |q|) histogram, conflict-free: a CTA covers 128 columns, each warp
// one row per step with lane L loading the 4 bytes of columns 4L..4L+3; the
// shared bins are laid out [|q|][e][lane] so the atomic for byte e of every
// lane lands in bank L whatever the |q| values (the round-1 column-major bins
// took random-bank conflicts and same-address collisions: ~2.5x slower).
// Row blocks (<= 65535 rows, so u16 counts) write partial histograms in the
// same layout; k_colhist4_sum adds them up.
constexpr int kH4Cols = 128;
constexpr int kH4Threads = 512;
constexpr int kH4Unr = 8;
constexpr int kH4Words = kBins * kH4Cols;  // [a][e][lane]
constexpr int kH4Smem = kH4Words * 4;

__global__ void __launch_bounds__(kH4Threads, 3) k_colhist4(const int8_t* __restrict__ q, int64_t rows, int64_t cols,
                                                             int64_t rows_per, bool vec4,
                                                             uint16_t* __restrict__ partial) {
    extern __shared__ __align__(16) uint32_t hb[];
    for (int i = threadIdx.x; i < kH4Words / 4; i += blockDim.x) reinterpret_cast<uint4*>(hb)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = kH4Threads / 32;
    const int64_t c0 = (int64_t)blockIdx.y * kH4Cols + lane * 4;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = min(rows, r0 + rows_per);
    uint32_t* hl = hb + lane;
#ifdef DC_PRUNE_NOATOMS
    uint32_t sink = 0;
#endif
    if (vec4) {  // cols % 4 == 0, q 4-byte aligned
        if (c0 < cols) {
            const int8_t* p = q + c0;
            for (int64_t r = r0 + warp; r < r1; r += nwarp * kH4Unr) {
                uint32_t w[kH4Unr];
#pragma unroll
                for (int u = 0; u < kH4Unr; ++u) {
                    const int64_t rr = r + u * nwarp;
                    w[u] = rr < r1 ? __ldg(reinterpret_cast<const uint32_t*>(p + rr * cols)) : 0u;
                }
#pragma unroll
                for (int u = 0; u < kH4Unr; ++u) {
                    if (r + u * nwarp >= r1) break;
                    const uint32_t a4 = __vabs4(w[u]);  // 0x80 -> 128 (unsigned)
#ifdef DC_PRUNE_NOATOMS
                    sink += a4;
#else
#pragma unroll
                    for (int e = 0; e < 4; ++e) atomicAdd(hl + ((a4 >> (8 * e)) & 0xFFu) * kH4Cols + e * 32, 1u);
#endif
                }
            }
        }
    } else {
        for (int64_t r = r0 + warp; r < r1; r += nwarp)
            for (int e = 0; e < 4; ++e)
                if (c0 + e < cols) atomicAdd(hl + absq(q[r * cols + c0 + e]) * kH4Cols + e * 32, 1u);
    }
#ifdef DC_PRUNE_NOATOMS
    hl[0] += sink;
#endif
    __syncthreads();
    uint32_t* out = reinterpret_cast<uint32_t*>(partial + ((int64_t)blockIdx.x * gridDim.y + blockIdx.y) * kH4Words);
    for (int i = threadIdx.x; i < kH4Words / 2; i += blockDim.x) {
        const uint2 v = reinterpret_cast<const uint2*>(hb)[i];
        out[i] = v.x | (v.y << 16);
    }
}

// Same with 16-byte loads: lane L holds columns 16L..16L+15 of a row (a warp
// reads 512 contiguous bytes), counters are u16 pairs (even / odd column of
// the lane's 16) in words laid out [|q|][e / 2][lane]: still bank L for every
// lane, 132 KB of shared bins for 512 columns, one CTA of 32 warps per SM.
constexpr int kH5Cols = 512;
constexpr int kH5Threads = 1024;
constexpr int kH5Unr = 4;
constexpr int kH5Words = kBins * kH5Cols / 2;  // [a][e/2 (8)][lane (32)], u16 pairs
constexpr int kH5Smem = kH5Words * 4;

__global__ void __launch_bounds__(kH5Threads, 1) k_colhist5(const int8_t* __restrict__ q, int64_t rows, int64_t cols,
                                                             int64_t rows_per, uint32_t* __restrict__ partial) {
    extern __shared__ __align__(16) uint32_t hb[];
    for (int i = threadIdx.x; i < kH5Words / 4; i += blockDim.x) reinterpret_cast<uint4*>(hb)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = kH5Threads / 32;
    const int64_t c0 = (int64_t)blockIdx.y * kH5Cols + lane * 16;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = min(rows, r0 + rows_per);
    uint32_t* hl = hb + lane;
#ifdef DC_PRUNE_NOATOMS
    uint32_t sink = 0;
#endif
    if (c0 < cols) {  // cols % 16 == 0, q 16-byte aligned (caller)
        const int8_t* p = q + c0;
        for (int64_t r = r0 + warp; r < r1; r += nwarp * kH5Unr) {
            uint4 v[kH5Unr];
#pragma unroll
            for (int u = 0; u < kH5Unr; ++u) {
                const int64_t rr = r + u * nwarp;
                v[u] = rr < r1 ? __ldcs(reinterpret_cast<const uint4*>(p + rr * cols)) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < kH5Unr; ++u) {
                if (r + u * nwarp >= r1) break;
                const uint32_t w[4] = {__vabs4(v[u].x), __vabs4(v[u].y), __vabs4(v[u].z), __vabs4(v[u].w)};
#ifdef DC_PRUNE_NOATOMS
                sink += w[0] + w[1] + w[2] + w[3];
#else
#pragma unroll
                for (int e = 0; e < 16; ++e)
                    atomicAdd(hl + ((w[e >> 2] >> (8 * (e & 3))) & 0xFFu) * (kH5Cols / 2) + (e >> 1) * 32,
                              (e & 1) ? 0x10000u : 1u);
#endif
            }
        }
    }
#ifdef DC_PRUNE_NOATOMS
    hl[0] += sink & 1;
#endif
    __syncthreads();
    uint4* out = reinterpret_cast<uint4*>(partial + ((int64_t)blockIdx.x * gridDim.y + blockIdx.y) * kH5Words);
    for (int i = threadIdx.x; i < kH5Words / 4; i += blockDim.x) out[i] = reinterpret_cast<const uint4*>(hb)[i];
}

// counts[c * 129 + a] from the k_colhist5 partials (u16 pairs)
__global__ void k_colhist5_sum(const uint32_t* __restrict__ partial, int64_t n_rb, int64_t n_cb, int64_t cols,
                               uint32_t* __restrict__ counts, uint32_t* __restrict__ hist,
                               uint32_t* __restrict__ eqmask, SelectOut* __restrict__ so) {
    const int64_t per_rb = n_cb * kH5Words;
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = gt; i < per_rb; i += gs) {
        const uint32_t cb = (uint32_t)(i / kH5Words), rem = (uint32_t)(i - (int64_t)cb * kH5Words);
        const uint32_t a = rem / (kH5Cols / 2), slot = rem % (kH5Cols / 2);  // slot = (e/2) * 32 + lane
        const int64_t c = (int64_t)cb * kH5Cols + (slot & 31) * 16 + (slot >> 5) * 2;
        uint32_t s0 = 0, s1 = 0;
        for (int64_t rb = 0; rb < n_rb; rb += 8) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = rb + u < n_rb ? partial[(rb + u) * per_rb + i] : 0u;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                s0 += v[u] & 0xFFFFu;
                s1 += v[u] >> 16;
            }
        }
        if (c < cols) counts[c * kBins + a] = s0;
        if (c + 1 < cols) counts[(c + 1) * kBins + a] = s1;
    }
    for (int64_t i = gt; i < 2 * kSelHBins / 4; i += gs) reinterpret_cast<uint4*>(hist)[i] = make_uint4(0, 0, 0, 0);
    for (int64_t i = gt; i < (cols + 31) / 32; i += gs) eqmask[i] = 0;
    if (gt == 0) so->n_cand = 0;
}

// counts[c * 129 + a] = sum over row blocks of the k_colhist4 partials (read
// in their layout, coalesced; n_rb loads in flight); also zeroes k_select4's
// histograms, tie-column bits and candidate counter.
__global__ void k_colhist4_sum(const uint16_t* __restrict__ partial, int64_t n_rb, int64_t n_cb, int64_t cols,
                               uint32_t* __restrict__ counts, uint32_t* __restrict__ hist,
                               uint32_t* __restrict__ eqmask, SelectOut* __restrict__ so) {
    const int64_t per_rb = n_cb * kH4Words;
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = gt; i < per_rb; i += gs) {
        const uint32_t cb = (uint32_t)(i / kH4Words), rem = (uint32_t)(i - (int64_t)cb * kH4Words);
        const uint32_t a = rem / kH4Cols, slot = rem % kH4Cols;
        const int64_t c = (int64_t)cb * kH4Cols + (slot & 31) * 4 + (slot >> 5);
        uint32_t s = 0;
        for (int64_t rb = 0; rb < n_rb; rb += 8) {
            uint32_t v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = rb + u < n_rb ? partial[(rb + u) * per_rb + i] : 0u;
#pragma unroll
            for (int u = 0; u < 8; ++u) s += v[u];
        }
        if (c < cols) counts[c * kBins + a] = s;
    }
    for (int64_t i = gt; i < 2 * kSelHBins / 4; i += gs) reinterpret_cast<uint4*>(hist)[i] = make_uint4(0, 0, 0, 0);
    for (int64_t i = gt; i < (cols + 31) / 32; i += gs) eqmask[i] = 0;
    if (gt == 0) so->n_cand = 0;
}

// The whole k-th-score selection and the tie cut in ONE cooperative launch
// (grid = SMs, 4 grid barriers, 6 when only some ties stay):
//   A  every CTA: histogram of the top 12 key bits (sign + exponent) of its
//      (column, |q|) items in shared memory, flushed with one global atomic
//      per non-empty bin; every CTA then picks the bin holding rank k;
//   A2 the same for the next 12 bits, over the items inside that exponent
//      (global atomics on a few thousand hot bins of a flat 2^20-bin table
//      were 20 us of L2 atomic serialization);
//   D  every CTA appends the items whose top 24 key bits match to a list;
//   E  every CTA redundantly: the k-th key among those (few) candidates by
//      direct rank comparison in shared memory (8-bit radix passes from L2
//      when there are many) -> T, the ties to zero (kk), the entries == T;
//   F  every CTA, its own column slice: |q| bounds of score < T and score ==
//      T by binary search (keys are nondecreasing in |q|) and a bit per
//      column holding ties;
//   G/H only when some ties stay: ties (only in those columns) counted per
//      CTA over row ranges; the CTA holding the kk-th tie in row-major order
//      records its flat index as the cut.
// Loops over global data batch their loads (the serial L2 round trips of a
// plain loop dominated).  Replaces a 4 x 16-bit grid-wide radix select (12
// grid barriers) and the look-back tie scan of the round-1 apply pass.
// rank-k entry of v[0..m) for any m: thread t sums a contiguous run of
// ceil(m / blockDim) entries (independent loads), one block scan picks the run,
// its owner walks it.  Returns the index; `base` becomes the count before it.
__device__ int block_find_all(const uint32_t* v, bool gmem, int m, unsigned long long k, unsigned long long& base,
                              int* s_idx, unsigned long long* s_before, unsigned long long* wsum) {
    const int per = (m + blockDim.x - 1) / blockDim.x;
    const int j0 = threadIdx.x * per, j1 = min(m, j0 + per);
    auto ld = [&](int j) -> uint32_t { return j < j1 ? (gmem ? __ldcg(v + j) : v[j]) : 0u; };
    unsigned long long x = 0;
    for (int j = j0; j < j1; j += 8) {  // 8 independent loads in flight
        uint32_t e[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) e[u] = ld(j + u);
#pragma unroll
        for (int u = 0; u < 8; ++u) x += e[u];
    }
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    unsigned long long inc = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    if (t == 0) *s_idx = m - 1;  // unreachable for 1 <= k <= total
    if (lane == 31) wsum[w] = inc;
    __syncthreads();
    unsigned long long before = base;
    for (int i = 0; i < w; ++i) before += wsum[i];
    inc += before;
    if (j0 < j1 && inc - x < k && k <= inc) {
        unsigned long long c = inc - x;
        bool found = false;
        for (int j = j0; j < j1 && !found; j += 8) {
            uint32_t e[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) e[u] = ld(j + u);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (!found && j + u < j1 && k <= c + e[u]) {
                    *s_idx = j + u;
                    *s_before = c;
                    found = true;
                }
                c += e[u];
            }
        }
    }
    __syncthreads();
    const int idx = *s_idx;
    base = *s_before;
    __syncthreads();
    return idx;
}

// exclusive prefix of a 0/1 flag over the CTA (in thread order) + total
__device__ __forceinline__ uint32_t block_excl(bool f, uint32_t* wcnt, uint32_t& total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) wcnt[w] = __popc(m);
    __syncthreads();
    uint32_t before = 0, tot = 0;
    for (int i = 0; i < (int)blockDim.x / 32; ++i) {
        before += i < w ? wcnt[i] : 0u;
        tot += wcnt[i];
    }
    __syncthreads();
    total = tot;
    return before + __popc(m & ((1u << lane) - 1u));
}

constexpr int kCandCap = 1024;  // candidates cached in shared memory (else re-read from L2)
constexpr int kEqCap = 4096;    // tie columns listed in shared memory (else whole rows are scanned)
constexpr int kUnr = 8;

__global__ void __launch_bounds__(kSelThreads) k_select4(const uint32_t* __restrict__ counts,
                                                         const double* __restrict__ cm, const int8_t* __restrict__ q,
                                                         int64_t rows, int64_t cols, unsigned long long k,
                                                         SelectOut* __restrict__ so, uint32_t* __restrict__ hist,
                                                         uint32_t* __restrict__ psum, uint32_t* __restrict__ cand,
                                                         uint32_t* __restrict__ eqmask, uint8_t* __restrict__ bound,
                                                         uint8_t* __restrict__ lo, uint8_t* __restrict__ hi) {
    // hist (2 x 4096 u32), eqmask and so->n_cand are zeroed by k_colhist4_sum
    cg::grid_group grid = cg::this_grid();
    const int64_t n = cols * kBins;
    const int lane = threadIdx.x & 31;
    __shared__ unsigned long long wsum[kSelThreads / 32], s_before;
    __shared__ uint32_t wcnt[kSelThreads / 32], h[256], hs[kSelHBins];
    __shared__ int s_idx;
    __shared__ __align__(16) unsigned char pool[kCandCap * 12 > kEqCap * 4 ? kCandCap * 12 : kEqCap * 4];
    auto* ckey = reinterpret_cast<unsigned long long*>(pool);
    auto* ccnt = reinterpret_cast<uint32_t*>(pool + kCandCap * 8);
    auto* elist = reinterpret_cast<uint32_t*>(pool);
#ifdef DC_PRUNE_TIMING
    unsigned long long tm[12];
    int ntm = 0;
#define TMARK() do { if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm[ntm++])); } while (0)
#else
#define TMARK() do {} while (0)
#endif
    TMARK();
    const int64_t per = (n + gridDim.x - 1) / gridDim.x;  // contiguous items per CTA (A and D)
    const int64_t i0 = (int64_t)blockIdx.x * per, i1 = min(n, i0 + per);
    auto item_key = [&](uint32_t i) {
        const uint32_t col = i / (uint32_t)kBins;
        return key_of(cm[col], (int)(i - col * (uint32_t)kBins));
    };
    // ---- A: (sign, exponent) histogram in shared memory, flushed to hist[0..4096)
    for (int j = threadIdx.x; j < kSelHBins; j += blockDim.x) hs[j] = 0;
    __syncthreads();
    auto hist_pass = [&](int pass, uint32_t want) {
        for (int64_t ib = i0 + threadIdx.x; ib < i1; ib += kUnr * blockDim.x) {
            uint32_t c[kUnr];
#pragma unroll
            for (int u = 0; u < kUnr; ++u) {
                const int64_t i = ib + (int64_t)u * blockDim.x;
                c[u] = i < i1 ? counts[i] : 0u;
            }
#pragma unroll
            for (int u = 0; u < kUnr; ++u) {
                if (!c[u]) continue;
                const unsigned long long key = item_key((uint32_t)(ib + (int64_t)u * blockDim.x));
                if (pass == 0)
                    atomicAdd(&hs[key >> 52], c[u]);
                else if ((uint32_t)(key >> 52) == want)
                    atomicAdd(&hs[(key >> 40) & 0xFFF], c[u]);
            }
        }
        __syncthreads();
        uint32_t* g = hist + pass * kSelHBins;
        for (int j = threadIdx.x; j < kSelHBins; j += blockDim.x) {
            const uint32_t v = hs[j];
            if (v) atomicAdd(g + j, v);
            hs[j] = 0;
        }
    };
    hist_pass(0, 0);
    TMARK();
    grid.sync();
    unsigned long long base = 0;
    const uint32_t e0 = (uint32_t)block_find_all(hist, true, kSelHBins, k, base, &s_idx, &s_before, wsum);
    // ---- A2: the next 12 bits inside that exponent
    hist_pass(1, e0);
    TMARK();
    grid.sync();
    const uint32_t bin = (e0 << 12) |
                         (uint32_t)block_find_all(hist + kSelHBins, true, kSelHBins, k, base, &s_idx, &s_before, wsum);
    TMARK();
    // ---- D: candidates = items whose top 24 key bits are `bin`
    for (int64_t ib = i0; ib < i1; ib += kUnr * blockDim.x) {
        uint32_t c[kUnr];
#pragma unroll
        for (int u = 0; u < kUnr; ++u) {
            const int64_t i = ib + (int64_t)u * blockDim.x + threadIdx.x;
            c[u] = i < i1 ? counts[i] : 0u;
        }
#pragma unroll
        for (int u = 0; u < kUnr; ++u) {
            const int64_t i = ib + (int64_t)u * blockDim.x + threadIdx.x;
            const bool f = c[u] && (item_key((uint32_t)i) >> 40) == bin;
            const uint32_t m = __ballot_sync(0xffffffffu, f);
            if (m) {
                uint32_t pos = 0;
                if (lane == 0) pos = atomicAdd(&so->n_cand, (uint32_t)__popc(m));
                pos = __shfl_sync(0xffffffffu, pos, 0);
                if (f) cand[pos + __popc(m & ((1u << lane) - 1u))] = (uint32_t)i;
            }
        }
    }
    TMARK();
    grid.sync();
    // ---- E (every CTA, same answer): the k-th key among the candidates
    const uint32_t nc = __ldcg(&so->n_cand);
    unsigned long long kk = k - base, T;
    uint32_t eq_total = 0;
    if (nc <= (uint32_t)kCandCap) {
        // cached: each candidate's rank range [below, below + eq) by direct
        // comparison with all others (nc is small: 24 key bits are fixed)
        __shared__ unsigned long long s_T, s_kk;
        __shared__ uint32_t s_eq;
        for (uint32_t j = threadIdx.x; j < nc; j += blockDim.x) {
            const uint32_t i = __ldcg(cand + j);
            ckey[j] = item_key(i);
            ccnt[j] = counts[i];
        }
        __syncthreads();
        for (uint32_t j = threadIdx.x; j < nc; j += blockDim.x) {
            const unsigned long long kj = ckey[j];
            unsigned long long below = 0;
            uint32_t eq = 0;
            for (uint32_t i = 0; i < nc; ++i) {
                const unsigned long long ki = ckey[i];
                const uint32_t ci = ccnt[i];
                below += ki < kj ? ci : 0u;
                eq += ki == kj ? ci : 0u;
            }
            if (below < kk && kk <= below + eq) {  // every candidate with key T writes the same values
                s_T = kj;
                s_kk = kk - below;
                s_eq = eq;
            }
        }
        __syncthreads();
        T = s_T;
        kk = s_kk;
        eq_total = s_eq;
        __syncthreads();
    } else {  // many candidates: 8-bit radix passes over the other 40 bits, from L2
        unsigned long long prefix = bin;
        for (int shift = 32; shift >= 0; shift -= 8) {
            for (int j = threadIdx.x; j < 256; j += blockDim.x) h[j] = 0;
            __syncthreads();
            for (uint32_t j = threadIdx.x; j < nc; j += blockDim.x) {
                const uint32_t i = __ldcg(cand + j);
                const unsigned long long key = item_key(i);
                if ((key >> (shift + 8)) == prefix) atomicAdd(&h[(key >> shift) & 0xFFu], counts[i]);
            }
            __syncthreads();
            unsigned long long b2 = 0;
            const int d = block_find_all(h, false, 256, kk, b2, &s_idx, &s_before, wsum);
            prefix = (prefix << 8) | (unsigned long long)d;
            kk -= b2;
            eq_total = h[d];
            __syncthreads();
        }
        T = prefix;
    }
    const bool all_ties = kk == eq_total;
    TMARK();
    // ---- F: bounds of this CTA's columns (lo = #|q| with score < T, hi = ... <= T)
    {
        const int64_t cper = (cols + gridDim.x - 1) / gridDim.x;
        const int64_t c1 = min(cols, ((int64_t)blockIdx.x + 1) * cper);
        for (int64_t c = (int64_t)blockIdx.x * cper + threadIdx.x; c < c1; c += blockDim.x) {
            const double w = cm[c];
            int a = 0, b = kBins;  // first a with key >= T
            while (a < b) {
                const int mid = (a + b) >> 1;
                if (key_of(w, mid) < T) a = mid + 1; else b = mid;
            }
            const int l = a;
            b = kBins;  // first a with key > T
            while (a < b) {
                const int mid = (a + b) >> 1;
                if (key_of(w, mid) <= T) a = mid + 1; else b = mid;
            }
            lo[c] = (uint8_t)l;
            hi[c] = (uint8_t)a;
            bound[c] = (uint8_t)(all_ties ? a : l);
            if (l < a) atomicOr(&eqmask[c >> 5], 1u << (c & 31));
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            so->T = T;
            so->kk = kk;
            so->eq_total = eq_total;
            so->bin = bin;
            so->cut = all_ties ? ~0ull : 0ull;
        }
    }
    TMARK();
#ifdef DC_PRUNE_TIMING
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        printf("select4 nc=%u all_ties=%d:", nc, (int)all_ties);
        for (int i = 1; i < ntm; ++i) printf(" %.2f", (tm[i] - tm[i - 1]) * 1e-3);
        printf(" us\n");
    }
#endif
    if (all_ties) return;  // grid-uniform; k_apply4 runs after this launch
    grid.sync();
    TMARK();
    // ---- G: the tie columns in ascending order (shared list), ties per CTA
    const int nw = (int)((cols + 31) >> 5);
    uint32_t E;
    {
        const int per_w = (nw + blockDim.x - 1) / blockDim.x;
        const int w0 = threadIdx.x * per_w, w1 = min(nw, w0 + per_w);
        uint32_t c = 0;
        for (int j = w0; j < w1; ++j) c += __popc(__ldcg(eqmask + j));
        uint32_t inc = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += o;
        }
        if (lane == 31) wcnt[threadIdx.x >> 5] = inc;
        __syncthreads();
        uint32_t before = 0, tot = 0;
        for (int i = 0; i < kSelThreads / 32; ++i) {
            before += i < (int)(threadIdx.x >> 5) ? wcnt[i] : 0u;
            tot += wcnt[i];
        }
        E = tot;
        if (E <= (uint32_t)kEqCap) {
            uint32_t pos = before + inc - c;
            for (int j = w0; j < w1; ++j)
                for (uint32_t m = __ldcg(eqmask + j); m; m &= m - 1) elist[pos++] = (uint32_t)j * 32 + __ffs(m) - 1;
        }
        __syncthreads();
    }
    const bool listed = E <= (uint32_t)kEqCap;
    const uint32_t width = listed ? E : (uint32_t)cols;  // unlisted: whole rows (non-tie columns never match)
    const int64_t rper = (rows + gridDim.x - 1) / gridDim.x;
    const int64_t r0 = min(rows, (int64_t)blockIdx.x * rper), r1 = min(rows, r0 + rper);
    const uint32_t np = (uint32_t)((r1 - r0) * (int64_t)width);
    auto tie_at = [&](uint32_t p, int64_t& idx) -> bool {
        const uint32_t rr = p / width, j = p - rr * width;
        const uint32_t c = listed ? elist[j] : j;
        idx = (r0 + rr) * cols + c;
        const int a = absq(q[idx]);
        return a >= __ldcg(lo + c) && a < __ldcg(hi + c);
    };
    {
        uint32_t cnt = 0;
        for (uint32_t pb = threadIdx.x; pb < np; pb += kUnr * blockDim.x) {
#pragma unroll
            for (int u = 0; u < kUnr; ++u) {
                const uint32_t p = pb + u * blockDim.x;
                int64_t idx;
                if (p < np) cnt += tie_at(p, idx);
            }
        }
        cnt = __reduce_add_sync(0xffffffffu, cnt);
        if (lane == 0) wcnt[threadIdx.x >> 5] = cnt;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (int j = 0; j < kSelThreads / 32; ++j) t += wcnt[j];
            psum[blockIdx.x] = t;
        }
    }
    TMARK();
    grid.sync();
    TMARK();
    // ---- H: the CTA holding the kk-th tie finds its flat index
    unsigned long long before = 0;
    {
        uint32_t v = 0;  // ties before this CTA's rows (parallel loads, block sum)
        for (int j = threadIdx.x; j < (int)blockIdx.x; j += blockDim.x) v += __ldcg(psum + j);
        v = __reduce_add_sync(0xffffffffu, v);
        __syncthreads();
        if (lane == 0) wcnt[threadIdx.x >> 5] = v;
        __syncthreads();
        for (int j = 0; j < kSelThreads / 32; ++j) before += wcnt[j];
        __syncthreads();
    }
    const unsigned long long mine = __ldcg(psum + blockIdx.x);
    if (!(before < kk && kk <= before + mine)) return;
    for (uint32_t pb = 0; pb < np; pb += blockDim.x) {
        const uint32_t p = pb + threadIdx.x;
        int64_t idx = 0;
        const bool t = p < np && tie_at(p, idx);
        uint32_t tot;
        const uint32_t r = block_excl(t, wcnt, tot);
        if (t && before + r + 1 == kk) so->cut = (unsigned long long)idx;
        before += tot;
        if (before >= kk) break;  // block-uniform
    }
#ifdef DC_PRUNE_TIMING
    TMARK();
    if (threadIdx.x == 0) {
        printf("select4 G/H (CTA %d holds the cut):", (int)blockIdx.x);
        for (int i = 1; i < ntm; ++i) printf(" %.2f", (tm[i] - tm[i - 1]) * 1e-3);
        printf(" us\n");
    }
#endif
}

// out = q with |q| < bound[c] zeroed, and the ties (bound <= |q| in [lo, hi))
// at flat index <= cut: one streaming pass, 16 B per thread step, four in flight.
constexpr int kApThreads = 256, kApVec = 4;

__device__ __forceinline__ uint32_t zero_mask4(uint32_t qw, uint32_t bw, uint32_t lw, uint32_t hw, uint32_t cw) {
    const uint32_t a = __vabs4(qw);
    const uint32_t lt = __vcmpltu4(a, bw);
    const uint32_t tie = __vcmpltu4(a, hw) & ~__vcmpltu4(a, lw) & cw;
    return qw & ~(lt | tie);
}

__global__ void __launch_bounds__(kApThreads) k_apply4(const int8_t* __restrict__ q, const uint8_t* __restrict__ bound,
                                                       const uint8_t* __restrict__ lo, const uint8_t* __restrict__ hi,
                                                       int64_t n, int64_t cols, bool vec,
                                                       const SelectOut* __restrict__ so, int8_t* __restrict__ out) {
    const unsigned long long cut = so->cut;
    const int64_t stride = (int64_t)gridDim.x * kApThreads * 16 * kApVec;
    if (vec) {  // cols % 16 == 0, 16-B aligned: each vector lies in one row
        for (int64_t base = ((int64_t)blockIdx.x * kApThreads * kApVec + threadIdx.x) * 16; base < n; base += stride) {
            uint4 v[kApVec];
#pragma unroll
            for (int u = 0; u < kApVec; ++u) {
                const int64_t i0 = base + (int64_t)u * kApThreads * 16;
                v[u] = i0 < n ? __ldcs(reinterpret_cast<const uint4*>(q + i0)) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < kApVec; ++u) {
                const int64_t i0 = base + (int64_t)u * kApThreads * 16;
                if (i0 >= n) break;
                const uint32_t c0 = (uint32_t)((uint64_t)i0 % (uint64_t)cols);
                const uint4 b = *reinterpret_cast<const uint4*>(bound + c0);
                const uint4 l = *reinterpret_cast<const uint4*>(lo + c0);
                const uint4 h = *reinterpret_cast<const uint4*>(hi + c0);
                // ties at index <= cut: byte j of word w is element 4w + j
                uint32_t cw[4];
                const long long ck = (long long)cut - i0;  // cut = ~0: every tie (ck < 0 as signed, handled)
                if (cut == ~0ull || ck >= 15) {
                    cw[0] = cw[1] = cw[2] = cw[3] = 0xFFFFFFFFu;
                } else if (ck < 0) {
                    cw[0] = cw[1] = cw[2] = cw[3] = 0u;
                } else {
#pragma unroll
                    for (int w = 0; w < 4; ++w)
                        cw[w] = __vcmpleu4(0x03020100u + 0x04040404u * w, 0x01010101u * (uint32_t)ck);
                }
                uint4 o;
                o.x = zero_mask4(v[u].x, b.x, l.x, h.x, cw[0]);
                o.y = zero_mask4(v[u].y, b.y, l.y, h.y, cw[1]);
                o.z = zero_mask4(v[u].z, b.z, l.z, h.z, cw[2]);
                o.w = zero_mask4(v[u].w, b.w, l.w, h.w, cw[3]);
                __stcs(reinterpret_cast<uint4*>(out + i0), o);
            }
        }
        return;
    }
    for (int64_t i = (int64_t)blockIdx.x * kApThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kApThreads) {
        const int64_t c = i % cols;
        const int8_t v = q[i];
        const int a = absq(v);
        const bool z = a < bound[c] || (a >= lo[c] && a < hi[c] && (cut == ~0ull || (unsigned long long)i <= cut));
        out[i] = z ? (int8_t)0 : v;
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

static int64_t colhist4_rb(int64_t rows, int64_t cols) {
    const int64_t n_cb = (cols + kH4Cols - 1) / kH4Cols;
    int64_t n_rb = 3 * (int64_t)sm_count_pr() / n_cb;  // 3 CTAs per SM, one wave
    n_rb = n_rb < 1 ? 1 : (n_rb > 64 ? 64 : n_rb);
    if (n_rb > rows) n_rb = rows > 0 ? rows : 1;
    const int64_t need = (rows + 65534) / 65535;  // u16 partial counts
    return n_rb < need ? need : n_rb;
}

static int64_t colhist5_rb(int64_t rows, int64_t cols) {
    const int64_t n_cb = (cols + kH5Cols - 1) / kH5Cols;
    int64_t n_rb = (int64_t)sm_count_pr() / n_cb;  // one CTA per SM, one wave
    n_rb = n_rb < 1 ? 1 : (n_rb > 64 ? 64 : n_rb);
    if (n_rb > rows) n_rb = rows > 0 ? rows : 1;
    const int64_t need = (rows + 65534) / 65535;  // u16 partial counts
    return n_rb < need ? need : n_rb;
}

extern "C" int dc_prune_scratch_bytes(int64_t rows, int64_t cols, uint64_t* out) {
    const uint64_t n_cb = (uint64_t)((cols + kH4Cols - 1) / kH4Cols);
    const uint64_t items = (uint64_t)cols * kBins;
    *out = 8ull * kSelHBins + 256 + 4ull * 4096 + 256 + sizeof(SelectOut) + 256 + 4ull * items + 256 + 4ull * cols +
           256 + 4ull * items + 256 + 3ull * (uint64_t)cols + 256 +
           2ull * kH4Words * n_cb * (uint64_t)colhist4_rb(rows, cols) +
           4ull * kH5Words * (uint64_t)((cols + kH5Cols - 1) / kH5Cols) * (uint64_t)colhist5_rb(rows, cols) + 256;
    return DC_OK;
}

// Per tensor: (column, |q|) histogram (+ sum) -> one cooperative selection
// launch -> one streaming apply pass (4 launches, was 20 in round 1).
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
    const int64_t items = cols * kBins;
    uint8_t* p = align(scratch);
    auto* hist = reinterpret_cast<uint32_t*>(p);
    p = align(p + 8ull * kSelHBins);
    auto* psum = reinterpret_cast<uint32_t*>(p);
    p = align(p + 4ull * 4096);
    auto* so = reinterpret_cast<SelectOut*>(p);
    p = align(p + sizeof(SelectOut));
    auto* cand = reinterpret_cast<uint32_t*>(p);
    p = align(p + 4ull * items);
    auto* eqmask = reinterpret_cast<uint32_t*>(p);
    p = align(p + 4ull * ((cols + 31) / 32));
    auto* counts = reinterpret_cast<uint32_t*>(p);
    p = align(p + 4ull * items);
    uint8_t* bound = p;
    uint8_t* lo = p + cols;
    uint8_t* hi = p + 2 * cols;
    p = align(p + 3ull * cols);
    auto* partial = reinterpret_cast<uint16_t*>(p);
    const bool vec = cols % 16 == 0 && (reinterpret_cast<uintptr_t>(q) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(out) & 15) == 0;

    if (vec) {  // 16-B path
        const int64_t n_cb = (cols + kH5Cols - 1) / kH5Cols;
        int64_t n_rb = colhist5_rb(rows, cols);
        const int64_t rows_per = (rows + n_rb - 1) / n_rb;
        n_rb = (rows + rows_per - 1) / rows_per;
        static bool attr5 = false;
        if (!attr5) {
            cudaFuncSetAttribute(k_colhist5, cudaFuncAttributeMaxDynamicSharedMemorySize, kH5Smem);
            attr5 = true;
        }
        auto* part = reinterpret_cast<uint32_t*>(partial);
        k_colhist5<<<dim3((unsigned)n_rb, (unsigned)n_cb), kH5Threads, kH5Smem, st>>>(q, rows, cols, rows_per, part);
        DC_CHECK_LAUNCH("k_colhist5");
        k_colhist5_sum<<<(unsigned)(sm_count_pr() * 8), 256, 0, st>>>(part, n_rb, n_cb, cols, counts, hist, eqmask,
                                                                       so);
        DC_CHECK_LAUNCH("k_colhist5_sum");
    } else {
        const int64_t n_cb = (cols + kH4Cols - 1) / kH4Cols;
        int64_t n_rb = colhist4_rb(rows, cols);
        const int64_t rows_per = (rows + n_rb - 1) / n_rb;
        n_rb = (rows + rows_per - 1) / rows_per;
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_colhist4, cudaFuncAttributeMaxDynamicSharedMemorySize, kH4Smem);
            attr = true;
        }
        const bool vec4 = cols % 4 == 0 && (reinterpret_cast<uintptr_t>(q) & 3) == 0;
        k_colhist4<<<dim3((unsigned)n_rb, (unsigned)n_cb), kH4Threads, kH4Smem, st>>>(q, rows, cols, rows_per, vec4,
                                                                                      partial);
        DC_CHECK_LAUNCH("k_colhist4");
        k_colhist4_sum<<<(unsigned)(sm_count_pr() * 8), 256, 0, st>>>(partial, n_rb, n_cb, cols, counts, hist, eqmask,
                                                                       so);
        DC_CHECK_LAUNCH("k_colhist4_sum");
    }
    {  // the k-th score, the per-column bounds and the tie cut: one cooperative launch
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_select4, kSelThreads, 0);
        if (per_sm < 1) {
            set_error_msg("k_select4: not resident");
            return DC_ERR_CUDA;
        }
        int grid = sm_count_pr();
        if (grid > 4096) grid = 4096;  // psum slots
        unsigned long long kk = (unsigned long long)k;
        void* args[] = {(void*)&counts, (void*)&cm, (void*)&q, (void*)&rows, (void*)&cols, (void*)&kk, (void*)&so,
                        (void*)&hist, (void*)&psum, (void*)&cand, (void*)&eqmask, (void*)&bound, (void*)&lo, (void*)&hi};
        cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_select4, dim3((unsigned)grid), dim3(kSelThreads),
                                                    args, 0, st);
        if (e != cudaSuccess) {
            set_error("k_select4", e);
            return DC_ERR_CUDA;
        }
    }
    const int64_t want = (n + (int64_t)kApThreads * 16 * kApVec - 1) / ((int64_t)kApThreads * 16 * kApVec);
    const int64_t cap = (int64_t)sm_count_pr() * 8;
    const int64_t g = vec ? (want < cap ? want : cap) : cap;
    k_apply4<<<(unsigned)g, kApThreads, 0, st>>>(q, bound, lo, hi, n, cols, vec, so, out);
    DC_CHECK_LAUNCH("k_apply4");
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
