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
constexpr int kSelHBins = 4096;  // selection histogram bins (shared memory)

struct SelectOut {
    unsigned long long T;         // the k-th smallest score's bits
    unsigned long long kk;        // ties (score == T) to zero, the first kk in row-major order
    unsigned long long eq_total;  // elements with score == T
    unsigned long long cut;       // flat index of the last tie to zero (~0: every tie goes)
    unsigned long long kmin;      // key of the smallest positive score (min cm > 0, |q| = 1); ~0 if none
    unsigned long long kmax;      // key bound of the largest score (max cm, |q| = 128)
    uint32_t n_cand, n_eqc, bin, pad;
};

__device__ __forceinline__ unsigned long long key_of(double cm, int a) {
    return (unsigned long long)__double_as_longlong(__dmul_rn(cm, (double)a));
}

__device__ __forceinline__ int absq(int8_t v) { return v < 0 ? -(int)v : (int)v; }

// ------------------------------------------------------------ per tensor
// (column, |q|) histogram, conflict-free: a CTA covers 512 columns, each warp
// one row per step with lane L loading the 16 bytes of columns 16L..16L+15
// (a warp reads 512 contiguous bytes); counters are u16 pairs (even / odd
// column of the lane's 16) in words laid out [|q|][e / 2][lane], so the
// atomic for byte e of every lane lands in bank L whatever the |q| values
// (column-major bins took random-bank conflicts and same-address collisions:
// 2.3x slower).  132 KB of shared bins, one CTA of 32 warps per SM, one wave;
// row blocks of <= 65535 rows (u16) write partial histograms in the same
// layout, summed by k_select4's first phase.  CTA (0, 0) also zeroes the
// selection's histograms, tie-column bits and candidate counter.
constexpr int kH5Cols = 512;
constexpr int kH5Threads = 1024;
constexpr int kH5Unr = 4;
constexpr int kH5Words = kBins * kH5Cols / 2;  // [a][e/2 (8)][lane (32)], u16 pairs
constexpr int kH5Smem = kH5Words * 4;

__global__ void __launch_bounds__(kH5Threads, 1) k_colhist5(const int8_t* __restrict__ q, const double* __restrict__ cm,
                                                             int64_t rows, int64_t cols, int64_t rows_per, bool vec,
                                                             uint32_t* __restrict__ partial,
                                                             uint32_t* __restrict__ hist, uint32_t* __restrict__ eqmask,
                                                             SelectOut* __restrict__ so) {
    extern __shared__ __align__(16) uint32_t hb[];
    if (blockIdx.x == 0 && blockIdx.y == 0) {
        for (int i = threadIdx.x; i < 2 * kSelHBins; i += blockDim.x) hist[i] = 0;
        for (int64_t i = threadIdx.x; i < (cols + 31) / 32; i += blockDim.x) eqmask[i] = 0;
        // the key range of the selection's bins: smallest positive cm, largest cm
        __shared__ double rmin[kH5Threads / 32], rmax[kH5Threads / 32];
        double mn = INFINITY, mx = 0.0;
        for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
            const double v = cm[c];
            if (v > 0.0) mn = fmin(mn, v);
            mx = fmax(mx, v);
        }
#pragma unroll
        for (int d = 16; d; d >>= 1) {
            mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, d));
            mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
        }
        if ((threadIdx.x & 31) == 0) {
            rmin[threadIdx.x >> 5] = mn;
            rmax[threadIdx.x >> 5] = mx;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int i = 1; i < kH5Threads / 32; ++i) {
                mn = fmin(mn, rmin[i]);
                mx = fmax(mx, rmax[i]);
            }
            so->n_cand = 0;
            so->kmin = mn == INFINITY ? ~0ull : (unsigned long long)__double_as_longlong(mn);
            so->kmax = key_of(mx, 128);
        }
    }
    for (int i = threadIdx.x; i < kH5Words / 4; i += blockDim.x) reinterpret_cast<uint4*>(hb)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = kH5Threads / 32;
    const int64_t c0 = (int64_t)blockIdx.y * kH5Cols + lane * 16;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per, r1 = min(rows, r0 + rows_per);
    uint32_t* hl = hb + lane;
#ifdef DC_PRUNE_NOATOMS
    uint32_t sink = 0;
#endif
    if (vec && c0 < cols) {  // cols % 16 == 0, q 16-byte aligned
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
    if (!vec) {  // ragged widths / unaligned: byte loads
        for (int64_t r = r0 + warp; r < r1; r += nwarp)
            for (int e = 0; e < 16; ++e)
                if (c0 + e < cols)
                    atomicAdd(hl + absq(q[r * cols + c0 + e]) * (kH5Cols / 2) + (e >> 1) * 32, (e & 1) ? 0x10000u : 1u);
    }
#ifdef DC_PRUNE_NOATOMS
    hl[0] += sink & 1;
#endif
    __syncthreads();
    uint4* out = reinterpret_cast<uint4*>(partial + ((int64_t)blockIdx.x * gridDim.y + blockIdx.y) * kH5Words);
    for (int i = threadIdx.x; i < kH5Words / 4; i += blockDim.x) out[i] = reinterpret_cast<const uint4*>(hb)[i];
}

// The whole k-th-score selection and the tie cut in ONE cooperative launch
// (grid = SMs, 3 grid barriers, 5 when only some ties stay):
//   A  every CTA sums the row-block partials of its item slice (the counts
//      are kept for D) into a 4096-bin shared histogram over the keys' actual
//      range (bin_of below), flushed with one global atomic per non-empty
//      bin; every CTA then picks the bin holding rank k;
//   D  every CTA appends the (key, count) of that bin's items to a list;
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
// grid barriers, hot-bin global atomics) and the look-back tie scan of the
// round-1 apply pass.  (One cluster of 16 CTAs with DSMEM reductions instead
// of grid barriers was tried: 98 us -- the item passes need all SMs.)
// rank-k entry of v[0..m) for any m: thread t sums a contiguous run of
// ceil(m / blockDim) entries (independent loads), one block scan picks the run,
// its owner walks it.  Returns the index; `base` becomes the count before it.
__device__ int block_find_all(const uint32_t* v, bool gmem, int m, unsigned long long k, unsigned long long& base,
                              int* s_idx, unsigned long long* s_before, unsigned long long* wsum) {
    const int per = (m + blockDim.x - 1) / blockDim.x;
    const int j0 = threadIdx.x * per, j1 = min(m, j0 + per);
    auto ld = [&](int j) -> uint32_t { return j < j1 ? (gmem ? __ldcg(v + j) : v[j]) : 0u; };
    uint32_t e0[8];  // the first 8 entries of the run stay in registers for the walk
#pragma unroll
    for (int u = 0; u < 8; ++u) e0[u] = ld(j0 + u);
    unsigned long long x = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) x += e0[u];
    for (int j = j0 + 8; j < j1; j += 8) {  // 8 independent loads in flight
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
            for (int u = 0; u < 8; ++u) e[u] = j == j0 ? e0[u] : ld(j + u);
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

__global__ void __launch_bounds__(kSelThreads) k_select4(const uint32_t* __restrict__ partial, int64_t n_rb,
                                                         int64_t n_cb, uint32_t* __restrict__ counts,
                                                         const double* __restrict__ cm, const int8_t* __restrict__ q,
                                                         int64_t rows, int64_t cols, unsigned long long k,
                                                         SelectOut* __restrict__ so, uint32_t* __restrict__ hist,
                                                         uint32_t* __restrict__ psum, uint32_t* __restrict__ cand,
                                                         uint32_t* __restrict__ eqmask, uint8_t* __restrict__ bound,
                                                         uint8_t* __restrict__ lo, uint8_t* __restrict__ hi) {
    // hist (2 x 4096 u32), eqmask and so->n_cand are zeroed by k_colhist5
    cg::grid_group grid = cg::this_grid();
    const int64_t nw = n_cb * kH5Words;  // partial words = item pairs
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
    // items follow the k_colhist5 layout: item j = 2 * word + half, word =
    // (cb * 129 + a) * 256 + (e / 2) * 32 + lane, column cb * 512 + 16 lane +
    // e (e = 2 (e / 2) + half); counts[j] is written by phase A
    const int64_t per = ((nw + gridDim.x - 1) / gridDim.x + 3) & ~3ll;  // contiguous words per CTA (A, A2, D)
    const int64_t w0 = min(nw, (int64_t)blockIdx.x * per), w1 = min(nw, w0 + per);  // nw % 4 == 0
    auto item_col_a = [&](uint32_t j, uint32_t& col) -> uint32_t {
        const uint32_t w = j >> 1, cb = w / (uint32_t)kH5Words, rem = w - cb * (uint32_t)kH5Words;
        const uint32_t a = rem / (kH5Cols / 2), slot = rem % (kH5Cols / 2);
        col = cb * kH5Cols + (slot & 31) * 16 + (slot >> 5) * 2 + (j & 1);
        return a;
    };
    auto item_key = [&](uint32_t j) {
        uint32_t col;
        const uint32_t a = item_col_a(j, col);
        return key_of(cm[col], (int)a);
    };
    // ---- A: one histogram of 4096 bins over the keys' actual range: bin 0
    // holds score 0, bins 1.. the positive keys >> sh, offset so that the
    // smallest positive key (min cm > 0 at |q| = 1) is bin 1 and sh is the
    // least shift that fits the largest (max cm at |q| = 128) -- for cm
    // spanning <= 2^8 that is 2^-8-octave resolution, so few items share the
    // chosen bin.  Keys are monotone in the bin, so the rank-k bin is exact.
    const unsigned long long kmin = __ldcg(&so->kmin), kmax = __ldcg(&so->kmax);
    int sh = 0;
    while (sh < 63 && kmin != ~0ull && (kmax >> sh) - (kmin >> sh) > (unsigned long long)(kSelHBins - 2)) ++sh;
    auto bin_of = [&](unsigned long long key) -> uint32_t {
        return key == 0 ? 0u : 1u + (uint32_t)((key >> sh) - (kmin >> sh));
    };
    for (int j = threadIdx.x; j < kSelHBins; j += blockDim.x) hs[j] = 0;
    __syncthreads();
    for (int64_t w = w0 + 4 * threadIdx.x; w < w1; w += 4 * blockDim.x) {
        // sum the row-block partials, 4 words per thread (16-B loads, 6 in flight)
        uint32_t s0[4] = {0, 0, 0, 0}, s1[4] = {0, 0, 0, 0};
        for (int64_t rb = 0; rb < n_rb; rb += 6) {
            uint4 v[6];
#pragma unroll
            for (int u = 0; u < 6; ++u)
                v[u] = rb + u < n_rb ? *reinterpret_cast<const uint4*>(partial + (rb + u) * nw + w) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < 6; ++u) {
                const uint32_t x[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    s0[t] += x[t] & 0xFFFFu;
                    s1[t] += x[t] >> 16;
                }
            }
        }
        reinterpret_cast<uint4*>(counts)[w >> 1] = make_uint4(s0[0], s1[0], s0[1], s1[1]);
        reinterpret_cast<uint4*>(counts)[(w >> 1) + 1] = make_uint4(s0[2], s1[2], s0[3], s1[3]);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            const uint32_t c = (t & 1) ? s1[t >> 1] : s0[t >> 1];
            if (c) atomicAdd(&hs[bin_of(item_key((uint32_t)(2 * (w + (t >> 1)) + (t & 1))))], c);
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < kSelHBins; j += blockDim.x) {
        const uint32_t v = hs[j];
        if (v) atomicAdd(hist + j, v);
    }
    TMARK();
    grid.sync();
    unsigned long long base = 0;
    const uint32_t bin = (uint32_t)block_find_all(hist, true, kSelHBins, k, base, &s_idx, &s_before, wsum);
    TMARK();
    // ---- D: candidates = the items of that bin
    for (int64_t wb = w0; wb < w1; wb += kUnr * blockDim.x) {
        uint2 c[kUnr];
#pragma unroll
        for (int u = 0; u < kUnr; ++u) {
            const int64_t w = wb + (int64_t)u * blockDim.x + threadIdx.x;
            c[u] = w < w1 ? reinterpret_cast<const uint2*>(counts)[w] : make_uint2(0, 0);
        }
#pragma unroll
        for (int u = 0; u < 2 * kUnr; ++u) {
            const int64_t j = 2 * (wb + (int64_t)(u >> 1) * blockDim.x + threadIdx.x) + (u & 1);
            const uint32_t cnt = (u & 1) ? c[u >> 1].y : c[u >> 1].x;
            const unsigned long long key = cnt ? item_key((uint32_t)j) : 0ull;
            const bool f = cnt && bin_of(key) == bin;
            const uint32_t m = __ballot_sync(0xffffffffu, f);
            if (m) {
                uint32_t pos = 0;
                if (lane == 0) pos = atomicAdd(&so->n_cand, (uint32_t)__popc(m));
                pos = __shfl_sync(0xffffffffu, pos, 0);
                if (f)  // (key, count) so that the ranking needs one load per candidate
                    reinterpret_cast<ulonglong2*>(cand)[pos + __popc(m & ((1u << lane) - 1u))] =
                        make_ulonglong2(key, cnt);
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
        // comparison with all others (nc is small at 2^-8-octave bins)
        __shared__ unsigned long long s_T, s_kk;
        __shared__ uint32_t s_eq;
        for (uint32_t j = threadIdx.x; j < nc; j += blockDim.x) {
            const ulonglong2 e = __ldcg(reinterpret_cast<const ulonglong2*>(cand) + j);
            ckey[j] = e.x;
            ccnt[j] = (uint32_t)e.y;
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
    } else {  // many candidates: 8-bit radix passes over the whole key, from L2
        unsigned long long prefix = 0;
        for (int shift = 56; shift >= 0; shift -= 8) {
            for (int j = threadIdx.x; j < 256; j += blockDim.x) h[j] = 0;
            __syncthreads();
            for (uint32_t j = threadIdx.x; j < nc; j += blockDim.x) {
                const ulonglong2 e = __ldcg(reinterpret_cast<const ulonglong2*>(cand) + j);
                if (shift == 56 || (e.x >> (shift + 8)) == prefix)
                    atomicAdd(&h[(e.x >> shift) & 0xFFu], (uint32_t)e.y);
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
    const int nmw = (int)((cols + 31) >> 5);
    uint32_t E;
    {
        const int per_w = (nmw + blockDim.x - 1) / blockDim.x;
        const int m0 = threadIdx.x * per_w, m1 = min(nmw, m0 + per_w);
        uint32_t c = 0;
        for (int j = m0; j < m1; ++j) c += __popc(__ldcg(eqmask + j));
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
            for (int j = m0; j < m1; ++j)
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

// out = q with |q| < bound[c] zeroed, and the ties (|q| in [lo, hi)) at flat
// index <= cut.  16-B path: a thread owns 16 columns (bounds in registers,
// loaded once) and streams rows, a warp covering 512 contiguous bytes of a
// row, kApUnr rows in flight.
constexpr int kApThreads = 256, kApUnr = 4;

__device__ __forceinline__ uint32_t zero_mask4(uint32_t qw, uint32_t bw, uint32_t lw, uint32_t hw, uint32_t cw) {
    const uint32_t a = __vabs4(qw);
    const uint32_t lt = __vcmpltu4(a, bw);
    const uint32_t tie = __vcmpltu4(a, hw) & ~__vcmpltu4(a, lw) & cw;
    return qw & ~(lt | tie);
}

__global__ void __launch_bounds__(kApThreads) k_apply5(const int8_t* __restrict__ q, const uint8_t* __restrict__ bound,
                                                       const uint8_t* __restrict__ lo, const uint8_t* __restrict__ hi,
                                                       int64_t rows, int64_t cols, const SelectOut* __restrict__ so,
                                                       int8_t* __restrict__ out) {
    const int64_t c0 = ((int64_t)blockIdx.x * kApThreads + threadIdx.x) * 16;
    if (c0 >= cols) return;
    const unsigned long long cut = so->cut;
    const uint4 b = *reinterpret_cast<const uint4*>(bound + c0);
    const uint4 l = *reinterpret_cast<const uint4*>(lo + c0);
    const uint4 h = *reinterpret_cast<const uint4*>(hi + c0);
    const int64_t G = gridDim.y;
    for (int64_t r = blockIdx.y; r < rows; r += G * kApUnr) {
        uint4 v[kApUnr];
#pragma unroll
        for (int u = 0; u < kApUnr; ++u) {
            const int64_t rr = r + u * G;
            v[u] = rr < rows ? __ldcs(reinterpret_cast<const uint4*>(q + rr * cols + c0)) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < kApUnr; ++u) {
            const int64_t rr = r + u * G;
            if (rr >= rows) break;
            const int64_t i0 = rr * cols + c0;
            // ties at index <= cut: byte j of word w is element 4w + j
            uint32_t cw[4];
            const long long ck = (long long)cut - i0;
            if (cut == ~0ull || ck >= 15) {
                cw[0] = cw[1] = cw[2] = cw[3] = 0xFFFFFFFFu;
            } else if (ck < 0) {
                cw[0] = cw[1] = cw[2] = cw[3] = 0u;
            } else {
#pragma unroll
                for (int w = 0; w < 4; ++w) cw[w] = __vcmpleu4(0x03020100u + 0x04040404u * w, 0x01010101u * (uint32_t)ck);
            }
            uint4 o;
            o.x = zero_mask4(v[u].x, b.x, l.x, h.x, cw[0]);
            o.y = zero_mask4(v[u].y, b.y, l.y, h.y, cw[1]);
            o.z = zero_mask4(v[u].z, b.z, l.z, h.z, cw[2]);
            o.w = zero_mask4(v[u].w, b.w, l.w, h.w, cw[3]);
            __stcs(reinterpret_cast<uint4*>(out + i0), o);
        }
    }
}

// scalar path (ragged widths / unaligned buffers)
__global__ void __launch_bounds__(kApThreads) k_apply_bytes(const int8_t* __restrict__ q,
                                                            const uint8_t* __restrict__ bound,
                                                            const uint8_t* __restrict__ lo,
                                                            const uint8_t* __restrict__ hi, int64_t n, int64_t cols,
                                                            const SelectOut* __restrict__ so,
                                                            int8_t* __restrict__ out) {
    const unsigned long long cut = so->cut;
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
constexpr int kRowBins = 2048;  // per-row key-range histogram
constexpr int kRowCand = 512;   // candidates ranked directly (else radix over the bin)

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
    __shared__ uint32_t hist[256], rbins[kRowBins];
    __shared__ uint32_t wsum[kPrThreads / 32], s_nc, s_bin;
    __shared__ unsigned long long s_prefix, s_k[2], s_min[kPrThreads / 32], s_max[kPrThreads / 32];
    __shared__ unsigned long long cand[kRowCand];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int c0 = t * 16;
    double cmr[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) cmr[j] = c0 + j < cols ? cm[c0 + j] : 0.0;
    const bool vec = (cols & 15) == 0 && ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    // the next row's 16 bytes are loaded before this row is processed (the
    // load latency was the largest stall: one row per CTA at a time)
    uint4 qnext = make_uint4(0, 0, 0, 0);
    if (vec && c0 < cols && blockIdx.x < rows) qnext = *reinterpret_cast<const uint4*>(q + (int64_t)blockIdx.x * cols + c0);
    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        const int8_t* qr = q + row * cols;
        int8_t* orow = out + row * cols;
        int8_t v[16];
        if (vec) {
            const uint4 qv = qnext;
            if (c0 < cols && row + gridDim.x < rows)
                qnext = *reinterpret_cast<const uint4*>(q + (row + gridDim.x) * cols + c0);
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
                if (key[j]) kmin = min(kmin, key[j]);  // smallest POSITIVE key (0 has its own bin)
                kmax = max(kmax, key[j]);
            }
        }
        unsigned long long prefix, kk;
        {
        // One histogram pass over the row's key range (kRowBins bins: bin 0 =
        // score 0, then positive keys >> sh offset to the smallest), the
        // rank-k bin by a block scan, then the exact k-th key among that bin's
        // (few) candidates by direct ranking -- instead of up to eight 8-bit
        // radix passes of 64-bit compares and shifts per element (ALU-bound).
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
        for (int i = t; i < kRowBins; i += kPrThreads) rbins[i] = 0;
        if (t == 0) s_nc = 0;
        __syncthreads();
        for (int i = 0; i < kPrThreads / 32; ++i) {
            kmin = min(kmin, s_min[i]);
            kmax = max(kmax, s_max[i]);
        }
        // kmin here is the smallest positive key (zero keys were excluded below)
        // (kmax >> sh) - (kmin >> sh) <= ((kmax - kmin) >> sh) + 1 < 1025 bins
        const unsigned long long span = kmin == ~0ull ? 0ull : kmax - kmin;
        const int sh = max(0, 64 - __clzll(span) - 10);
        auto rbin = [&](unsigned long long key) -> uint32_t {
            return key == 0 ? 0u : 1u + (uint32_t)((key >> sh) - (kmin >> sh));
        };
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (c0 + j < cols) atomicAdd(&rbins[rbin(key[j])], 1u);
        __syncthreads();
        // block scan over the bins: kRowBins / kPrThreads consecutive bins per thread
        constexpr int kPer = kRowBins / kPrThreads;
        uint32_t loc[kPer], tot = 0;
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            loc[i] = rbins[t * kPer + i];
            tot += loc[i];
        }
        uint32_t inc = tot;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += o;
        }
        if (lane == 31) wsum[w] = inc;
        __syncthreads();
        uint32_t before = 0;
        for (int i = 0; i < w; ++i) before += wsum[i];
        uint32_t c = before + inc - tot;
        const unsigned long long kq = (unsigned long long)k;
        if (c < kq && kq <= c + tot) {
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
                if (c < kq && kq <= c + loc[i]) {
                    s_bin = (uint32_t)(t * kPer + i);
                    s_k[0] = kq - c;  // rank inside the bin (1-based)
                }
                c += loc[i];
            }
        }
        __syncthreads();
        const uint32_t bsel = s_bin;
        kk = s_k[0];
        // candidates: the keys of the chosen bin
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            if (c0 + j < cols && rbin(key[j]) == bsel) {
                const uint32_t pos = atomicAdd(&s_nc, 1u);
                if (pos < kRowCand) cand[pos] = key[j];
            }
        }
        __syncthreads();
        const uint32_t nc = s_nc;
        if (nc <= kRowCand) {
            for (uint32_t i = t; i < nc; i += kPrThreads) {
                const unsigned long long ki = cand[i];
                uint32_t lt = 0, eq = 0;
                for (uint32_t m = 0; m < nc; ++m) {
                    lt += cand[m] < ki;
                    eq += cand[m] == ki;
                }
                if (lt < kk && kk <= lt + eq) {  // every candidate equal to T writes the same
                    s_prefix = ki;
                    s_k[1] = kk - lt;
                }
            }
            __syncthreads();
            prefix = s_prefix;
            kk = s_k[1];
        } else {  // many equal-bin keys (e.g. constant channel maxima): 8-bit radix over the bin's keys
            prefix = 0;
            for (int pass = 0; pass < 8; ++pass) {
                const int shift = 56 - 8 * pass;
                hist[t] = 0;
                __syncthreads();
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < cols && rbin(key[j]) == bsel && (pass == 0 || (key[j] >> (shift + 8)) == prefix))
                        atomicAdd(&hist[(key[j] >> shift) & 0xFF], 1u);
                __syncthreads();
                block_pick256(hist, prefix, kk, &s_prefix, s_k, wsum);
            }
        }
        __syncthreads();
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

// Per row, one WARP per row (no block barriers): lane L holds the 16-byte
// pieces at columns 512 m + 16 L (m = 0..7: up to 4096 columns, 16-aligned)
// in registers; the channel maxima sit in shared memory in the matching
// order (column 512 m + 16 L + e at index 512 m + 32 e + L: conflict-free
// LDS.64 for every lane).  Keys are recomputed per pass (one DMUL each)
// rather than stored.  The histogram bins are fixed for the whole tensor:
// the high words of the keys between those of (min cm > 0) x 1 and
// (max cm) x 128, >> s so they fit kRwBins (bin 0: high word 0, i.e. score 0
// or subnormal) -- no per-row min / max pass, 32-bit bin arithmetic.  Then
// the rank-k bin by a warp scan, the (few) candidates of that bin ranked
// directly on their full keys (8-bit radix passes if there are many), and the
// apply pass, with the tie ranks in column order by per-chunk warp scans only
// when some ties stay.
constexpr int kRwWarps = 16;
constexpr int kRwBins = 1056;  // 33 per lane
constexpr int kRwCand = 64;

struct RwSmem {
    double cm[kRowMax];  // permuted channel maxima
    uint32_t hist[kRwWarps][kRwBins];
    unsigned long long cand[kRwWarps][kRwCand];
    uint16_t ccol[kRwWarps][kRwCand];
    double red[2][kRwWarps];
};

template <bool FULL>  // cols % 512 == 0: every lane holds every chunk
__global__ void __launch_bounds__(kRwWarps * 32, 2) k_prune_rowsw(const int8_t* __restrict__ q,
                                                                  const double* __restrict__ cm, int64_t rows,
                                                                  int64_t cols, int64_t k, int8_t* __restrict__ out) {
    extern __shared__ __align__(16) uint8_t rw_raw[];
    RwSmem& S = *reinterpret_cast<RwSmem*>(rw_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double mn = INFINITY, mx = 0.0;
    for (int c = threadIdx.x; c < kRowMax; c += blockDim.x) {
        const int m = c >> 9, L = (c >> 4) & 31, e = c & 15;
        const double v = c < cols ? cm[c] : 0.0;
        S.cm[(m << 9) + (e << 5) + L] = v;
        if (c < cols) {
            if (v > 0.0) mn = fmin(mn, v);
            mx = fmax(mx, v);
        }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, d));
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
    }
    if (lane == 0) {
        S.red[0][warp] = mn;
        S.red[1][warp] = mx;
    }
    __syncthreads();
    for (int i = 0; i < kRwWarps; ++i) {
        mn = fmin(mn, S.red[0][i]);
        mx = fmax(mx, S.red[1][i]);
    }
    // bin(key) = hi == 0 ? 0 : 1 + ((hi - hmin) >> s), hi = key's high word
    const uint32_t hmin = mn == INFINITY ? 0xFFFFFFFFu : (uint32_t)(__double_as_longlong(mn) >> 32);
    const uint32_t hmax = (uint32_t)(key_of(mx, 128) >> 32);
    const uint32_t hspan = hmin == 0xFFFFFFFFu || hmax < hmin ? 0u : hmax - hmin;
    const int s = max(0, 32 - __clz(hspan) - 10);  // (hspan >> s) < 1024
    // = hi == 0 ? 0 : 1 + ((hi - hmin) >> s): no positive key has 0 < hi < hmin,
    // and hi - hmin2 < 2^31 (hi <= 0x7FF00000, hmin2 >= -2^22), so one signed
    // shift and a clamp at 0 give it
    const int32_t hmin2 = (int32_t)hmin - (1 << s);
    auto bin_of = [&](unsigned long long key) -> uint32_t {
        const int32_t hi = (int32_t)(key >> 32);
        return (uint32_t)max(0, (hi - hmin2) >> s);
    };
    const int nm = (int)((cols + 511) >> 9);  // 512-column chunks
    uint32_t* H = S.hist[warp];
    unsigned long long* C = S.cand[warp];
    uint16_t* CC = S.ccol[warp];
    const unsigned long long kq = (unsigned long long)k;
    const int64_t nwarp = (int64_t)gridDim.x * kRwWarps;
    auto valid = [&](int m) { return FULL || (int64_t)((m << 9) + (lane << 4)) < cols; };
    auto keyat = [&](const uint4 (&qv)[8], int m, int e) -> unsigned long long {
        const uint32_t w = (&qv[m].x)[e >> 2];
        const uint32_t a = __byte_perm(__vabs4(w), 0, 0x4440 + (e & 3));
        return key_of(S.cm[(m << 9) + (e << 5) + lane], (int)a);
    };
    for (int64_t row = (int64_t)blockIdx.x * kRwWarps + warp; row < rows; row += nwarp) {
        const int8_t* qr = q + row * cols;
        uint4 qv[8];
#pragma unroll
        for (int m = 0; m < 8; ++m)
            qv[m] = (m < nm && valid(m)) ? *reinterpret_cast<const uint4*>(qr + (m << 9) + (lane << 4))
                                         : make_uint4(0, 0, 0, 0);
        for (int i = lane; i < kRwBins; i += 32) H[i] = 0;
        __syncwarp();
        // ---- histogram
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            if (m >= nm || !valid(m)) continue;
#pragma unroll
            for (int e = 0; e < 16; ++e) atomicAdd(&H[bin_of(keyat(qv, m, e))], 1u);
        }
        __syncwarp();
        // ---- rank-k bin: lane L sums bins [33 L, 33 L + 33)
        constexpr int kPer = kRwBins / 32;
        uint32_t tot = 0;
#pragma unroll
        for (int i = 0; i < kPer; ++i) tot += H[lane * kPer + i];
        uint32_t inc = tot;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += o;
        }
        uint32_t bsel = 0, kin = 0;  // chosen bin, rank inside it
        {
            uint32_t c = inc - tot;
            const bool mine = c < kq && kq <= (unsigned long long)inc;
            if (mine) {
                for (int i = 0; i < kPer; ++i) {
                    const uint32_t h = H[lane * kPer + i];
                    if (kq <= (unsigned long long)c + h) {
                        bsel = (uint32_t)(lane * kPer + i);
                        kin = (uint32_t)(kq - c);
                        break;
                    }
                    c += h;
                }
            }
            const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
            bsel = __shfl_sync(0xffffffffu, bsel, src);
            kin = __shfl_sync(0xffffffffu, kin, src);
        }
        // ---- one pass: bins below the chosen one are zeroed now, bins above
        // kept, the chosen bin's entries (key + column) listed
        uint32_t nc = 0;
        int8_t* orow = out + row * cols;
#pragma unroll
        for (int m = 0; m < 8; ++m) {
            if (m >= nm) continue;
            uint32_t zm = 0;
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const unsigned long long key = valid(m) ? keyat(qv, m, e) : ~0ull;
                const uint32_t bn = valid(m) ? bin_of(key) : 0xFFFFFFFFu;
                zm |= (uint32_t)(bn < bsel) << e;
                const bool f = bn == bsel;
                const uint32_t msk = __ballot_sync(0xffffffffu, f);
                if (msk) {  // warp-uniform and rare (a dozen of 128 steps)
                    const uint32_t pos = nc + __popc(msk & ((1u << lane) - 1u));
                    if (f && pos < (uint32_t)kRwCand) {
                        C[pos] = key;
                        CC[pos] = (uint16_t)((m << 9) + (lane << 4) + e);
                    }
                    nc += __popc(msk);
                }
            }
            uint32_t* w4 = &qv[m].x;
#pragma unroll
            for (int b4 = 0; b4 < 4; ++b4)
                w4[b4] &= ~((((zm >> (4 * b4)) & 15u) * 0x00204081u & 0x01010101u) * 0xFFu);
        }
        __syncwarp();
        if (nc <= (uint32_t)kRwCand) {
            // rank the candidates: T = the kin-th smallest key; zero those < T and
            // the first kk (column order) of those == T, in their owners' registers
            unsigned long long T = 0, kk = 0;
            for (uint32_t i = lane; i < nc; i += 32) {
                const unsigned long long ki = C[i];
                uint32_t lt = 0, eq = 0;
                for (uint32_t j = 0; j < nc; ++j) {
                    lt += C[j] < ki;
                    eq += C[j] == ki;
                }
                if (lt < kin && kin <= lt + eq) {
                    T = ki;
                    kk = kin - lt;
                }
            }
            const int src = __ffs(__ballot_sync(0xffffffffu, kk != 0)) - 1;
            T = __shfl_sync(0xffffffffu, T, src);
            kk = __shfl_sync(0xffffffffu, kk, src);
            for (uint32_t i = 0; i < nc; ++i) {  // uniform loop; the owner lane applies
                const uint32_t col = CC[i];
                if ((int)((col >> 4) & 31) != lane) continue;
                const unsigned long long ki = C[i];
                bool z = ki < T;
                if (ki == T) {  // tie: its rank among the ties in column order
                    uint32_t r = 0;
                    for (uint32_t j = 0; j < nc; ++j) r += C[j] == T && CC[j] < col;
                    z = r < kk;
                }
                if (z) {
                    const int m = col >> 9, e = col & 15;
                    (&qv[m].x)[e >> 2] &= ~(0xFFu << (8 * (e & 3)));
                }
            }
        } else {  // many keys in one bin (e.g. equal channel maxima): 8-bit radix passes over the bin
            unsigned long long prefix = 0, kr = kin;
            for (int pass = 0; pass < 8; ++pass) {
                const int shift = 56 - 8 * pass;
                for (int i = lane; i < 256; i += 32) H[i] = 0;
                __syncwarp();
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    if (m >= nm || !valid(m)) continue;
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const unsigned long long key = keyat(qv, m, e);
                        if (bin_of(key) == bsel && (pass == 0 || (key >> (shift + 8)) == prefix))
                            atomicAdd(&H[(key >> shift) & 0xFF], 1u);
                    }
                }
                __syncwarp();
                uint32_t hv[8], ht = 0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    hv[i] = H[lane * 8 + i];
                    ht += hv[i];
                }
                uint32_t hi2 = ht;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t o = __shfl_up_sync(0xffffffffu, hi2, d);
                    if (lane >= d) hi2 += o;
                }
                uint32_t c = hi2 - ht, dsel = 0, kn = 0;
                const bool mine = c < kr && kr <= (unsigned long long)hi2;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    if (mine && c < kr && kr <= (unsigned long long)c + hv[i]) {
                        dsel = (uint32_t)(lane * 8 + i);
                        kn = (uint32_t)(kr - c);
                    }
                    c += hv[i];
                }
                const int src = __ffs(__ballot_sync(0xffffffffu, mine)) - 1;
                dsel = __shfl_sync(0xffffffffu, dsel, src);
                kr = __shfl_sync(0xffffffffu, kn, src);
                prefix = (prefix << 8) | dsel;
                __syncwarp();
            }
            const unsigned long long T = prefix, kk = kr;
            // the chosen bin's entries: < T zeroed, ties in column order
            uint32_t eqm[8];
            uint32_t myeq = 0;
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                eqm[m] = 0;
                if (m >= nm || !valid(m)) continue;
                uint32_t ltm = 0;
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    const unsigned long long key = keyat(qv, m, e);
                    if (bin_of(key) != bsel) continue;
                    ltm |= (uint32_t)(key < T) << e;
                    eqm[m] |= (uint32_t)(key == T) << e;
                }
                myeq += __popc(eqm[m]);
                uint32_t* w4 = &qv[m].x;
#pragma unroll
                for (int b4 = 0; b4 < 4; ++b4)
                    w4[b4] &= ~((((ltm >> (4 * b4)) & 15u) * 0x00204081u & 0x01010101u) * 0xFFu);
            }
            const uint32_t eq_total = __reduce_add_sync(0xffffffffu, myeq);
            const bool some = (unsigned long long)eq_total > kk;
            unsigned long long before = 0;
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                if (m >= nm) continue;
                uint32_t z = eqm[m];
                if (some) {
                    const uint32_t cnt = __popc(eqm[m]);
                    uint32_t ic = cnt;
#pragma unroll
                    for (int d = 1; d < 32; d <<= 1) {
                        const uint32_t o = __shfl_up_sync(0xffffffffu, ic, d);
                        if (lane >= d) ic += o;
                    }
                    unsigned long long r = before + ic - cnt;
                    z = 0;
                    for (uint32_t e = eqm[m]; e; e &= e - 1) {
                        if (r < kk) z |= e & (0u - e);
                        ++r;
                    }
                    before += __shfl_sync(0xffffffffu, ic, 31);
                }
                uint32_t* w4 = &qv[m].x;
#pragma unroll
                for (int b4 = 0; b4 < 4; ++b4)
                    w4[b4] &= ~((((z >> (4 * b4)) & 15u) * 0x00204081u & 0x01010101u) * 0xFFu);
            }
        }
#pragma unroll
        for (int m = 0; m < 8; ++m)
            if (m < nm && valid(m)) *reinterpret_cast<uint4*>(orow + (m << 9) + (lane << 4)) = qv[m];
        __syncwarp();  // the candidate list is rewritten by the next row
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

static int64_t colhist5_rb(int64_t rows, int64_t cols) {
    const int64_t n_cb = (cols + kH5Cols - 1) / kH5Cols;
    int64_t n_rb = (int64_t)sm_count_pr() / n_cb;  // one CTA per SM, one wave
    n_rb = n_rb < 1 ? 1 : (n_rb > 64 ? 64 : n_rb);
    if (n_rb > rows) n_rb = rows > 0 ? rows : 1;
    const int64_t need = (rows + 65534) / 65535;  // u16 partial counts
    return n_rb < need ? need : n_rb;
}

// items of the selection = u16 counters of one row block's partial histogram
static int64_t prune_items(int64_t cols) { return 2 * ((cols + kH5Cols - 1) / kH5Cols) * (int64_t)kH5Words; }

extern "C" int dc_prune_scratch_bytes(int64_t rows, int64_t cols, uint64_t* out) {
    const uint64_t items = (uint64_t)prune_items(cols);
    *out = 8ull * kSelHBins + 256 + 4ull * 4096 + 256 + sizeof(SelectOut) + 256 + 16ull * items + 256 +
           4ull * (uint64_t)((cols + 31) / 32) + 256 + 4ull * items + 256 + 3ull * (uint64_t)cols + 256 +
           2ull * items * (uint64_t)colhist5_rb(rows, cols) + 256;
    return DC_OK;
}

// Per tensor: (column, |q|) partial histograms -> one cooperative selection
// launch (sums them) -> one streaming apply pass (3 launches, 20 in round 1).
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
    const int64_t items = prune_items(cols);
    uint8_t* p = align(scratch);
    auto* hist = reinterpret_cast<uint32_t*>(p);
    p = align(p + 8ull * kSelHBins);
    auto* psum = reinterpret_cast<uint32_t*>(p);
    p = align(p + 4ull * 4096);
    auto* so = reinterpret_cast<SelectOut*>(p);
    p = align(p + sizeof(SelectOut));
    auto* cand = reinterpret_cast<uint32_t*>(p);  // 16-B (key, count) entries
    p = align(p + 16ull * items);
    auto* eqmask = reinterpret_cast<uint32_t*>(p);
    p = align(p + 4ull * ((cols + 31) / 32));
    auto* counts = reinterpret_cast<uint32_t*>(p);
    p = align(p + 4ull * items);
    uint8_t* bound = p;
    uint8_t* lo = p + cols;
    uint8_t* hi = p + 2 * cols;
    p = align(p + 3ull * cols);
    auto* partial = reinterpret_cast<uint32_t*>(p);
    const bool vec = cols % 16 == 0 && (reinterpret_cast<uintptr_t>(q) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(out) & 15) == 0;

    int64_t n_cb = (cols + kH5Cols - 1) / kH5Cols;
    int64_t n_rb = colhist5_rb(rows, cols);
    const int64_t rows_per = (rows + n_rb - 1) / n_rb;
    n_rb = (rows + rows_per - 1) / rows_per;
    static bool attr5 = false;
    if (!attr5) {
        cudaFuncSetAttribute(k_colhist5, cudaFuncAttributeMaxDynamicSharedMemorySize, kH5Smem);
        attr5 = true;
    }
    k_colhist5<<<dim3((unsigned)n_rb, (unsigned)n_cb), kH5Threads, kH5Smem, st>>>(q, cm, rows, cols, rows_per, vec,
                                                                                  partial, hist, eqmask, so);
    DC_CHECK_LAUNCH("k_colhist5");
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
        void* args[] = {(void*)&partial, (void*)&n_rb, (void*)&n_cb, (void*)&counts, (void*)&cm, (void*)&q,
                        (void*)&rows, (void*)&cols, (void*)&kk, (void*)&so, (void*)&hist, (void*)&psum,
                        (void*)&cand, (void*)&eqmask, (void*)&bound, (void*)&lo, (void*)&hi};
        cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_select4, dim3((unsigned)grid), dim3(kSelThreads),
                                                    args, 0, st);
        if (e != cudaSuccess) {
            set_error("k_select4", e);
            return DC_ERR_CUDA;
        }
    }
    if (vec) {
        const int64_t gx = (cols / 16 + kApThreads - 1) / kApThreads;
        int64_t gy = (int64_t)sm_count_pr() * 8 / gx;
        gy = gy < 1 ? 1 : (gy > rows ? rows : gy);
        k_apply5<<<dim3((unsigned)gx, (unsigned)gy), kApThreads, 0, st>>>(q, bound, lo, hi, rows, cols, so, out);
        DC_CHECK_LAUNCH("k_apply5");
    } else {
        k_apply_bytes<<<(unsigned)(sm_count_pr() * 8), kApThreads, 0, st>>>(q, bound, lo, hi, n, cols, so, out);
        DC_CHECK_LAUNCH("k_apply_bytes");
    }
    return DC_OK;
}

extern "C" int dc_prune_rows(const int8_t* q, const double* cm, int64_t rows, int64_t cols, int64_t k, int8_t* out,
                             void* stream) {
    if (rows < 0 || cols < 0 || k < 0 || k > cols) return DC_ERR_ARG;
    if (rows == 0 || cols == 0) return DC_OK;
    const bool vec = (cols & 15) == 0 && ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    if (k > 0 && cols <= kRowMax && vec) {
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_prune_rowsw<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RwSmem));
            cudaFuncSetAttribute(k_prune_rowsw<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RwSmem));
            attr = true;
        }
        const int64_t need = (rows + kRwWarps - 1) / kRwWarps, cap = (int64_t)sm_count_pr() * 2;
        if (cols % 512 == 0)
            k_prune_rowsw<true><<<(unsigned)(need < cap ? need : cap), kRwWarps * 32, sizeof(RwSmem),
                                  (cudaStream_t)stream>>>(q, cm, rows, cols, k, out);
        else
            k_prune_rowsw<false><<<(unsigned)(need < cap ? need : cap), kRwWarps * 32, sizeof(RwSmem),
                                   (cudaStream_t)stream>>>(q, cm, rows, cols, k, out);
        DC_CHECK_LAUNCH("k_prune_rowsw");
        return DC_OK;
    }
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
