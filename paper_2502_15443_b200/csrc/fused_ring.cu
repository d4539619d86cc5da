// Fused decompress -> W8A8 GEMM, TMEM-ring version (north-star kernel 3).
//
// One persistent CTA per SM of 16 decoder warps (512 threads: 4 warps per SM
// sub-partition, so 128 registers per thread and no spills).  A work item is
// (layer, 8 row-tiles = 1024 weight rows, K-slice of up to kFK bytes).  Each
// thread owns TMEM lane 32*(warp&3)+lane and decodes two rows of that lane
// (tiles 2*(warp>>2) and 2*(warp>>2)+1) along K, in lockstep with every other
// chain of the CTA:
//   * stream bytes come from a private 128-byte ring per chain, refilled 32 B
//     at a time with cp.async (LDGSTS) ahead of consumption;
//   * every 16 decoded bytes go registers -> TMEM (tcgen05.st) into a ring of
//     kRSlots 32-byte K-steps;
//   * after each K-step every warp bumps the slot's arrival counter (shared
//     atomic, acq_rel); the LAST warp to arrive issues one
//     tcgen05.mma.kind::i8 per tile (A from TMEM, X from SW128 smem) and
//     commits to the slot's "empty" mbarrier.  No dedicated MMA warp: the
//     issue cost lands on whichever warp completes the step.
// Accumulators live in TMEM (8 tiles x 16 columns).  Decoded weights never
// touch shared memory or HBM.  Each chain is checked at the end of its
// K-slice against the split-point index (or 2^20 / stream end); a mismatch
// flags the chunk DC_CHUNK_CHAIN for an exact fallback.
#include "common.cuh"
#include "rans_common.cuh"
#include "tc.cuh"

namespace dc {

struct GemmTensorR {  // identical layout to GemmTensor (gemm_grouped.cu)
    const int8_t* x;
    int32_t* acc;
    int64_t t_off;
    int32_t n_rows;
    int32_t k;
};

// Optional dequant epilogue per layer (W8A8 numerics, scaling.py:127-152):
// y[t, n] = acc[t, n] * scale with scale = sx * sw.  Accumulation stays exact
// int32 across K-slices; the LAST item of a 1024-row block (per-block counter)
// converts that block, so the launch emits fp32 outputs directly.
struct RingEpi {
    float* y;          // fp32 [ntok, n_rows] or null (int32 accumulators only)
    uint32_t* cnt;     // per 1024-row block: items finished (zero between launches)
    float scale;       // sx * sw when sx is null
    int32_t n_slices;  // K-slices per row block
    const double* sx;  // device activation scale (dc_act_quant) or null
    double sw;         // weight scale: y = acc * (float)(sx * sw)
};

constexpr int kRDec = 16;                     // decoder warps
constexpr int kRThreads = kRDec * 32;
constexpr int kRTiles = 8;                    // row-tiles per item (1024 rows)
constexpr int kFK = 2048;                     // max K bytes per item
constexpr int kRSlots = 6;                    // TMEM ring depth (32-byte K-steps)
constexpr int kRRing = 128;                   // stream ring bytes per chain
constexpr int kRNT = 16;                      // tokens (UMMA N)
constexpr uint32_t kRAcc = kRSlots * 64;      // accumulator columns [kRAcc, kRAcc + 128)
static_assert(kRAcc + kRTiles * kRNT <= 512, "TMEM columns");

struct RingSmem {
    TableSmem tab[2];
    alignas(1024) uint8_t x[kFK / 128][kRNT * 128];      // X slice: SW128 atoms of 16 rows x 128 B
    alignas(128) uint8_t ring[kRDec * 64][kRRing];       // chain (warp, u, lane)
    uint64_t empty[kRSlots];
    uint64_t done;
    uint32_t cnt[kRSlots];
    uint32_t tmem;
    int32_t cur[2];
    int32_t last;
};

__device__ __forceinline__ void tmem_st4(uint32_t taddr, const uint32_t (&w)[4]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(w[0]), "r"(w[1]),
                 "r"(w[2]), "r"(w[3])
                 : "memory");
}

__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t* p, uint32_t v) {
    uint32_t old;
    asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// One decode step from the chain's stream ring.  `pr` is a free-running
// byte counter whose low 7 bits are the ring offset of the next unread byte;
// the shared address of a byte is (pr & 127) | rb (one LOP3, rb = the
// 128-B aligned ring base), so the counter itself never wraps.
__device__ __forceinline__ uint32_t ring_step(uint32_t& x, uint32_t& pr, uint32_t& nb, uint32_t tab, uint32_t rb,
                                              const FmaK&) {  // FMA-pipe variant measured slower here
    uint32_t e;
    asm volatile(
        "{\n\t.reg .pred q;\n\t.reg .u32 a, f, b, t, a1, a2;\n\t"
        "and.b32 a, %0, 4095;\n\t"
        "mad.lo.u32 a, a, 4, %4;\n\t"
        "ld.shared.u32 %3, [a];\n\t"
        "shr.u32 f, %3, 20;\n\t"
        "shr.u32 b, %3, 8;\n\t"
        "shr.u32 t, %0, 12;\n\t"
        "sub.u32 t, t, 4096;\n\t"
        "mad.lo.u32 %0, f, t, b;\n\t"
        "setp.lt.u32 q, %0, 0x100000;\n\t"
        "@q mad.lo.u32 %0, %0, 256, %2;\n\t"
        "@q add.u32 %1, %1, 1;\n\t"
        "lop3.b32 a1, %1, 127, %5, 0xEA;\n\t"
        "@q ld.shared.u8 %2, [a1];\n\t"
        "setp.lt.u32 q, %0, 0x100000;\n\t"
        "@q mad.lo.u32 %0, %0, 256, %2;\n\t"
        "@q add.u32 %1, %1, 1;\n\t"
        "lop3.b32 a2, %1, 127, %5, 0xEA;\n\t"
        "@q ld.shared.u8 %2, [a2];\n\t}"
        : "+r"(x), "+r"(pr), "+r"(nb), "=r"(e)
        : "r"(tab), "r"(rb));
    return e;
}

struct Chain {
    uint32_t x, pr, nb, tab, rb;  // pr: free-running ring counter, rb: ring base
    uint32_t w0, w1, o;           // word window (kWindow): pr = ring counter of w1's byte address
    uint64_t gfill;   // next global address to request (16-B aligned)
    uint32_t xe;      // expected end state
    uint64_t gend;    // expected end position (global address of the next byte)
    uint64_t gstart;  // global address of the first byte
    int mode;         // 0 ANS, 1 stored raw, 2 single symbol, 3 inactive
    int chunk;
    uint32_t sym;
};

// Stream reads: byte-at-a-time (LDS.U8 per refill) or through a two-word
// window (one predicated LDS.32 per step pair, see rans_common.cuh Win).
#ifndef DC_FUSED_WINDOW
#define DC_FUSED_WINDOW 1
#endif
constexpr bool kWindow = DC_FUSED_WINDOW != 0;

// bytes buffered ahead of the read position (ring invariant: < 128)
__device__ __forceinline__ uint32_t ring_avail(const Chain& c) {
    const uint32_t rd = kWindow ? c.pr - 4u + (c.o >> 3) : c.pr;
    return ((uint32_t)c.gfill - rd) & 127u;
}

__device__ __forceinline__ void fwin_init(Chain& c, uint32_t p) {  // p: ring offset of the first byte
    const uint32_t a = p & ~3u;
    c.w0 = lds_u32(c.rb | a);
    c.pr = a + 4u;
    c.w1 = lds_u32(c.rb | (c.pr & 127u));
    c.o = (p & 3u) * 8u;
}

__device__ __forceinline__ uint32_t fwin_bytes(const Chain& c) {
    uint32_t v;
    asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(v) : "r"(c.w0), "r"(c.w1), "r"(c.o));
    return v;
}

// consume s - kSelBase bytes (see win_advance); the word address wraps in the ring
__device__ __forceinline__ void fwin_advance(Chain& c, uint32_t s) {
    asm volatile(
        "{\n\t.reg .pred q;\n\t.reg .u32 a;\n\t"
        "mad.lo.u32 %3, %5, 8, %3;\n\t"
        "setp.ge.u32 q, %3, 0x10840;\n\t"
        "@q mov.b32 %0, %1;\n\t"
        "@q add.u32 %2, %2, 4;\n\t"
        "lop3.b32 a, %2, 127, %4, 0xEA;\n\t"
        "@q ld.shared.u32 %1, [a];\n\t"
        "and.b32 %3, %3, 31;\n\t}"
        : "+r"(c.w0), "+r"(c.w1), "+r"(c.pr), "+r"(c.o)
        : "r"(c.rb), "r"(s));
}

// Fast-path advance for pair J (0..7) of a 16-symbol group, as
// win_advance_g (rans_common.cuh): o carries the J+1 pairs' selector bias
// (multiples of 32), the crossing test uses a per-pair immediate, the word
// move is SEL + predicated add / LDS; fwin_rebase() once per group.
template <int J>
__device__ __forceinline__ void fwin_advance_g(Chain& c, uint32_t s) {
    asm volatile(
        "{\n\t.reg .pred q;\n\t.reg .u32 a;\n\t"
        "mad.lo.u32 %3, %5, 8, %3;\n\t"
        "setp.ge.u32 q, %3, %6;\n\t"
        "selp.b32 %0, %1, %0, q;\n\t"
        "@q add.u32 %2, %2, 4;\n\t"
        "lop3.b32 a, %2, 127, %4, 0xEA;\n\t"
        "@q ld.shared.u32 %1, [a];\n\t"
        "@q add.u32 %3, %3, -32;\n\t}"
        : "+r"(c.w0), "+r"(c.w1), "+r"(c.pr), "+r"(c.o)
        : "r"(c.rb), "r"(s), "n"(32u + (J + 1) * 0x10820u));
}
__device__ __forceinline__ void fwin_rebase(Chain& c) { c.o -= 8u * 0x10820u; }


#ifndef DC_FUSED_CLAMP
#define DC_FUSED_CLAMP 1  // never request stream bytes past the chain's end (+ the window's 8-byte look-ahead)
#endif
__device__ __forceinline__ void ring_refill(Chain& c, uint32_t ring_base) {
    if (c.mode <= 1 && ring_avail(c) < 96u && (!DC_FUSED_CLAMP || c.gfill < c.gend + 8)) {
        cp_async16(ring_base + ((uint32_t)c.gfill & 127u), reinterpret_cast<const void*>(c.gfill));
        cp_async16(ring_base + ((uint32_t)(c.gfill + 16) & 127u), reinterpret_cast<const void*>(c.gfill + 16));
        c.gfill += 32;
    }
}

// Generic (mixed-mode) step: returns the next weight byte of chain c.
__device__ __forceinline__ uint32_t chain_step(Chain& c, const FmaK& k) {
    if (kWindow) {
        if (c.mode == 0) {
            uint32_t sel = kSelBase;
            const uint32_t e = dec_sym(c.x, sel, fwin_bytes(c), c.tab);
            fwin_advance(c, sel);
            return e;
        }
        if (c.mode == 1) {
            const uint32_t e = fwin_bytes(c) & 0xFFu;
            fwin_advance(c, kSelBase + 1);
            return e;
        }
        return c.sym;
    }
    if (c.mode == 0) return ring_step(c.x, c.pr, c.nb, c.tab, c.rb, k);
    if (c.mode == 1) {
        const uint32_t e = c.nb;
        ++c.pr;
        c.nb = lds_u8((c.pr & 127u) | c.rb);
        return e;
    }
    return c.sym;
}

__global__ void __launch_bounds__(kRThreads, 1) k_fused_ring(
    const uint8_t* __restrict__ base, const uint64_t* __restrict__ blob_off, const uint64_t* __restrict__ blob_len,
    const uint64_t* __restrict__ out_len, const uint8_t* __restrict__ codec, uint64_t chunk_size,
    const int64_t* __restrict__ seg_base, const uint32_t* __restrict__ seg_state,
    const uint32_t* __restrict__ seg_off, const GemmTensorR* __restrict__ tens, const int4* __restrict__ items,
    int n_items, int ntok, int32_t* __restrict__ status, uint32_t one, const RingEpi* __restrict__ epi) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    const FmaK fk = fma_consts(one);
    RingSmem& S = *reinterpret_cast<RingSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int q = warp & 3, jj = warp >> 2;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kRSlots; ++s) {
            mbar_init(&S.empty[s], 1);
            S.cnt[s] = 0;
        }
        mbar_init(&S.done, 1);
        fence_mbar_init();
        S.cur[0] = S.cur[1] = -1;
    }
    if (warp == 0) tmem_alloc(&S.tmem, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);  // this thread's TMEM lane quarter
    uint32_t slot = 0, sphase = 0, dphase = 0;               // ring position of the next K-step

    for (int ii = blockIdx.x; ii < n_items; ii += gridDim.x) {
        const int4 it = items[ii];
        const GemmTensorR T = tens[it.x];
        const int m0 = it.y, k0 = it.z, klen = it.w;
        const int nsteps = klen / 32;
        const int last_row = min(m0 + kRTiles * 128 - 1, T.n_rows - 1);
        const int c_lo = (int)(((uint64_t)T.t_off + (uint64_t)m0 * T.k + k0) / chunk_size);
        const int c_hi = (int)(((uint64_t)T.t_off + (uint64_t)last_row * T.k + k0 + klen - 1) / chunk_size);
        __syncthreads();  // previous item: epilogue reads and X reads are finished
        if (c_hi - c_lo > 1) {  // host never builds such items
            if (threadIdx.x == 0) atomicExch(&status[c_lo], DC_CHUNK_CHAIN);
            continue;
        }
        // ---- decode tables for the (at most two) chunks of this item
        for (int t = 0; t <= c_hi - c_lo; ++t) {
            const int ct = c_lo + t;
            if (S.cur[t] != ct) {
                __syncthreads();
                if (codec[ct] == 1) build_decode_table(base + blob_off[ct], S.tab[t]);
                __syncthreads();
                if (threadIdx.x == 0) S.cur[t] = ct;
            }
        }
        // ---- X slice -> SW128 atoms (generic stores, then proxy fence)
        {
            const int chunks16 = kRNT * (klen >> 4);
            for (int i = threadIdx.x; i < chunks16; i += kRThreads) {
                const int r = i % kRNT, cj = i / kRNT, s = cj >> 3, j = cj & 7;
                uint4 v = make_uint4(0, 0, 0, 0);
                if (r < ntok) v = *reinterpret_cast<const uint4*>(T.x + (int64_t)r * T.k + k0 + (cj << 4));
                *reinterpret_cast<uint4*>(&S.x[s][r * 128 + ((j ^ (r & 7)) << 4)]) = v;
            }
            fence_proxy_async_smem();
        }

        // ---- decoder chains: u = 0, 1 -> tiles 2*jj, 2*jj+1
        Chain ch[2];
        uint32_t ring_base[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            Chain& c = ch[u];
            const int t = 2 * jj + u;
            const int row = m0 + t * 128 + q * 32 + lane;
            const bool valid = row < T.n_rows;
            const uint64_t g = (uint64_t)T.t_off + (uint64_t)(valid ? row : m0) * T.k + k0;
            c.chunk = (int)(g / chunk_size);
            const uint32_t o = (uint32_t)(g - (uint64_t)c.chunk * chunk_size);
            const uint8_t* blob = base + blob_off[c.chunk];
            const TableSmem& TB = S.tab[c.chunk - c_lo];
            c.tab = smem_u32(TB.tab);
            ring_base[u] = smem_u32(S.ring[(warp * 2 + u) * 32 + lane]);
            c.x = kStateLower;
            c.xe = kStateLower;
            c.sym = 0;
            if (!valid) {
                c.mode = 3;
                c.gstart = c.gend = reinterpret_cast<uint64_t>(blob);
            } else if (codec[c.chunk] != 1) {
                c.mode = 1;
                c.gstart = reinterpret_cast<uint64_t>(blob) + o;
                c.gend = c.gstart + klen;
            } else {
                const uint64_t nseg = (out_len[c.chunk] + 255) / 256;
                const int64_t j = seg_base[c.chunk] + (o >> 8);
                const int64_t je = j + (klen >> 8);
                const uint64_t sbase = reinterpret_cast<uint64_t>(blob) + kHeaderBytes;
                const uint32_t plen = (uint32_t)(blob_len[c.chunk] - kHeaderBytes);
                const bool tail = (uint64_t)(o >> 8) + (klen >> 8) >= nseg;
                const uint32_t so = seg_off[j], se = tail ? plen : seg_off[je];
                c.x = seg_state[j];
                c.xe = tail ? kStateLower : seg_state[je];
                if (so > se || se > plen) {  // damaged index: an empty span and an
                    c.x = kStateLower;       // unreachable end state flag the chain
                    c.xe = 0xFFFFFFFFu;
                    c.gstart = c.gend = sbase;
                } else {
                    c.gstart = sbase + so;
                    c.gend = sbase + se;
                }
                c.mode = TB.single >= 0 ? 2 : 0;
                c.sym = TB.single >= 0 ? (uint32_t)TB.single : 0u;
            }
            c.gfill = c.gstart & ~(uint64_t)15;
            c.rb = ring_base[u];
            c.pr = ring_base[u] + ((uint32_t)c.gstart & 127u);
            if (c.mode <= 1) {  // prime the ring with 112 B: buffered bytes stay < 128, so
                                // (gfill - read) & 127 never aliases a full ring to empty
                for (int k = 0; k < 7; ++k) {
                    if (DC_FUSED_CLAMP && c.gfill >= c.gend + 8) break;
                    cp_async16(ring_base[u] + ((uint32_t)c.gfill & 127u), reinterpret_cast<const void*>(c.gfill));
                    c.gfill += 16;
                }
            }
        }
        cp_async_commit();
        cp_async_wait<0>();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (kWindow)
                fwin_init(ch[u], (uint32_t)ch[u].gstart & 127u);
            else
                ch[u].nb = lds_u8(ch[u].pr);
        }
        __syncthreads();  // tables and X slice visible (generic and async proxies)
        const bool fast = __all_sync(0xffffffffu, ch[0].mode == 0 && ch[1].mode == 0);

        for (int st = 0; st < nsteps; ++st) {
            mbar_wait(&S.empty[slot], sphase ^ 1u);  // MMAs of kRSlots steps ago have consumed this slot
            tc_fence_after();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t w[2][4];
                if (fast && kWindow) {
#pragma unroll
                    for (int v = 0; v < 16; v += 2) {  // a step pair shares one window word
                        uint32_t wv[2], sel[2], e0[2];
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            wv[u] = fwin_bytes(ch[u]);
                            sel[u] = kSelBase;
                            e0[u] = dec_sym_fa(ch[u].x, sel[u], wv[u], ch[u].tab - (1u << 26), fk);
                        }
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const uint32_t t = __byte_perm(
                                e0[u], dec_sym_fa(ch[u].x, sel[u], wv[u], ch[u].tab - (1u << 26), fk), 0x0040);
                            w[u][v >> 2] = (v & 2) ? __byte_perm(w[u][v >> 2], t, 0x5410) : t;
                        }
                        switch (v >> 1) {  // compile-time after unrolling
                            case 0: for (int u = 0; u < 2; ++u) fwin_advance_g<0>(ch[u], sel[u]); break;
                            case 1: for (int u = 0; u < 2; ++u) fwin_advance_g<1>(ch[u], sel[u]); break;
                            case 2: for (int u = 0; u < 2; ++u) fwin_advance_g<2>(ch[u], sel[u]); break;
                            case 3: for (int u = 0; u < 2; ++u) fwin_advance_g<3>(ch[u], sel[u]); break;
                            case 4: for (int u = 0; u < 2; ++u) fwin_advance_g<4>(ch[u], sel[u]); break;
                            case 5: for (int u = 0; u < 2; ++u) fwin_advance_g<5>(ch[u], sel[u]); break;
                            case 6: for (int u = 0; u < 2; ++u) fwin_advance_g<6>(ch[u], sel[u]); break;
                            default: for (int u = 0; u < 2; ++u) fwin_advance_g<7>(ch[u], sel[u]); break;
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 2; ++u) fwin_rebase(ch[u]);
                } else if (fast) {
#pragma unroll
                    for (int v = 0; v < 16; v += 2) {  // 3 PRMT per 4 output bytes
                        uint32_t e0[2];
#pragma unroll
                        for (int u = 0; u < 2; ++u)
                            e0[u] = ring_step(ch[u].x, ch[u].pr, ch[u].nb, ch[u].tab, ch[u].rb, fk);
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const uint32_t t = __byte_perm(
                                e0[u], ring_step(ch[u].x, ch[u].pr, ch[u].nb, ch[u].tab, ch[u].rb, fk), 0x0040);
                            w[u][v >> 2] = (v & 2) ? __byte_perm(w[u][v >> 2], t, 0x5410) : t;
                        }
                    }
                } else {  // bytes shift in from the top: no runtime index into w[]
#pragma unroll 1
                    for (int v = 0; v < 16; ++v) {
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            const uint32_t e = chain_step(ch[u], fk);
                            w[u][0] = __funnelshift_r(w[u][0], w[u][1], 8);
                            w[u][1] = __funnelshift_r(w[u][1], w[u][2], 8);
                            w[u][2] = __funnelshift_r(w[u][2], w[u][3], 8);
                            w[u][3] = __funnelshift_r(w[u][3], e, 8);
                        }
                    }
                }
                const uint32_t col = slot * 64 + h * 4;
                tmem_st4(tl + col + (2 * jj) * 8, w[0]);
                tmem_st4(tl + col + (2 * jj + 1) * 8, w[1]);
                ring_refill(ch[0], ring_base[0]);
                ring_refill(ch[1], ring_base[1]);
                cp_async_commit();
                cp_async_wait<1>();
            }
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0 && atom_add_acq_rel(&S.cnt[slot], 1u) == kRDec - 1) {
                // last warp of this K-step: every slice of the slot is in TMEM
                S.cnt[slot] = 0;
                tc_fence_after();
                constexpr uint32_t idesc = idesc_i8(128, kRNT);
                const int kk = st * 32;
                const uint64_t bdesc = sw128_kmajor_desc(smem_u32(S.x[kk >> 7]) + (kk & 127));
#pragma unroll
                for (int t = 0; t < kRTiles; ++t)
                    mma_ts(tmem + kRAcc + t * kRNT, tmem + slot * 64 + t * 8, bdesc, idesc, st > 0);
                mma_commit(&S.empty[slot]);
                if (st == nsteps - 1) mma_commit(&S.done);
            }
            __syncwarp();
            if (++slot == kRSlots) {
                slot = 0;
                sphase ^= 1u;
            }
        }

        // ---- chain checks (state and position must meet the next split point)
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const Chain& c = ch[u];
            if (c.mode == 0) {
                const uint64_t pos = c.gfill - (uint64_t)ring_avail(c);
                if (c.x != c.xe || pos != c.gend) atomicExch(&status[c.chunk], DC_CHUNK_CHAIN);
            } else if (c.mode == 2 && (c.x != c.xe || c.gstart != c.gend)) {
                atomicExch(&status[c.chunk], DC_CHUNK_CORRUPT);
            }
        }

        // ---- epilogue: accumulators of tiles 2*jj, 2*jj+1 for this lane quarter
        mbar_wait(&S.done, dphase);
        dphase ^= 1u;
        tc_fence_after();
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            uint32_t acc[16];
            tmem_ld_32x32b_x16(tl + kRAcc + (2 * jj + u) * kRNT, acc);
            const int row = m0 + (2 * jj + u) * 128 + q * 32 + lane;
            if (row < T.n_rows) {
#pragma unroll
                for (int t = 0; t < kRNT; ++t)
                    if (t < ntok) atomicAdd(&T.acc[(int64_t)t * T.n_rows + row], (int32_t)acc[t]);
            }
        }
        tc_fence_before();
        if (epi != nullptr && epi[it.x].y != nullptr) {  // uniform per item
            const RingEpi E = epi[it.x];
            const int blk = m0 / (kRTiles * 128);
            __syncthreads();  // every thread's accumulator atomics are issued
            if (threadIdx.x == 0) {
                __threadfence();
                S.last = atomicAdd(&E.cnt[blk], 1u) == (uint32_t)E.n_slices - 1;
            }
            __syncthreads();
            if (S.last) {
                __threadfence();
                const int rows = min(kRTiles * 128, T.n_rows - m0);
                const float scale = E.sx ? (float)(*E.sx * E.sw) : E.scale;
                for (int i = threadIdx.x; i < rows * ntok; i += kRThreads) {
                    const int t = i / rows, r = m0 + i % rows;
                    const int32_t a = __ldcg(&T.acc[(int64_t)t * T.n_rows + r]);
                    E.y[(int64_t)t * T.n_rows + r] = (float)a * scale;
                }
                if (threadIdx.x == 0) E.cnt[blk] = 0;  // ready for the next launch
            }
        }
    }
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, 512);
}

}  // namespace dc

using namespace dc;

extern "C" int dc_fused_item_rows(void) { return kRTiles * 128; }
extern "C" int dc_fused_item_k(void) { return kFK; }
extern "C" int dc_fused_epi_bytes(void) { return (int)sizeof(RingEpi); }

// items: int4 (layer, m0, k0, klen): 1024 rows from m0, K-slice [k0, k0+klen),
// klen a multiple of 256 and <= dc_fused_item_k(); index seg_shift 8;
// chunk_size and layer offsets multiples of 256; an item's rows span <= 2 chunks.
extern "C" int dc_fused_ring_gemm(const uint8_t* base, const uint64_t* blob_off, const uint64_t* blob_len,
                                  const uint64_t* out_len, const uint8_t* codec, uint64_t chunk_size,
                                  const int64_t* seg_base, const uint32_t* seg_state, const uint32_t* seg_off,
                                  const void* tens, const int32_t* items, int64_t n_items, int ntok,
                                  int32_t* status, const void* epi, int max_ctas, void* stream) {
    if (n_items <= 0 || ntok <= 0 || ntok > kRNT || chunk_size % 256) return DC_ERR_ARG;
    const size_t smem = sizeof(RingSmem) + 1024;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_fused_ring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (max_ctas > 0 && max_ctas < sms) sms = max_ctas;  // leave SMs to a concurrent INT8 GEMM
    const int64_t grid = n_items < sms ? n_items : sms;
    k_fused_ring<<<(unsigned)grid, kRThreads, smem, (cudaStream_t)stream>>>(
        base, blob_off, blob_len, out_len, codec, chunk_size, seg_base, seg_state, seg_off,
        reinterpret_cast<const GemmTensorR*>(tens), reinterpret_cast<const int4*>(items), (int)n_items, ntok, status, 1u,
        reinterpret_cast<const RingEpi*>(epi));
    DC_CHECK_LAUNCH("k_fused_ring");
    return DC_OK;
}
