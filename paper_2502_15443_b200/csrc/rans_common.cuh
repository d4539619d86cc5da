// Shared rANS decode building blocks (table build, one-symbol step).
// Reference semantics: /root/reference/pkg/src/dcomp/ans.py:71-94, :301-313.
#pragma once
#include "common.cuh"
#include "ptx.cuh"

namespace dc {

// ------------------------------------------------------------------ tables
struct alignas(128) TableSmem {
    uint32_t tab[kProbScale];  // slot -> sym | (slot - cum) << 8 | f << 20
    uint32_t freq[256];
    uint32_t cum[256];
    int32_t present[256];
    int32_t npresent;
    int32_t single;  // symbol of a single-symbol table, else -1
    uint32_t warp_tot[4];
};

// Whole CTA (blockDim a multiple of 32, >= 128): unpack the u12 wire table
// (ans.py:256-262), fix up the single-symbol case (ans.py:292-295), exclusive
// cumulative sums (ans.py:301-304), and the slot table (ans.py:306-313) with
// a compact u32 entry.  Tables are validated beforehand by k_validate.
static __device__ void build_decode_table(const uint8_t* __restrict__ tb, TableSmem& T) {
    const int t = threadIdx.x;
    const bool owner = t < 128;  // warps 0-3 own symbol pairs (2t, 2t+1)
    uint32_t a = 0, b = 0, v = 0, inc = 0;
    if (owner) {
        unpack_pair(tb, t, a, b);
        // pack (frequency sum, present count) and scan both at once
        v = (a + b) | (((a != 0) + (b != 0)) << 16);
        inc = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
            if ((t & 31) >= d) inc += o;
        }
        if ((t & 31) == 31) T.warp_tot[t >> 5] = inc;
    }
    __syncthreads();
    const uint32_t total = T.warp_tot[0] + T.warp_tot[1] + T.warp_tot[2] + T.warp_tot[3];
    if (owner) {
        uint32_t carry = 0;
        for (int w = 0; w < (t >> 5); ++w) carry += T.warp_tot[w];
        const uint32_t ex = carry + inc - v;
        const uint32_t c0 = ex & 0xFFFF;
        uint32_t k0 = ex >> 16;
        T.freq[2 * t] = a;
        T.freq[2 * t + 1] = b;
        T.cum[2 * t] = c0;
        T.cum[2 * t + 1] = c0 + a;
        if (a) T.present[k0++] = 2 * t;
        if (b) T.present[k0] = 2 * t + 1;
    }
    if (t == 0) {
        T.npresent = total >> 16;
        T.single = -1;
    }
    __syncthreads();
    if ((total & 0xFFFF) == kProbScale - 1) {  // validated: exactly one nonzero entry
        if (t == 0) {
            const int s = T.present[0];
            T.single = s;
            T.freq[s] = kProbScale;
        }
        __syncthreads();
        return;
    }
    // fill: warps take present symbols round-robin, lanes stride the slots
    const int np = T.npresent;
    const int lane = t & 31, nw = blockDim.x >> 5;
    for (int i = t >> 5; i < np; i += nw) {
        const uint32_t s = T.present[i];
        const uint32_t f = T.freq[s], c = T.cum[s];
        // bounded even for an invalid table (callers skip such chunks anyway)
        for (uint32_t k = lane; k < f && c + k < kProbScale; k += 32) T.tab[c + k] = s | (k << 8) | (f << 20);
    }
    __syncthreads();
}

// One symbol: table lookup, state update, renormalization.  `p` is the
// 32-bit shared address of the next unread stream byte and `nb` that byte
// (prefetched, so the common single-byte refill never waits on a load);
// x = f*(x>>12) + bias is formed as (e>>20)*((x>>12) - 4096) + (e>>8), since
// e>>8 == bias + 4096*f (mod 2^32, exact: the true value is < 2^28).  The
// second refill (only symbols with f < 16 can need it) is a warp-uniform
// branch when kConverged (all 32 lanes execute the step).
__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u8(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}

// ---- word-window decoding ------------------------------------------------
// The stream is read through an 8-byte window of two aligned shared words
// (w0 holds the next unread byte at bit offset o, w1 the word after; wa is
// the shared address of w1).  A step PAIR needs at most 4 stream bytes, so
// both steps take their bytes from one funnel-shifted word v = bytes[p, p+4)
// with PRMT (x = x << 8 | v.byte[s&3], selector s counts bytes used), and the
// window moves at most one word per pair: one predicated LDS.32 per pair
// instead of two predicated LDS.U8 per step.  Fully predicated-off shared
// loads cost no wavefront, and only ~1 in 4 lanes crosses a word per pair.
constexpr uint32_t kSelBase = 0x2104;  // PRMT: {x.b2, x.b1, x.b0, v.b[sel&3]}

struct Win {
    uint32_t w0, w1, wa, o;
};

__device__ __forceinline__ void win_init(Win& w, uint32_t p) {
    const uint32_t a = p & ~3u;
    w.w0 = lds_u32(a);
    w.w1 = lds_u32(a + 4);
    w.wa = a + 4;
    w.o = (p & 3u) * 8u;
}
// shared address of the next unread byte
__device__ __forceinline__ uint32_t win_pos(const Win& w) { return w.wa - 4u + (w.o >> 3); }

__device__ __forceinline__ uint32_t win_bytes(const Win& w) {
    uint32_t v;
    asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(v) : "r"(w.w0), "r"(w.w1), "r"(w.o));
    return v;
}

// One symbol: table lookup, state update, up to two refill bytes from v.
__device__ __forceinline__ uint32_t dec_sym(uint32_t& x, uint32_t& s, uint32_t v, uint32_t tab) {
    uint32_t e;
    asm volatile(
        "{\n\t.reg .pred q;\n\t.reg .u32 a, f, b, t;\n\t"
        "and.b32 a, %0, 4095;\n\t"
        "mad.lo.u32 a, a, 4, %4;\n\t"
        "ld.shared.u32 %2, [a];\n\t"
        "shr.u32 f, %2, 20;\n\t"
        "shr.u32 b, %2, 8;\n\t"
        "shr.u32 t, %0, 12;\n\t"
        "sub.u32 t, t, 4096;\n\t"
        "mad.lo.u32 %0, f, t, b;\n\t"
        "setp.lt.u32 q, %0, 0x100000;\n\t"
        "@q prmt.b32 %0, %0, %3, %1;\n\t"
        "@q add.u32 %1, %1, 1;\n\t"
        "setp.lt.u32 q, %0, 0x100000;\n\t"
        "@q prmt.b32 %0, %0, %3, %1;\n\t"
        "@q add.u32 %1, %1, 1;\n\t}"
        : "+r"(x), "+r"(s), "=r"(e)
        : "r"(v), "r"(tab));
    return e;
}

// Pipe balancing: shifts and LEA run on the ALU pipe, which the decode loop
// saturates; IMAD / IMAD.HI by a constant held in a register (opaque to ptxas,
// so it cannot turn them back into shifts) run on the FMA pipe instead.
struct FmaK {
    uint32_t c4, c2p12, c2p24, c2p20, cm4096, cm16384, c1;
};
__device__ __forceinline__ FmaK fma_consts(uint32_t one) {
    return FmaK{4u * one, 4096u * one, (1u << 24) * one, (1u << 20) * one, 0u - 4096u * one, 0u - 16384u * one,
                one};
}

// Slot address without the ALU mask: with t = (x >> 12) - 4096 (needed for the
// state update anyway), tab + 4*(x & 4095) = (tab - 2^26) + 4x - 16384 t: two
// IMADs on the FMA pipe instead of LOP3 + IMAD.  `tabm` = tab - 2^26.
__device__ __forceinline__ uint32_t dec_sym_fa(uint32_t& x, uint32_t& s, uint32_t v, uint32_t tabm, const FmaK& k) {
    uint32_t e;
    asm volatile(
        "{\n\t.reg .pred q;\n\t.reg .u32 a, f, b, t;\n\t"
        "shr.u32 t, %0, 12;\n\t"
        "sub.u32 t, t, 4096;\n\t"
        "mad.lo.u32 a, %0, %5, %4;\n\t"
        "mad.lo.u32 a, t, %6, a;\n\t"
        "ld.shared.u32 %2, [a];\n\t"
        "shr.u32 f, %2, 20;\n\t"
        "shr.u32 b, %2, 8;\n\t"
        "mad.lo.u32 %0, f, t, b;\n\t"
        "setp.lt.u32 q, %0, 0x100000;\n\t"
        "@q prmt.b32 %0, %0, %3, %1;\n\t"
        "@q add.u32 %1, %1, 1;\n\t"
        "setp.lt.u32 q, %0, 0x100000;\n\t"
        "@q prmt.b32 %0, %0, %3, %1;\n\t"
        "@q add.u32 %1, %1, 1;\n\t}"
        : "+r"(x), "+r"(s), "=r"(e)
        : "r"(v), "r"(tabm), "r"(k.c4), "r"(k.cm16384));
    return e;
}

__device__ __forceinline__ uint32_t dec_sym(uint32_t& x, uint32_t& s, uint32_t v, uint32_t tab, const FmaK& k) {
    uint32_t e;
    asm volatile(
        "{\n\t.reg .pred q;\n\t.reg .u32 a, f, b, t;\n\t"
        "and.b32 a, %0, 4095;\n\t"
        "mad.lo.u32 a, a, %5, %4;\n\t"
        "ld.shared.u32 %2, [a];\n\t"
        "mul.hi.u32 f, %2, %6;\n\t"
        "shr.u32 b, %2, 8;\n\t"
        "mad.hi.u32 t, %0, %8, %9;\n\t"
        "mad.lo.u32 %0, f, t, b;\n\t"
        "setp.lt.u32 q, %0, 0x100000;\n\t"
        "@q prmt.b32 %0, %0, %3, %1;\n\t"
        "@q add.u32 %1, %1, 1;\n\t"
        "setp.lt.u32 q, %0, 0x100000;\n\t"
        "@q prmt.b32 %0, %0, %3, %1;\n\t"
        "@q add.u32 %1, %1, 1;\n\t}"
        : "+r"(x), "+r"(s), "=r"(e)
        : "r"(v), "r"(tab), "r"(k.c4), "r"(k.c2p12), "r"(k.c2p24), "r"(k.c2p20), "r"(k.cm4096));
    return e;
}

// Consume s - kSelBase bytes; slide the window by a word when o crosses 32.
// (o + 8*s is biased by 8*kSelBase = 0x10820, a multiple of 32.)
__device__ __forceinline__ void win_advance(Win& w, uint32_t s) {
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "mad.lo.u32 %3, %4, 8, %3;\n\t"
        "setp.ge.u32 q, %3, 0x10840;\n\t"
        "@q mov.b32 %0, %1;\n\t"
        "@q add.u32 %2, %2, 4;\n\t"
        "@q ld.shared.u32 %1, [%2];\n\t"
        "and.b32 %3, %3, 31;\n\t}"
        : "+r"(w.w0), "+r"(w.w1), "+r"(w.wa), "+r"(w.o)
        : "r"(s));
}

// Fast-path advance for pair J (0..7) of a 16-symbol group.  o is not
// re-biased per pair: it carries the selector bias of the J+1 pairs so far
// (8 * kSelBase = 0x10820 each, a multiple of 32, so SHF.R.W's shift amount
// o mod 32 is unaffected), the crossing test compares against a per-pair
// immediate, and win_rebase() removes the 8 pairs' bias once per group.  The
// word move is a predicated IMAD by an opaque 1 (FMA pipe; a SEL would load
// the busy ALU pipe) plus a predicated LDS and two predicated adds.
template <int J>
__device__ __forceinline__ void win_advance_gf(Win& w, uint32_t s, uint32_t one) {
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "mad.lo.u32 %3, %4, 8, %3;\n\t"
        "setp.ge.u32 q, %3, %5;\n\t"
        "@q mad.lo.u32 %0, %1, %6, 0;\n\t"
        "@q ld.shared.u32 %1, [%2+4];\n\t"
        "@q add.u32 %2, %2, 4;\n\t"
        "@q add.u32 %3, %3, -32;\n\t}"
        : "+r"(w.w0), "+r"(w.w1), "+r"(w.wa), "+r"(w.o)
        : "r"(s), "n"(32u + (J + 1) * 0x10820u), "r"(one));
}
__device__ __forceinline__ void win_rebase(Win& w) { w.o -= 8u * 0x10820u; }


__device__ __forceinline__ uint32_t put_byte(uint32_t w, uint32_t e, int k) {
    // byte k of the result <- byte 0 of e (PRMT)
    return __byte_perm(w, e, k == 0 ? 0x3214 : k == 1 ? 0x3240 : k == 2 ? 0x3410 : 0x4210);
}

}  // namespace dc
