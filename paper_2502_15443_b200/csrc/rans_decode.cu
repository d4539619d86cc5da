// rANS decoding of the DCC1 chunk payloads on B200 (sm_100a).
//
// Reference semantics (/root/reference/pkg/src/dcomp/ans.py):
//   blob   = u12 table (384 B) | u32 LE start state | stream        (:1-12)
//   decode = e = tab[x & 4095]; sym = e.sym;
//            x = f * (x >> 12) + (slot - cum); refill bytes while x < 2^20   (:71-94)
//   verdict: ok iff final x == 2^20 and all stream bytes consumed; bytes
//            past the stream read as zero (padding, :333-343).
//
// Three kernels:
//   k_validate        warp per chunk: the prologue checks (:284-299, :333-343, :364-367)
//   k_decode_segments the hot path: a task = up to 256 split-point segments of
//                     one chunk; the task's stream bytes are staged into shared
//                     memory with one TMA bulk copy, every lane decodes two
//                     segments interleaved (ILP 2) from its split point and
//                     writes output through a per-warp staging buffer as
//                     coalesced 16-byte stores.  Chain checks flag chunks whose
//                     segments do not meet (corrupt data) for an exact re-run.
//   k_decode_serial   CTA per chunk, one lane walks the whole stream exactly as
//                     the reference does (the verdict of record) and records
//                     the split points every 2^seg_shift symbols.
#include "common.cuh"
#include "ptx.cuh"
#include "rans_common.cuh"

namespace dc {

// --------------------------------------------------------------- validate
__global__ void k_validate(const uint8_t* __restrict__ base, const uint64_t* __restrict__ blob_off,
                           const uint64_t* __restrict__ blob_len, const uint64_t* __restrict__ out_len,
                           const uint8_t* __restrict__ codec, int64_t n, int32_t* __restrict__ status) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (w >= n) return;
    int st = DC_CHUNK_OK;
    if (codec[w] == 1) {
        const uint64_t len = blob_len[w];
        if (len < kHeaderBytes) {
            st = DC_CHUNK_TRUNC_TABLE;  // ans.py:365-366
        } else {
            const uint8_t* b = base + blob_off[w];
            uint32_t sum = 0, nz = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                uint32_t fa, fb;
                unpack_pair(b, lane * 4 + k, fa, fb);
                sum += fa + fb;
                nz += (fa != 0) + (fb != 0);
            }
#pragma unroll
            for (int d = 16; d; d >>= 1) {
                sum += __shfl_xor_sync(0xffffffffu, sum, d);
                nz += __shfl_xor_sync(0xffffffffu, nz, d);
            }
            const bool single = (sum == kProbScale - 1 && nz == 1);
            if (!single && sum != kProbScale) {
                st = DC_CHUNK_BAD_TABLE;  // ans.py:296-297
            } else {
                const uint32_t x0 = ld_u32_le_unaligned(b + kTableBytes);
                if (x0 < kStateLower || x0 >= kStateUpper)
                    st = DC_CHUNK_STATE_RANGE;  // ans.py:338-339
                else if (out_len[w] == 0 && (len != kHeaderBytes || x0 != kStateLower))
                    st = DC_CHUNK_EMPTY_BAD;  // ans.py:388-390
            }
        }
    }
    if (lane == 0) status[w] = st;
}

// ------------------------------------------------------------- serial decode
// One latency-shortened symbol step for the serial chain.  `e` is the table
// entry of the current state (loaded during the previous step).  The next
// state's slot is one of three candidates -- no refill (xn & 4095), one
// refill ((xn & 15) << 8 | b0) or two refills ((b0 & 15) << 8 | b1, which
// does not depend on xn at all) -- so all three table entries are loaded
// right after xn = f*t + b is known and the refill compares / PRMTs run in
// parallel with the loads; the right entry is selected afterwards.  Critical
// path per symbol: IMAD, LOP + IMAD, LDS, two SEL, SHF (the refills and the
// next t are off it).  Returns the symbol (low byte of the old entry).
__device__ __forceinline__ uint32_t serial_step(uint32_t& x, uint32_t& e, uint32_t& s, uint32_t v, uint32_t tab) {
    const uint32_t sym = e;
    // written as one asm block so the three loads stay unconditional (issued
    // as soon as their addresses exist) and only the selection waits on the
    // refill compares; ptxas would otherwise turn the selects into
    // predicated loads into one register, serialising them behind the compare.
    asm volatile(
        "{\n\t.reg .pred p1, p2;\n\t.reg .u32 f, b, t, xn, y2, b0, a0, a1, a2, e0, e1, e2, r1, r2, k;\n\t"
        "shr.u32 f, %1, 20;\n\t"
        "shr.u32 b, %1, 8;\n\t"
        "shr.u32 t, %0, 12;\n\t"
        "sub.u32 t, t, 4096;\n\t"
        "mad.lo.u32 xn, f, t, b;\n\t"                 // f*(x>>12) + slot - cum (mod 2^32)
        "mad.lo.u32 k, %2, 17, %5;\n\t"              // selector of (b0 << 8 | b1)
        "prmt.b32 y2, %3, 0, k;\n\t"
        "add.u32 k, %2, %6;\n\t"                      // selector of b0 (zero-extended)
        "prmt.b32 b0, %3, 0, k;\n\t"
        "and.b32 a2, y2, 4095;\n\t"
        "mad.lo.u32 a2, a2, 4, %4;\n\t"               // two refills: slot (b0 & 15) << 8 | b1
        "mad.lo.u32 b0, b0, 4, %4;\n\t"
        "and.b32 a0, xn, 4095;\n\t"
        "mad.lo.u32 a0, a0, 4, %4;\n\t"               // no refill: slot xn & 4095
        "and.b32 a1, xn, 15;\n\t"
        "mad.lo.u32 a1, a1, 1024, b0;\n\t"            // one refill: slot (xn & 15) << 8 | b0
        "ld.shared.u32 e2, [a2];\n\t"
        "ld.shared.u32 e0, [a0];\n\t"
        "ld.shared.u32 e1, [a1];\n\t"
        "setp.lt.u32 p1, xn, 0x100000;\n\t"
        "setp.lt.u32 p2, xn, 4096;\n\t"
        "prmt.b32 r1, xn, %3, %2;\n\t"
        "add.u32 k, %2, 1;\n\t"
        "prmt.b32 r2, r1, %3, k;\n\t"
        "selp.b32 r1, r2, r1, p2;\n\t"
        "selp.b32 %0, r1, xn, p1;\n\t"
        "selp.b32 e1, e2, e1, p2;\n\t"
        "selp.b32 %1, e1, e0, p1;\n\t"
        "selp.b32 k, 1, 0, p1;\n\t"
        "add.u32 %2, %2, k;\n\t"
        "selp.b32 k, 1, 0, p2;\n\t"
        "add.u32 %2, %2, k;\n\t}"
        : "+r"(x), "+r"(e), "+r"(s)
        : "r"(v), "r"(tab), "n"(0x4401u - 17u * kSelBase), "n"(0x4440u - kSelBase));
    return sym;
}

// One CTA per chunk: the whole CTA builds the table, then one thread walks
// the stream exactly as the reference does.  That walk is a serial
// recurrence, so its speed is its dependency chain: the stream is staged into
// a 4 x 4 KB shared ring by bulk async copies issued ahead of the reader
// (no global-memory latency on the chain) and read through the same two-word
// window and PRMT refills as the segment decoder; output leaves as 16-byte
// stores.  Bytes past the stream are never consumed by a valid chunk; a
// corrupt one ends with p != plen whatever it read (verdict unchanged).
constexpr int kSerialThreads = 128;
constexpr uint32_t kSerSlot = 4096;
constexpr uint32_t kSerRing = 4 * kSerSlot;

struct SerialSmem {
    TableSmem T;
    alignas(128) uint8_t ring[kSerRing];
    uint64_t bar[4];
};

__global__ void __launch_bounds__(kSerialThreads) k_decode_serial(
    const uint8_t* __restrict__ base, const uint64_t* __restrict__ blob_off, const uint64_t* __restrict__ blob_len,
    const uint64_t* __restrict__ out_off, const uint64_t* __restrict__ out_len, const int32_t* __restrict__ ids,
    int64_t n_ids, uint8_t* __restrict__ out, uint32_t seg_shift, const int64_t* __restrict__ seg_base,
    uint32_t* __restrict__ seg_state, uint32_t* __restrict__ seg_off, int32_t* __restrict__ status) {
    __shared__ SerialSmem S;
    TableSmem& T = S.T;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&S.bar[i], 1);
        fence_mbar_init();
    }
    uint32_t ph_base = 0;  // completions per slot so far (same for every slot at a chunk start)
    for (int64_t id = blockIdx.x; id < n_ids; id += gridDim.x) {
        const int c = ids[id];
        const int32_t st0 = status[c];
        if (st0 != DC_CHUNK_OK && st0 != DC_CHUNK_CHAIN) continue;  // prologue error: never decoded
        const uint8_t* blob = base + blob_off[c];
        const uint64_t n = out_len[c];
        if (n == 0) continue;
        const uint64_t plen = blob_len[c] - kHeaderBytes;
        const uint32_t x0 = ld_u32_le_unaligned(blob + kTableBytes);
        uint8_t* o = out + out_off[c];
        __syncthreads();
        build_decode_table(blob, T);
        const uint32_t K = 1u << seg_shift;
        const int64_t sb = seg_state ? seg_base[c] : 0;
        if (T.single >= 0) {
            // f = 4096: the state never changes and no byte is ever read.
            const uint8_t sym = (uint8_t)T.single;
            for (uint64_t i = threadIdx.x; i < n; i += blockDim.x) o[i] = sym;
            if (seg_state)
                for (uint64_t j = threadIdx.x; j < ((n + K - 1) >> seg_shift); j += blockDim.x) {
                    seg_state[sb + j] = x0;
                    seg_off[sb + j] = 0;
                }
            if (threadIdx.x == 0) status[c] = (x0 == kStateLower && plen == 0) ? DC_CHUNK_OK : DC_CHUNK_CORRUPT;
            continue;
        }
        if (threadIdx.x != 0) continue;
        // ---- staged stream: bytes [a16, a16 + stage_len) in 4 KB blocks, block b in slot b & 3
        const uint64_t gs = reinterpret_cast<uint64_t>(blob) + kHeaderBytes;
        const uint64_t a16 = gs & ~(uint64_t)15;
        const uint32_t delta = (uint32_t)(gs - a16);
        const uint64_t stage_len = (delta + plen + 15) & ~(uint64_t)15;
        const uint64_t nblk = (stage_len + kSerSlot - 1) / kSerSlot;
        const uint32_t ring = smem_u32(S.ring);
        uint64_t issued = 0, ready = 0;
        auto issue_upto = [&](uint64_t lim) {  // blocks < lim, at most 4 in flight
            for (; issued < lim && issued < nblk; ++issued) {
                const uint32_t slot = (uint32_t)(issued & 3);
                const uint64_t off = issued * kSerSlot;
                const uint32_t bytes = (uint32_t)min((uint64_t)kSerSlot, stage_len - off);
                fence_proxy_async_smem();
                mbar_arrive_expect_tx(&S.bar[slot], bytes);
                bulk_g2s(S.ring + slot * kSerSlot, reinterpret_cast<const void*>(a16 + off), bytes, &S.bar[slot]);
            }
        };
        auto wait_upto = [&](uint64_t need) {  // blocks <= need are in the ring
            for (; ready <= need && ready < nblk; ++ready) {
                const uint32_t slot = (uint32_t)(ready & 3);
                mbar_wait(&S.bar[slot], (ph_base + (uint32_t)(ready >> 2)) & 1u);
            }
        };
        issue_upto(4);
        wait_upto((delta + 8) / kSerSlot);
        auto ldr = [&](uint32_t rel) { return lds_u32(ring + (rel & (kSerRing - 1))); };
        // window: w0 holds the next byte at bit offset o, w1 the next word; wrel = rel offset of w1
        // (32-bit: a chunk's stream is < 4 GiB).  One chain, so the step is
        // written for latency: the window moves with a predicated LDS instead
        // of a branch, and the symbol step uses the shortest (ALU) form.
        uint32_t wrel = (delta & ~3u) + 4;
        uint32_t w0 = ldr(wrel - 4), w1 = ldr(wrel), ob = (delta & 3u) * 8u;
        auto advance = [&](uint32_t sel) {
            asm volatile(
                "{\n\t.reg .pred q;\n\t.reg .u32 a;\n\t"
                "mad.lo.u32 %3, %5, 8, %3;\n\t"
                "setp.ge.u32 q, %3, 0x10840;\n\t"
                "@q mov.b32 %0, %1;\n\t"
                "@q add.u32 %2, %2, 4;\n\t"
                "and.b32 a, %2, 16383;\n\t"
                "add.u32 a, a, %4;\n\t"
                "@q ld.shared.u32 %1, [a];\n\t"
                "and.b32 %3, %3, 31;\n\t}"
                : "+r"(w0), "+r"(w1), "+r"(wrel), "+r"(ob)
                : "r"(ring), "r"(sel));
        };
        static_assert(kSerRing == 16384, "advance() masks ring offsets with 16383");
        auto rpos = [&]() { return (uint64_t)(wrel - 4 + (ob >> 3)); };  // rel offset of the next unread byte
        const uint32_t tab = smem_u32(T.tab);
        const bool oal = (reinterpret_cast<uintptr_t>(o) & 15) == 0;
        uint32_t x = x0;
        bool bad = false;
        uint64_t j = 0;
        // one 16-symbol group (split point recorded at segment starts)
        auto group16 = [&]() {
            if (seg_state && (j & (K - 1)) == 0) {
                seg_state[sb + (j >> seg_shift)] = x;
                seg_off[sb + (j >> seg_shift)] = (uint32_t)(rpos() - delta);
            }
            uint32_t w[4];
            uint32_t e = lds_u32(tab + 4u * (x & 4095u));  // entry of the current state
#pragma unroll
            for (int v = 0; v < 16; v += 2) {
                uint32_t vb, sel = kSelBase;
                asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(vb) : "r"(w0), "r"(w1), "r"(ob));
                const uint32_t e0 = serial_step(x, e, sel, vb, tab);
                const uint32_t t = __byte_perm(e0, serial_step(x, e, sel, vb, tab), 0x0040);
                w[v >> 2] = (v & 2) ? __byte_perm(w[v >> 2], t, 0x5410) : t;
                advance(sel);
            }
            if (oal) {
                *reinterpret_cast<uint4*>(o + j) = make_uint4(w[0], w[1], w[2], w[3]);
            } else {
#pragma unroll
                for (int k = 0; k < 16; ++k) o[j + k] = (uint8_t)(w[k >> 2] >> (8 * (k & 3)));
            }
            j += 16;
        };
        while (j < n) {
            // ring: a block of g groups reads at most 32 g bytes (+ the 8-byte window);
            // the waits and issues are done once per 64 symbols
            const uint64_t rp = rpos();
            const uint64_t left = n - j;
            const int groups = left >= 64 ? 4 : (left >= 16 ? 1 : 0);
            wait_upto((rp + 32 * (uint64_t)(groups ? groups : 1) + 8) / kSerSlot);
            issue_upto(rp / kSerSlot + 4);
            if (groups == 4) {
                group16();
                group16();
                group16();
                group16();
            } else if (groups == 1) {
                group16();
            } else {
                if (seg_state && (j & (K - 1)) == 0) {
                    seg_state[sb + (j >> seg_shift)] = x;
                    seg_off[sb + (j >> seg_shift)] = (uint32_t)(rp - delta);
                }
                for (; j < n; ++j) {
                    uint32_t vb, sel = kSelBase;
                    asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(vb) : "r"(w0), "r"(w1), "r"(ob));
                    o[j] = (uint8_t)dec_sym(x, sel, vb, tab);
                    advance(sel);
                }
            }
            if ((j & (kCheckBlock - 1)) == 0 || j == n) {
                if (rpos() - delta > plen) {  // ans.py:89-90 (memory safety; the verdict is corrupt)
                    bad = true;
                    break;
                }
            }
        }
        if (x != kStateLower || rpos() - delta != plen) bad = true;  // ans.py:92-93
        status[c] = bad ? DC_CHUNK_CORRUPT : DC_CHUNK_OK;
        // drain: every issued block completes before its slot's barrier is reused
        wait_upto(issued - 1);
        if (issued > 0) {
            // keep all four slots' phases in step for the next chunk
            const uint64_t rounds = (issued + 3) / 4;
            for (uint64_t b = issued; b < rounds * 4; ++b) {  // dummy completions for unused slots
                const uint32_t slot = (uint32_t)(b & 3);
                mbar_arrive(&S.bar[slot]);
                mbar_wait(&S.bar[slot], (ph_base + (uint32_t)(b >> 2)) & 1u);
            }
            ph_base += (uint32_t)rounds;
        }
    }
}

// ---------------------------------------------------------- segment decode
constexpr int kDecIlp = 2;                        // segments per lane, interleaved
constexpr uint32_t kStageSlack = 2 * 1024 + 128;  // over-read room (>= 2 * max segment + 1)
constexpr int kOutLine = 32;                      // bytes per lane-segment per flush
constexpr int kOutStride = 32;                    // + XOR swizzle of the 16-B halves (see swz)
constexpr int kOutWarpBytes = kDecIlp * 32 * kOutStride;

// Two CTA shapes.  Wide: 8 warps, 512-segment tasks, 72 KB stream staging,
// 2 CTAs/SM -- the large-chunk configuration.  Narrow: 4 warps, 256-segment
// tasks, 45 KB staging, 3 CTAs/SM -- a 64 KiB chunk (256 segments) then
// still gives every lane two interleaved chains instead of one.
template <int TH, int MINB, uint32_t STAGE, int DESC>
struct DecCfg {
    static constexpr int kDescBatch = DESC;
    static constexpr int kThreads = TH;
    static constexpr int kMinBlocks = MINB;
    static constexpr int kWarps = TH / 32;
    static constexpr int kTaskSegs = TH * kDecIlp;
    static constexpr uint32_t kStageCap = STAGE;
    // dynamic smem carve-up (constant offsets keep the shared address space visible)
    static constexpr uint32_t kOffTab = 0;
    static constexpr uint32_t kOffStage = ((sizeof(TableSmem) + 127) / 128) * 128;
    static constexpr uint32_t kOffOut = kOffStage + kStageCap + kStageSlack;
    static constexpr uint32_t kOffBar = kOffOut + kWarps * kOutWarpBytes;
    static constexpr uint32_t kOffDesc = kOffBar + 64;
    static constexpr size_t kSmem = kOffDesc + DESC * 64;
    static_assert(kOffStage % 128 == 0 && kOffOut % 16 == 0 && kOffBar % 8 == 0, "smem carve-up alignment");
};
using WideCfg = DecCfg<256, 2, 72 * 1024, 32>;
using NarrowCfg = DecCfg<128, 3, 44 * 1024, 16>;
static_assert(WideCfg::kSmem * 2 + 2048 <= 228 * 1024 && NarrowCfg::kSmem * 3 + 3072 <= 228 * 1024,
              "CTAs per SM must fit in shared memory");

// 16-B half `h` of lane-segment `ls` in the output staging buffer.  Halves are
// swapped when bit 2 of the lane is set, which makes both the per-lane
// 16-B stores (8 lanes per phase) and the per-line 16-B reads conflict-free.
__device__ __forceinline__ uint32_t swz(int ls, int h) { return (uint32_t)(ls * kOutStride + ((h ^ ((ls >> 2) & 1)) << 4)); }

// One warp decodes NU segments per lane (segment r = warp*32 + lane + u*TH
// of the task) and writes them out through its staging buffer `ob`.
// Split points of a lane's (up to) two segments, loaded before the task's
// stream staging completes so the load latency hides behind the bulk copy.
struct LaneSplits {
    uint32_t x[2], so[2], xe[2], pe[2];
};

template <int NU, int TH>
__device__ __forceinline__ void decode_warp(uint32_t seg_shift, int s0, int ns, uint32_t lo, uint32_t hi,
                                            uint32_t delta, uint64_t olen, const LaneSplits& L,
                                            const uint32_t* tab_ptr, const uint8_t* stage_ptr, uint8_t* ob,
                                            uint8_t* __restrict__ obase, bool out_aligned, int32_t* st,
                                            const FmaK& fk) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t tab = smem_u32(tab_ptr), stage = smem_u32(stage_ptr);
    const uint32_t tabm = tab - (1u << 26);
    const uint32_t K = 1u << seg_shift;
    const int G = (int)(K >> 4);
    uint32_t x[NU], n[NU], xe[NU], pe[NU];
    Win W[NU];
    bool wild = false;  // a split point outside the staged span: never used as an address
#pragma unroll
    for (int u = 0; u < NU; ++u) {
        const int r = warp * 32 + lane + u * TH;
        const uint32_t rel = (uint32_t)(s0 + r);
        xe[u] = L.xe[u];
        pe[u] = L.pe[u];
        uint32_t p;
        if (r < ns) {
            x[u] = L.x[u];
            const uint32_t so = L.so[u];
            wild = wild || so < lo || so > hi;
            p = (so < lo || so > hi) ? stage : stage + so - lo + delta;
            const uint64_t rem = olen - ((uint64_t)rel << seg_shift);
            n[u] = rem < K ? (uint32_t)rem : K;
        } else {  // decodes harmless garbage from stage[0..2K), never written
            x[u] = kStateLower;
            p = stage;
            n[u] = 0;
        }
        win_init(W[u], p);
    }
    // Fast flush when every segment this warp writes is a whole K-byte
    // segment and the output is 16-B aligned (all but a chunk's last task):
    // per-line destinations are precomputed 32-bit offsets from the task base.
    bool ff = out_aligned;
#pragma unroll
    for (int u = 0; u < NU; ++u) ff = ff && (warp * 32 + lane + u * TH < ns) && n[u] == K;
    const bool fast_flush = __all_sync(0xffffffffu, ff);
    uint8_t* const tb = obase + ((uint64_t)(uint32_t)s0 << seg_shift);
    uint32_t dk[NU * 2];
#pragma unroll
    for (int k = 0; k < NU * 2; ++k) {
        const int pc = k * 32 + lane;
        dk[k] = ((uint32_t)(warp * 32 + ((pc >> 1) & 31) + (pc >> 6) * TH) << seg_shift) + (pc & 1) * 16;
    }
    // groups [0, g_full) are whole 16-symbol groups for every chain of the
    // warp (one warp-wide min instead of a vote per group)
    uint32_t my_full = 0xFFFFFFFFu;
#pragma unroll
    for (int u = 0; u < NU; ++u) my_full = min(my_full, n[u] == 0 ? 0xFFFFFFFFu : n[u] >> 4);
    const int g_full = (int)__reduce_min_sync(0xffffffffu, my_full);
    // staging slots of this lane's segments (shared addresses, loop-invariant)
    uint32_t stg[NU][2];
#pragma unroll
    for (int u = 0; u < NU; ++u) {
        stg[u][0] = smem_u32(ob) + swz(u * 32 + lane, 0);
        stg[u][1] = smem_u32(ob) + swz(u * 32 + lane, 1);
    }
    for (int g = 0; g < G; ++g) {
        const uint32_t g0 = (uint32_t)g << 4;
        uint32_t w[NU][4];
        if (g < g_full) {
#pragma unroll
            for (int v = 0; v < 16; v += 2) {  // step pairs share one window word
                uint32_t wv[NU], sel[NU];
#pragma unroll
                for (int u = 0; u < NU; ++u) {
                    wv[u] = win_bytes(W[u]);
                    sel[u] = kSelBase;
                }
                uint32_t e0[NU];
#pragma unroll
                for (int u = 0; u < NU; ++u) e0[u] = dec_sym_fa(x[u], sel[u], wv[u], tabm, fk);
#pragma unroll
                for (int u = 0; u < NU; ++u) {
                    // two symbols -> bytes 0,1 of t; two pairs -> one word (3 PRMT per 4 bytes)
                    const uint32_t t = __byte_perm(e0[u], dec_sym_fa(x[u], sel[u], wv[u], tabm, fk), 0x0040);
                    w[u][v >> 2] = (v & 2) ? __byte_perm(w[u][v >> 2], t, 0x5410) : t;
                }
#define WADV(J) win_advance_gf<J>(W[u], sel[u], fk.c1)
                switch (v >> 1) {  // compile-time after unrolling
                    case 0: for (int u = 0; u < NU; ++u) WADV(0); break;
                    case 1: for (int u = 0; u < NU; ++u) WADV(1); break;
                    case 2: for (int u = 0; u < NU; ++u) WADV(2); break;
                    case 3: for (int u = 0; u < NU; ++u) WADV(3); break;
                    case 4: for (int u = 0; u < NU; ++u) WADV(4); break;
                    case 5: for (int u = 0; u < NU; ++u) WADV(5); break;
                    case 6: for (int u = 0; u < NU; ++u) WADV(6); break;
                    default: for (int u = 0; u < NU; ++u) WADV(7); break;
                }
#undef WADV
            }
#pragma unroll
            for (int u = 0; u < NU; ++u) win_rebase(W[u]);
        } else {
#pragma unroll
            for (int u = 0; u < NU; ++u) w[u][0] = w[u][1] = w[u][2] = w[u][3] = 0;
#pragma unroll
            for (int v = 0; v < 16; ++v) {
#pragma unroll
                for (int u = 0; u < NU; ++u) {
                    if (g0 + v < n[u]) {
                        uint32_t sel = kSelBase;
                        const uint32_t e = dec_sym(x[u], sel, win_bytes(W[u]), tab, fk);
                        win_advance(W[u], sel);
                        w[u][v >> 2] = put_byte(w[u][v >> 2], e, v & 3);
                    }
                }
            }
        }
        const int slot = g & 1;
#pragma unroll
        for (int u = 0; u < NU; ++u)
            asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(stg[u][slot]), "r"(w[u][0]),
                         "r"(w[u][1]), "r"(w[u][2]), "r"(w[u][3])
                         : "memory");
        if (slot == 1) {  // G is even (K >= 64)
            __syncwarp();
            const uint32_t line0 = (uint32_t)(g >> 1) * kOutLine;
            if (fast_flush) {
#pragma unroll
                for (int k = 0; k < NU * 2; ++k) {
                    const int pc = k * 32 + lane;
                    st_na_v4(tb + dk[k] + line0,
                             *reinterpret_cast<const uint4*>(ob + swz((pc >> 6) * 32 + ((pc >> 1) & 31), pc & 1)));
                }
                __syncwarp();
                continue;
            }
#pragma unroll
            for (int k = 0; k < NU * 2; ++k) {
                const int pc = k * 32 + lane;
                const int u = pc >> 6, ln = (pc >> 1) & 31, part = pc & 1;
                const int r = warp * 32 + ln + u * TH;
                if (r >= ns) continue;
                const uint64_t seg_start = (uint64_t)(s0 + r) << seg_shift;
                const uint64_t rem = olen - seg_start;
                const uint32_t slen = rem < K ? (uint32_t)rem : K;
                const uint32_t boff = line0 + part * 16;
                if (boff >= slen) continue;
                const uint8_t* src = ob + swz(u * 32 + ln, part);
                uint8_t* dst = obase + seg_start + boff;
                const uint32_t nbytes = min(16u, slen - boff);
                if (nbytes == 16 && out_aligned) {
                    st_na_v4(dst, *reinterpret_cast<const uint4*>(src));
                } else {
                    for (uint32_t i = 0; i < nbytes; ++i) dst[i] = src[i];
                }
            }
            __syncwarp();
        }
    }
    if (wild) atomicExch(st, DC_CHUNK_CHAIN);
    // chain checks: every segment must end exactly where the next one starts
#pragma unroll
    for (int u = 0; u < NU; ++u) {
        const int r = warp * 32 + lane + u * TH;
        if (r >= ns) continue;
        if (x[u] != xe[u] || win_pos(W[u]) - stage - delta + lo != pe[u]) atomicExch(st, DC_CHUNK_CHAIN);
    }
}

// Per-task header, filled for kDescBatch tasks at a time by warp 0 (one lane
// per task, the dependent task -> chunk -> split-point loads all in flight at
// once) so a task starts its stream copy without a global-load round trip.
struct alignas(16) TaskDesc {
    uint64_t blob;   // blob address (table | state | stream)
    uint64_t obase;  // chunk output address
    int64_t sb;      // first segment of the chunk in the index
    uint64_t olen;   // chunk output bytes
    uint32_t plen, lo, hi, nseg;
    int32_t c, s0, ns, st0;
};
static_assert(sizeof(TaskDesc) == 64, "TaskDesc layout");

template <class Cfg>
__global__ void __launch_bounds__(Cfg::kThreads, Cfg::kMinBlocks) k_decode_segments(
    const uint8_t* __restrict__ base, const uint64_t* __restrict__ blob_off, const uint64_t* __restrict__ blob_len,
    const uint64_t* __restrict__ out_off, const uint64_t* __restrict__ out_len, uint32_t seg_shift,
    const int64_t* __restrict__ seg_base, const uint32_t* __restrict__ seg_state,
    const uint32_t* __restrict__ seg_off, const int4* __restrict__ tasks, int64_t n_tasks,
    uint8_t* __restrict__ out, int32_t* __restrict__ status, uint32_t one) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const FmaK fk = fma_consts(one);
    TableSmem& T = *reinterpret_cast<TableSmem*>(smem + Cfg::kOffTab);
    uint8_t* stage = smem + Cfg::kOffStage;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::kOffBar);
    TaskDesc* desc = reinterpret_cast<TaskDesc*>(smem + Cfg::kOffDesc);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* ob = smem + Cfg::kOffOut + warp * kOutWarpBytes;
    const uint32_t K = 1u << seg_shift;

    const int64_t t_begin = (int64_t)blockIdx.x * n_tasks / gridDim.x;
    const int64_t t_end = (int64_t)(blockIdx.x + 1) * n_tasks / gridDim.x;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    int cur_chunk = -1;
    uint32_t phase = 0;

    for (int64_t ti = t_begin; ti < t_end; ++ti) {
        const int bi = (int)((ti - t_begin) % Cfg::kDescBatch);
        if (bi == 0) {
            __syncthreads();  // the previous batch's descriptors are no longer read
            if (warp == 0 && lane < Cfg::kDescBatch && ti + lane < t_end) {
                const int4 task = tasks[ti + lane];
                TaskDesc d;
                d.c = task.x;
                d.s0 = task.y;
                d.ns = task.z;
                d.st0 = status[d.c];
                d.blob = reinterpret_cast<uint64_t>(base + blob_off[d.c]);
                d.obase = reinterpret_cast<uint64_t>(out + out_off[d.c]);
                d.plen = (uint32_t)(blob_len[d.c] - kHeaderBytes);
                d.olen = out_len[d.c];
                d.nseg = (uint32_t)((d.olen + K - 1) >> seg_shift);
                d.sb = seg_base[d.c];
                d.lo = seg_off[d.sb + d.s0];
                d.hi = ((uint32_t)(d.s0 + d.ns) < d.nseg) ? seg_off[d.sb + d.s0 + d.ns] : d.plen;
                desc[lane] = d;
            }
        }
        __syncthreads();  // previous task done with stage[] and T; descriptors visible
        const TaskDesc& D = desc[bi];
        const int c = D.c, s0 = D.s0, ns = D.ns;
        // prologue errors (k_validate, same stream) are never decoded
        if (D.st0 >= DC_CHUNK_TRUNC_TABLE && D.st0 <= DC_CHUNK_EMPTY_BAD) continue;
        const uint8_t* blob = reinterpret_cast<const uint8_t*>(D.blob);
        const uint32_t plen = D.plen, lo = D.lo, hi = D.hi, nseg_chunk = D.nseg;
        const uint64_t olen = D.olen;
        const int64_t sb = D.sb;
        const uintptr_t gsrc = reinterpret_cast<uintptr_t>(blob) + kHeaderBytes + lo;
        const uintptr_t a16 = gsrc & ~(uintptr_t)15;
        const uint32_t delta = (uint32_t)(gsrc - a16);
        // a damaged index (hi < lo, or past the stream) is never staged: the
        // chunk goes to the exact serial decoder
        const uint32_t bytes = (hi >= lo && hi <= plen) ? ((hi - lo + delta + 15u) & ~15u) : 0xFFFFFFFFu;
        const bool stage_ok = bytes <= Cfg::kStageCap;

        if (threadIdx.x == 0) {
            fence_proxy_async_smem();
            const uint32_t nbytes = stage_ok ? bytes : 0u;
            mbar_arrive_expect_tx(bar, nbytes);
            for (uint32_t off = 0; off < nbytes; off += 16384u)
                bulk_g2s(stage + off, reinterpret_cast<const void*>(a16 + off), min(16384u, nbytes - off), bar);
        }
        // this lane's split points (and the chain-check targets: the next
        // split point), in flight while the stream is staged
        LaneSplits L;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int r = warp * 32 + lane + u * Cfg::kThreads;
            const uint32_t rel = (uint32_t)(s0 + r);
            const bool valid = r < ns, inner = valid && rel + 1 < nseg_chunk;
            L.x[u] = valid ? seg_state[sb + rel] : kStateLower;
            L.so[u] = valid ? seg_off[sb + rel] : 0u;
            L.xe[u] = inner ? seg_state[sb + rel + 1] : kStateLower;
            L.pe[u] = inner ? seg_off[sb + rel + 1] : plen;
        }
        if (c != cur_chunk) {
            build_decode_table(blob, T);  // overlaps the bulk copy
            cur_chunk = c;
        }
        mbar_wait(bar, phase);
        phase ^= 1u;
        if (!stage_ok) {  // index/host invariant broken: let the exact path decide
            if (threadIdx.x == 0) atomicExch(&status[c], DC_CHUNK_CHAIN);
            continue;
        }

        uint8_t* obase = reinterpret_cast<uint8_t*>(D.obase);
        const bool out_aligned = ((reinterpret_cast<uintptr_t>(obase) | (uintptr_t)K) & 15) == 0;

        if (T.single >= 0) {  // f = 4096: output is one repeated byte
            const uint64_t from = (uint64_t)s0 << seg_shift;
            uint64_t to = (uint64_t)(s0 + ns) << seg_shift;
            if (to > olen) to = olen;
            const uint8_t sym = (uint8_t)T.single;
            for (uint64_t i = from + threadIdx.x; i < to; i += blockDim.x) obase[i] = sym;
            if (threadIdx.x == 0 && s0 == 0) {
                const uint32_t x0 = ld_u32_le_unaligned(blob + kTableBytes);
                if (x0 != kStateLower || plen != 0) atomicExch(&status[c], DC_CHUNK_CORRUPT);
            }
            continue;
        }
        if (warp * 32 >= ns) continue;  // idle warp in a short task
        if (warp * 32 + Cfg::kThreads < ns)
            decode_warp<2, Cfg::kThreads>(seg_shift, s0, ns, lo, hi, delta, olen, L, T.tab, stage, ob, obase,
                                          out_aligned, &status[c], fk);
        else
            decode_warp<1, Cfg::kThreads>(seg_shift, s0, ns, lo, hi, delta, olen, L, T.tab, stage, ob, obase,
                                          out_aligned, &status[c], fk);
    }
}

// -------------------------------------------------------------- store copy
__global__ void k_store_copy(const uint8_t* __restrict__ base, const uint64_t* __restrict__ blob_off,
                             const uint64_t* __restrict__ out_off, const uint64_t* __restrict__ out_len,
                             const uint8_t* __restrict__ codec, int64_t n, uint8_t* __restrict__ out) {
    for (int64_t c = blockIdx.y; c < n; c += gridDim.y) {
        if (codec[c] != 0) continue;
        const uint8_t* s = base + blob_off[c];
        uint8_t* d = out + out_off[c];
        const uint64_t len = out_len[c];
        // align the destination, then 16-byte stores fed by funnel-shifted loads
        const uint32_t head = (uint32_t)((16 - (reinterpret_cast<uintptr_t>(d) & 15)) & 15);
        const uint64_t h = head < len ? head : len;
        for (uint64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < h; i += gridDim.x * blockDim.x) d[i] = s[i];
        const uint64_t body = (len - h) & ~(uint64_t)15;
        const uint8_t* s2 = s + h;
        uint8_t* d2 = d + h;
        const uint32_t mis = (uint32_t)(reinterpret_cast<uintptr_t>(s2) & 3);
        const uint32_t* sw = reinterpret_cast<const uint32_t*>(s2 - mis);
        for (uint64_t v = (uint64_t)(blockIdx.x * blockDim.x + threadIdx.x) * 16; v < body;
             v += (uint64_t)gridDim.x * blockDim.x * 16) {
            uint32_t wv[5];
#pragma unroll
            for (int k = 0; k < 5; ++k) wv[k] = (k < 4 || mis) ? __ldg(sw + v / 4 + k) : 0u;
            uint4 r;
            r.x = __funnelshift_r(wv[0], wv[1], 8 * mis);
            r.y = __funnelshift_r(wv[1], wv[2], 8 * mis);
            r.z = __funnelshift_r(wv[2], wv[3], 8 * mis);
            r.w = __funnelshift_r(wv[3], wv[4], 8 * mis);
            *reinterpret_cast<uint4*>(d2 + v) = r;
        }
        for (uint64_t i = h + body + blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x)
            d[i] = s[i];
    }
}

static int g_sm_count = 0;
int sm_count() {
    if (!g_sm_count) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
        if (g_sm_count <= 0) g_sm_count = 148;
    }
    return g_sm_count;
}

}  // namespace dc

using namespace dc;

extern "C" int dc_ans_validate(const uint8_t* base, const uint64_t* blob_off, const uint64_t* blob_len,
                               const uint64_t* out_len, const uint8_t* codec, int64_t n_chunks, int32_t* status,
                               void* stream) {
    if (n_chunks < 0) return DC_ERR_ARG;
    if (n_chunks == 0) return DC_OK;
    const int threads = 256;
    const int64_t blocks = (n_chunks * 32 + threads - 1) / threads;
    k_validate<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(base, blob_off, blob_len, out_len, codec,
                                                                      n_chunks, status);
    DC_CHECK_LAUNCH("k_validate");
    return DC_OK;
}

extern "C" int dc_ans_decode_serial(const uint8_t* base, const uint64_t* blob_off, const uint64_t* blob_len,
                                    const uint64_t* out_off, const uint64_t* out_len, const int32_t* chunk_ids,
                                    int64_t n_ids, uint8_t* out, uint32_t seg_shift, const int64_t* seg_base,
                                    uint32_t* seg_state, uint32_t* seg_off, int32_t* status, void* stream) {
    if (n_ids < 0 || (seg_state && (seg_shift < 4 || seg_shift > 20))) return DC_ERR_ARG;
    if (n_ids == 0) return DC_OK;
    const int64_t grid = n_ids < (int64_t)sm_count() * 12 ? n_ids : (int64_t)sm_count() * 12;
    k_decode_serial<<<(unsigned)grid, kSerialThreads, 0, (cudaStream_t)stream>>>(
        base, blob_off, blob_len, out_off, out_len, chunk_ids, n_ids, out, seg_shift, seg_base, seg_state, seg_off,
        status);
    DC_CHECK_LAUNCH("k_decode_serial");
    return DC_OK;
}

extern "C" int dc_decode_task_segments(void) { return WideCfg::kTaskSegs; }
extern "C" int dc_decode_narrow_segments(void) { return NarrowCfg::kTaskSegs; }
extern "C" int dc_decode_stage_cap(int narrow) { return (int)(narrow ? NarrowCfg::kStageCap : WideCfg::kStageCap); }

template <class Cfg>
static int launch_segments(const uint8_t* base, const uint64_t* blob_off, const uint64_t* blob_len,
                           const uint64_t* out_off, const uint64_t* out_len, uint32_t seg_shift,
                           const int64_t* seg_base, const uint32_t* seg_state, const uint32_t* seg_off,
                           const int32_t* tasks, int64_t n_tasks, uint8_t* out, int32_t* status, void* stream) {
    if (n_tasks < 0 || seg_shift < 6 || seg_shift > 10) return DC_ERR_ARG;
    if (n_tasks == 0) return DC_OK;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_decode_segments<Cfg>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::kSmem);
        attr = true;
    }
    const int64_t cap = (int64_t)sm_count() * Cfg::kMinBlocks;
    const int64_t grid = n_tasks < cap ? n_tasks : cap;
    k_decode_segments<Cfg><<<(unsigned)grid, Cfg::kThreads, Cfg::kSmem, (cudaStream_t)stream>>>(
        base, blob_off, blob_len, out_off, out_len, seg_shift, seg_base, seg_state, seg_off,
        reinterpret_cast<const int4*>(tasks), n_tasks, out, status, 1u);
    DC_CHECK_LAUNCH("k_decode_segments");
    return DC_OK;
}

extern "C" int dc_ans_decode_segments(const uint8_t* base, const uint64_t* blob_off, const uint64_t* blob_len,
                                      const uint64_t* out_off, const uint64_t* out_len, uint32_t seg_shift,
                                      const int64_t* seg_base, const uint32_t* seg_state, const uint32_t* seg_off,
                                      const int32_t* tasks, int64_t n_tasks, uint8_t* out, int32_t* status,
                                      void* stream) {
    return launch_segments<WideCfg>(base, blob_off, blob_len, out_off, out_len, seg_shift, seg_base, seg_state,
                                    seg_off, tasks, n_tasks, out, status, stream);
}

extern "C" int dc_ans_decode_segments_narrow(const uint8_t* base, const uint64_t* blob_off,
                                             const uint64_t* blob_len, const uint64_t* out_off,
                                             const uint64_t* out_len, uint32_t seg_shift, const int64_t* seg_base,
                                             const uint32_t* seg_state, const uint32_t* seg_off,
                                             const int32_t* tasks, int64_t n_tasks, uint8_t* out, int32_t* status,
                                             void* stream) {
    return launch_segments<NarrowCfg>(base, blob_off, blob_len, out_off, out_len, seg_shift, seg_base, seg_state,
                                      seg_off, tasks, n_tasks, out, status, stream);
}

extern "C" int dc_store_copy(const uint8_t* base, const uint64_t* blob_off, const uint64_t* out_off,
                             const uint64_t* out_len, const uint8_t* codec, int64_t n_chunks, uint8_t* out,
                             void* stream) {
    if (n_chunks < 0) return DC_ERR_ARG;
    if (n_chunks == 0) return DC_OK;
    dim3 grid(8, (unsigned)(n_chunks < 65535 ? n_chunks : 65535));
    k_store_copy<<<grid, 256, 0, (cudaStream_t)stream>>>(base, blob_off, out_off, out_len, codec, n_chunks, out);
    DC_CHECK_LAUNCH("k_store_copy");
    return DC_OK;
}
