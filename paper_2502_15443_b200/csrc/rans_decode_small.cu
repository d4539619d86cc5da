// Split-point rANS decode for SMALL chunks (<= 32 KiB; BASELINE config C3's
// 16-64 KiB end).  Reference semantics as rans_decode.cu (ans.py:71-94).
//
// The main kernel (k_decode_segments) works on CTA-wide tasks of up to 512
// segments of ONE chunk with a 16 KB slot table per CTA: a 16 KiB chunk has
// only 64 segments, so 7/8 of its lanes idle and every task rebuilds a table.
// Here the unit is a WARP task (<= 64 segments, 2 per lane, ILP 2) and each
// warp owns a compact table:
//   symtab[slot] = symbol (4096 x u8)            slot -> symbol
//   info[sym]    = (f, 4096*f - cum)  (256 x u64) symbol -> state update
//   x' = f*((x >> 12) - 4096) + slot + (4096 f - cum) = f*(x >> 12) + slot - cum
// 6 KB instead of 16 KB, so 8 warps x 8 KB fit two CTAs per SM.  Stream bytes
// are read straight from global memory (L1-resident after a per-lane
// prefetch of the segment) through the same two-word window as the main
// kernel; outputs leave through the same swizzled per-warp staging.
#include "common.cuh"
#include "ptx.cuh"
#include "rans_common.cuh"

namespace dc {

constexpr int kSmThreads = 256;
constexpr int kSmWarps = kSmThreads / 32;
constexpr int kSmSegs = 64;  // segments per warp task (2 per lane)
constexpr int kSmStride = 32;
constexpr int kSmOutBytes = 2 * 32 * kSmStride;  // per warp: 64 lane-segments x 32 B
struct __align__(16) SmallWarpSmem {
    uint8_t symtab[kProbScale];
    uint2 info[256];
    uint8_t out[kSmOutBytes];
};

__device__ __forceinline__ uint32_t swz_s(int ls, int h) {
    return (uint32_t)(ls * kSmStride + ((h ^ ((ls >> 2) & 1)) << 4));
}

// global-memory word window (see rans_common.cuh Win): w0 holds the next
// byte at bit offset o, w1 the next word, ga = global address of w1
struct GWin {
    uint32_t w0, w1, o;
    uint64_t ga;
};

__device__ __forceinline__ uint32_t ldg_nc_u32(uint64_t a) {
    uint32_t v;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(a));
    return v;
}

__device__ __forceinline__ void gwin_init(GWin& w, uint64_t p) {
    const uint64_t a = p & ~(uint64_t)3;
    w.w0 = ldg_nc_u32(a);
    w.w1 = ldg_nc_u32(a + 4);
    w.ga = a + 4;
    w.o = (uint32_t)(p & 3) * 8u;
}
__device__ __forceinline__ uint64_t gwin_pos(const GWin& w) { return w.ga - 4 + (w.o >> 3); }
__device__ __forceinline__ uint32_t gwin_bytes(const GWin& w) {
    uint32_t v;
    asm("shf.r.wrap.b32 %0, %1, %2, %3;" : "=r"(v) : "r"(w.w0), "r"(w.w1), "r"(w.o));
    return v;
}
__device__ __forceinline__ void gwin_advance(GWin& w, uint32_t s) {
    asm volatile(
        "{\n\t.reg .pred q;\n\t"
        "mad.lo.u32 %3, %4, 8, %3;\n\t"
        "setp.ge.u32 q, %3, 0x10840;\n\t"
        "@q mov.b32 %0, %1;\n\t"
        "@q add.u64 %2, %2, 4;\n\t"
        "@q ld.global.nc.u32 %1, [%2];\n\t"
        "and.b32 %3, %3, 31;\n\t}"
        : "+r"(w.w0), "+r"(w.w1), "+l"(w.ga), "+r"(w.o)
        : "r"(s));
}

// compact-table symbol step: returns the symbol, updates x, consumes window bytes
__device__ __forceinline__ uint32_t dec_sym_compact(uint32_t& x, uint32_t& s, uint32_t v, uint32_t symtab,
                                                    uint32_t info) {
    uint32_t sym;
    asm volatile(
        "{\n\t.reg .pred q;\n\t.reg .u32 slot, a, f, k, t;\n\t"
        "and.b32 slot, %0, 4095;\n\t"
        "add.u32 a, slot, %4;\n\t"
        "ld.shared.u8 %2, [a];\n\t"
        "mad.lo.u32 a, %2, 8, %5;\n\t"
        "ld.shared.v2.u32 {f, k}, [a];\n\t"
        "shr.u32 t, %0, 12;\n\t"
        "sub.u32 t, t, 4096;\n\t"
        "add.u32 k, k, slot;\n\t"
        "mad.lo.u32 %0, f, t, k;\n\t"
        "setp.lt.u32 q, %0, 0x100000;\n\t"
        "@q prmt.b32 %0, %0, %3, %1;\n\t"
        "@q add.u32 %1, %1, 1;\n\t"
        "setp.lt.u32 q, %0, 0x100000;\n\t"
        "@q prmt.b32 %0, %0, %3, %1;\n\t"
        "@q add.u32 %1, %1, 1;\n\t}"
        : "+r"(x), "+r"(s), "=r"(sym)
        : "r"(v), "r"(symtab), "r"(info));
    return sym;
}

// Warp-cooperative compact table from the blob's u12 wire table (validated
// beforehand by k_validate).  `cumend` scratch: 256 u32 (the out staging).
__device__ void build_compact_table(const uint8_t* __restrict__ tb, SmallWarpSmem& W, uint32_t* cumend, int lane) {
    uint32_t f[8], sum = 0, nz = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        unpack_pair(tb, lane * 4 + k, f[2 * k], f[2 * k + 1]);
        sum += f[2 * k] + f[2 * k + 1];
        nz += (f[2 * k] != 0) + (f[2 * k + 1] != 0);
    }
    uint32_t tot = sum, tnz = nz;
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        tot += __shfl_xor_sync(0xffffffffu, tot, d);
        tnz += __shfl_xor_sync(0xffffffffu, tnz, d);
    }
    if (tot == kProbScale - 1 && tnz == 1) {  // single symbol: stored 4095 means 4096 (ans.py:292-295)
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = f[k] ? kProbScale : 0;
        sum = sum ? kProbScale : 0;
    }
    uint32_t inc = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t o = __shfl_up_sync(0xffffffffu, inc, d);
        if (lane >= d) inc += o;
    }
    uint32_t cum = inc - sum;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        W.info[lane * 8 + k] = make_uint2(f[k], kProbScale * f[k] - cum);
        cum += f[k];
        cumend[lane * 8 + k] = cum;
    }
    __syncwarp();
    // lane fills slots [128 lane, 128 lane + 128), word by word, starting at
    // its own word `lane` and wrapping: at every step the 32 lanes store to 32
    // different banks (in order, all lanes would hit one bank: 32-way conflict)
    const uint32_t s0 = (uint32_t)lane * 128;
    auto first_sym = [&](uint32_t slot) {  // first symbol whose range ends past the slot
        int lo = 0, hi = 255;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (cumend[mid] > slot) hi = mid; else lo = mid + 1;
        }
        return lo;
    };
    const int sy_range = first_sym(s0);
    int sy = first_sym(s0 + 4u * (uint32_t)lane);
    uint32_t* dst = reinterpret_cast<uint32_t*>(W.symtab + s0);
    for (int i = 0; i < 32; ++i) {
        const int wv = (lane + i) & 31;
        if (wv == 0) sy = sy_range;  // wrapped to the start of the lane's range
        uint32_t word = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint32_t slot = s0 + wv * 4 + b;
            while (sy < 255 && cumend[sy] <= slot) ++sy;
            word |= (uint32_t)sy << (8 * b);
        }
        dst[wv] = word;
    }
    __syncwarp();
}

__global__ void __launch_bounds__(kSmThreads, 3) k_decode_small(
    const uint8_t* __restrict__ base, const uint64_t* __restrict__ blob_off, const uint64_t* __restrict__ blob_len,
    const uint64_t* __restrict__ out_off, const uint64_t* __restrict__ out_len, uint32_t seg_shift,
    const int64_t* __restrict__ seg_base, const uint32_t* __restrict__ seg_state,
    const uint32_t* __restrict__ seg_off, const int4* __restrict__ tasks, int64_t n_tasks,
    uint8_t* __restrict__ out, int32_t* __restrict__ status) {
    extern __shared__ __align__(1024) uint8_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    SmallWarpSmem& W = reinterpret_cast<SmallWarpSmem*>(smem)[warp];
    const uint32_t symtab = smem_u32(W.symtab), info = smem_u32(W.info);
    uint8_t* ob = W.out;
    const uint32_t K = 1u << seg_shift;
    const int G = (int)(K >> 4);
    int cached = -1;

    for (int64_t ti = (int64_t)blockIdx.x * kSmWarps + warp; ti < n_tasks; ti += (int64_t)gridDim.x * kSmWarps) {
        const int4 task = tasks[ti];
        const int c = task.x, s0 = task.y, ns = task.z;
        {
            const int32_t st0 = status[c];  // prologue errors (k_validate) are never decoded
            if (st0 >= DC_CHUNK_TRUNC_TABLE && st0 <= DC_CHUNK_EMPTY_BAD) continue;
        }
        const uint8_t* blob = base + blob_off[c];
        if (c != cached) {
            build_compact_table(blob, W, reinterpret_cast<uint32_t*>(ob), lane);
            cached = c;
        }
        const uint64_t gstream = reinterpret_cast<uint64_t>(blob) + kHeaderBytes;
        const uint32_t plen = (uint32_t)(blob_len[c] - kHeaderBytes);
        const uint64_t olen = out_len[c];
        const uint32_t nseg_chunk = (uint32_t)((olen + K - 1) >> seg_shift);
        const int64_t sb = seg_base[c];
        uint8_t* obase = out + out_off[c];
        const bool out_aligned = ((reinterpret_cast<uintptr_t>(obase) | (uintptr_t)K) & 15) == 0;

        uint32_t x[2], n[2];
        GWin Wn[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int r = lane + 32 * u;
            const uint32_t rel = (uint32_t)(s0 + r);
            uint64_t p = gstream;
            if (r < ns) {
                x[u] = seg_state[sb + rel];
                const uint32_t so = seg_off[sb + rel];
                const uint64_t rem = olen - ((uint64_t)rel << seg_shift);
                n[u] = rem < K ? (uint32_t)rem : K;
                const uint32_t se = rel + 1 < nseg_chunk ? seg_off[sb + rel + 1] : plen;
                if (so <= se && se <= plen) {
                    p = gstream + so;
                    for (uint32_t b = 0; b < se - so + 8; b += 128)  // segment stream -> L1
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(p + b));
                } else {  // damaged index: never an address; the exact decoder re-runs the chunk
                    atomicExch(&status[c], DC_CHUNK_CHAIN);
                }
            } else {  // decodes harmless garbage from the stream start, never written
                x[u] = kStateLower;
                n[u] = 0;
            }
            gwin_init(Wn[u], p);
        }
        for (int g = 0; g < G; ++g) {
            const uint32_t g0 = (uint32_t)g << 4;
            uint32_t w[2][4];
            const bool full = (n[0] == 0 || g0 + 16 <= n[0]) && (n[1] == 0 || g0 + 16 <= n[1]);
            if (__all_sync(0xffffffffu, full)) {
#pragma unroll
                for (int v = 0; v < 16; v += 2) {
                    uint32_t wv[2], sel[2], e0[2];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        wv[u] = gwin_bytes(Wn[u]);
                        sel[u] = kSelBase;
                        e0[u] = dec_sym_compact(x[u], sel[u], wv[u], symtab, info);
                    }
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const uint32_t t = __byte_perm(e0[u], dec_sym_compact(x[u], sel[u], wv[u], symtab, info),
                                                       0x0040);
                        w[u][v >> 2] = (v & 2) ? __byte_perm(w[u][v >> 2], t, 0x5410) : t;
                    }
#pragma unroll
                    for (int u = 0; u < 2; ++u) gwin_advance(Wn[u], sel[u]);
                }
            } else {
#pragma unroll
                for (int u = 0; u < 2; ++u) w[u][0] = w[u][1] = w[u][2] = w[u][3] = 0;
#pragma unroll
                for (int v = 0; v < 16; ++v) {
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        if (g0 + v < n[u]) {
                            uint32_t sel = kSelBase;
                            const uint32_t e = dec_sym_compact(x[u], sel, gwin_bytes(Wn[u]), symtab, info);
                            gwin_advance(Wn[u], sel);
                            w[u][v >> 2] = put_byte(w[u][v >> 2], e, v & 3);
                        }
                    }
                }
            }
            const int slot = g & 1;
#pragma unroll
            for (int u = 0; u < 2; ++u)
                *reinterpret_cast<uint4*>(ob + swz_s(u * 32 + lane, slot)) =
                    make_uint4(w[u][0], w[u][1], w[u][2], w[u][3]);
            if (slot == 1) {
                __syncwarp();
                const uint32_t line0 = (uint32_t)(g >> 1) * 32;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int pc = k * 32 + lane;
                    const int u = pc >> 6, ln = (pc >> 1) & 31, part = pc & 1;
                    const int r = ln + 32 * u;
                    if (r >= ns) continue;
                    const uint64_t seg_start = (uint64_t)(s0 + r) << seg_shift;
                    const uint64_t rem = olen - seg_start;
                    const uint32_t slen = rem < K ? (uint32_t)rem : K;
                    const uint32_t boff = line0 + part * 16;
                    if (boff >= slen) continue;
                    const uint8_t* src = ob + swz_s(u * 32 + ln, part);
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
        // chain checks: every segment must end exactly where the next one starts
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int r = lane + 32 * u;
            if (r >= ns) continue;
            const uint32_t rel = (uint32_t)(s0 + r);
            uint32_t xe, pe;
            if (rel + 1 < nseg_chunk) {
                xe = seg_state[sb + rel + 1];
                pe = seg_off[sb + rel + 1];
            } else {
                xe = kStateLower;
                pe = plen;
            }
            if (x[u] != xe || gwin_pos(Wn[u]) - gstream != pe) atomicExch(&status[c], DC_CHUNK_CHAIN);
        }
        __syncwarp();  // the out staging doubles as table-build scratch
    }
}

}  // namespace dc

using namespace dc;

extern "C" int dc_decode_small_segments(void) { return kSmSegs; }
extern "C" int dc_decode_small_max_chunk(void) { return 32 * 1024; }  // measured crossover: 16-32 KiB small wins, 64 KiB main wins

extern "C" int dc_ans_decode_small(const uint8_t* base, const uint64_t* blob_off, const uint64_t* blob_len,
                                   const uint64_t* out_off, const uint64_t* out_len, uint32_t seg_shift,
                                   const int64_t* seg_base, const uint32_t* seg_state, const uint32_t* seg_off,
                                   const int32_t* tasks, int64_t n_tasks, uint8_t* out, int32_t* status,
                                   void* stream) {
    if (n_tasks < 0 || seg_shift < 6 || seg_shift > 10) return DC_ERR_ARG;
    if (n_tasks == 0) return DC_OK;
    const int smem = kSmWarps * (int)sizeof(SmallWarpSmem);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_decode_small, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (n_tasks + kSmWarps - 1) / kSmWarps, cap = (int64_t)sms * 3;
    k_decode_small<<<(unsigned)(want < cap ? want : cap), kSmThreads, smem, (cudaStream_t)stream>>>(
        base, blob_off, blob_len, out_off, out_len, seg_shift, seg_base, seg_state, seg_off,
        reinterpret_cast<const int4*>(tasks), n_tasks, out, status);
    DC_CHECK_LAUNCH("k_decode_small");
    return DC_OK;
}
