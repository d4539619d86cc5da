// Compression-aware INT8 quantization on B200, bit-exact with the reference
// (scaling.py:78-117):
//   v = W[r,c] * s[c]                      (f64 multiply, scale_weights)
//   m = max |v|; w_scale = m / 127         (host, f64)
//   q = clip(sign(x) * floor(|x| + 0.5), -127, 127),  x = v / w_scale
//       (IEEE f64 division, half-away-from-zero rounding, _round_half_away)
// Inputs may be f64 (the reference type) or f32 / bf16 / f16 device tensors,
// widened to f64 exactly in registers.  Everything is HBM-bound: each kernel
// streams its input once with 16-byte loads.  No FMA contraction: the
// multiply, divide and add use explicit _rn intrinsics.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "common.cuh"

namespace dc {

int sm_count();  // rans_decode.cu

enum : int { kF64 = 0, kF32 = 1, kBF16 = 2, kF16 = 3 };

template <int T>
struct In;
template <>
struct In<kF64> {
    using type = double;
    __device__ static double f64(double v) { return v; }
};
template <>
struct In<kF32> {
    using type = float;
    __device__ static double f64(float v) { return (double)v; }
};
template <>
struct In<kBF16> {
    using type = __nv_bfloat16;
    __device__ static double f64(__nv_bfloat16 v) { return (double)__bfloat162float(v); }
};
template <>
struct In<kF16> {
    using type = __half;
    __device__ static double f64(__half v) { return (double)__half2float(v); }
};

constexpr int kQThreads = 256;

// rows are processed whole by a CTA slab; threads stride the columns.
template <int T>
__global__ void __launch_bounds__(kQThreads) k_absmax(const typename In<T>::type* __restrict__ w,
                                                       const double* __restrict__ s, int64_t rows, int64_t cols,
                                                       int64_t rows_per_cta, unsigned long long* __restrict__ out,
                                                       int* __restrict__ nonfinite) {
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
    const int64_t r1 = min(rows, r0 + rows_per_cta);
    double m = 0.0;
    bool bad = false;
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
        const double sc = s ? s[c] : 1.0;
        for (int64_t r = r0; r < r1; ++r) {
            const double raw = In<T>::f64(w[r * cols + c]);
            bad |= !isfinite(raw);
            const double v = fabs(__dmul_rn(raw, sc));
            m = v > m ? v : m;
        }
    }
    __shared__ double red[kQThreads / 32];
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, m, d);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    const int anybad = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int i = 0; i < kQThreads / 32; ++i) b = red[i] > b ? red[i] : b;
        // non-negative doubles order like their bit patterns
        atomicMax(out, (unsigned long long)__double_as_longlong(b));
        if (anybad) atomicExch(nonfinite, 1);
    }
}

__device__ __forceinline__ int8_t q_of(double v, double w_scale) {
    const double x = __ddiv_rn(v, w_scale);
    double a = floor(__dadd_rn(fabs(x), 0.5));
    a = a > 127.0 ? 127.0 : a;
    const double sg = x < 0.0 ? -a : (x > 0.0 ? a : 0.0);
    return (int8_t)(int)sg;
}

// Same result as q_of without the IEEE division on the common path: x' = v * (1/w_scale)
// is within 2 ulp of the correctly rounded quotient x (|x| <= 127.5 + ulp), so
// floor(|x| + 0.5) and the clip can only differ from the exact ones when |x'| is
// within 1e-9 of a half-integer; those (rare) elements take the exact division.
__device__ __forceinline__ int8_t q_of_fast(double v, double w_scale, double inv) {
    const double xa = __dmul_rn(v, inv);
    const double a = fabs(xa);
    const double h = a - floor(a);  // fractional part
    if (fabs(h - 0.5) < 1e-9) return q_of(v, w_scale);
    double r = floor(a + 0.5);
    r = r > 127.0 ? 127.0 : r;
    const double sg = xa < 0.0 ? -r : (xa > 0.0 ? r : 0.0);
    return (int8_t)(int)sg;
}

// q from the f32 product xf = w * c with c = s[col] / w_scale rounded to
// f32 (FP32 pipe only): |xf - x| < 2e-5 for the exact f64 quotient
// x = (w * s) / w_scale (|x| <= 127.5), so round-half-away(xf) equals the
// reference's floor(|x| + 0.5) unless |xf| is within 1e-4 of a half-integer,
// where the exact f64 path decides (rare).  The nearest integer comes from the
// mantissa of |xf| + 2^23 (no conversion instruction).
__device__ __forceinline__ int8_t q_of_f32(float wf, float cf, double w64, double sc, double w_scale) {
    const float xf = wf * cf;
    const float a = fabsf(xf);
    const float t = __fadd_rn(a, 8388608.0f);  // 2^23
    const float d = __fsub_rn(a, __fsub_rn(t, 8388608.0f));
    if (fabsf(fabsf(d) - 0.5f) < 1e-4f) return q_of(__dmul_rn(w64, sc), w_scale);
    int r = (int)(__float_as_uint(t) & 0x7FFFFFu);
    r = r > 127 ? 127 : r;
    return (int8_t)(xf < 0.0f ? -r : r);
}

// q[r, c] plus, optionally, the per-(column, |q|) histogram used by pruning
// (counts[c * 129 + |q|], u32, must be zeroed).
template <int T>
__global__ void __launch_bounds__(kQThreads) k_quantize(const typename In<T>::type* __restrict__ w,
                                                         const double* __restrict__ s, int64_t rows, int64_t cols,
                                                         int64_t rows_per_cta, double w_scale,
                                                         int8_t* __restrict__ q) {
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
    const int64_t r1 = min(rows, r0 + rows_per_cta);
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
        const double sc = s ? s[c] : 1.0;
        for (int64_t r = r0; r < r1; ++r) {
            const double v = __dmul_rn(In<T>::f64(w[r * cols + c]), sc);
            q[r * cols + c] = q_of(v, w_scale);
        }
    }
}

// ---- vectorized grid-stride variants (cols % 8 == 0, 16-B aligned input) --
// A thread owns 8 consecutive elements of one row: 16-byte loads of W (4 for
// f64, 2 for f32, 1 for bf16/f16) and of s, one 8-byte store of q.  Enough
// CTAs to keep every SM's load queue full; HBM-bound.
template <int T>
__device__ __forceinline__ void load8(const typename In<T>::type* __restrict__ w, int64_t e, double (&v)[8]) {
    if constexpr (T == kF64) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double2 d = __ldg(reinterpret_cast<const double2*>(w + e) + k);
            v[2 * k] = d.x;
            v[2 * k + 1] = d.y;
        }
    } else if constexpr (T == kF32) {
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(w + e) + k);
            v[4 * k] = f.x;
            v[4 * k + 1] = f.y;
            v[4 * k + 2] = f.z;
            v[4 * k + 3] = f.w;
        }
    } else {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(w + e));
        const uint32_t uw[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            typename In<T>::type lo, hi;
            const uint16_t a = (uint16_t)(uw[k] & 0xFFFF), b = (uint16_t)(uw[k] >> 16);
            memcpy(&lo, &a, 2);
            memcpy(&hi, &b, 2);
            v[2 * k] = In<T>::f64(lo);
            v[2 * k + 1] = In<T>::f64(hi);
        }
    }
}

// Raw 16-byte vectors of 8 consecutive elements (4 for f64, 2 for f32, 1 for
// bf16/f16): kept un-widened so several rows can be in flight per thread
// without the register cost of 8 doubles per row.
template <int T>
struct Raw8 {
    static constexpr int kVec = T == kF64 ? 4 : (T == kF32 ? 2 : 1);
    uint4 u[kVec];
};
template <int T>
__device__ __forceinline__ void load_raw8(const typename In<T>::type* __restrict__ w, int64_t e, Raw8<T>& r) {
#pragma unroll
    for (int k = 0; k < Raw8<T>::kVec; ++k) r.u[k] = __ldg(reinterpret_cast<const uint4*>(w + e) + k);
}
template <int T>
__device__ __forceinline__ double raw_at(const Raw8<T>& r, int k) {
    const uint32_t* x = reinterpret_cast<const uint32_t*>(r.u);
    if constexpr (T == kF64) {
        return __hiloint2double((int)x[2 * k + 1], (int)x[2 * k]);
    } else if constexpr (T == kF32) {
        return (double)__uint_as_float(x[k]);
    } else {
        const uint16_t h = (uint16_t)(x[k >> 1] >> (16 * (k & 1)));
        typename In<T>::type v;
        memcpy(&v, &h, 2);
        return In<T>::f64(v);
    }
}
template <int T>
__device__ __forceinline__ float raw_at_f32(const Raw8<T>& r, int k) {
    const uint32_t* x = reinterpret_cast<const uint32_t*>(r.u);
    if constexpr (T == kF64) return __double2float_rn(__hiloint2double((int)x[2 * k + 1], (int)x[2 * k]));
    else if constexpr (T == kF32) return __uint_as_float(x[k]);
    else if constexpr (T == kBF16) return __uint_as_float((x[k >> 1] >> (16 * (k & 1))) << 16);
    else return __half2float(__ushort_as_half((uint16_t)(x[k >> 1] >> (16 * (k & 1)))));
}

__device__ __forceinline__ void load_s8(const double* __restrict__ s, int64_t c, double (&sc)[8]) {
    if (s) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const double2 d = __ldg(reinterpret_cast<const double2*>(s + c) + k);
            sc[2 * k] = d.x;
            sc[2 * k + 1] = d.y;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) sc[k] = 1.0;
    }
}

// Thread layout: t = rp * gpr + cg owns the 8 columns [8*cg, 8*cg+8) of rows
// rp, rp + rows_par, ...; its 8 scales are loaded once.
template <int T>
__global__ void __launch_bounds__(kQThreads) k_absmax_v(const typename In<T>::type* __restrict__ w,
                                                         const double* __restrict__ s, int64_t rows, int64_t cols,
                                                         int64_t rows_par, unsigned long long* __restrict__ out,
                                                         int* __restrict__ nonfinite) {
    double m = 0.0;
    bool bad = false;
    const int64_t gpr = cols / 8, t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t cg = t % gpr, rp = t / gpr;
    double sc[8];
    load_s8(s, cg * 8, sc);
#ifndef DC_ABSMAX_ROWS_H
#define DC_ABSMAX_ROWS_H 4
#endif
    constexpr int kQR = T == kF64 ? 2 : (sizeof(typename In<T>::type) == 2 ? DC_ABSMAX_ROWS_H : 4);  // rows in flight per thread
    for (int64_t r0 = rp; r0 < rows && rp < rows_par; r0 += kQR * rows_par) {
        Raw8<T> v[kQR];
#pragma unroll
        for (int j = 0; j < kQR; ++j) {
            const int64_t r = r0 + j * rows_par;
            if (r < rows) load_raw8<T>(w, r * cols + cg * 8, v[j]);
        }
#pragma unroll
        for (int j = 0; j < kQR; ++j) {
            if (r0 + j * rows_par >= rows) break;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const double x = raw_at<T>(v[j], k);
                bad |= !isfinite(x);
                const double a = fabs(__dmul_rn(x, sc[k]));
                m = a > m ? a : m;
            }
        }
    }
    __shared__ double red[kQThreads / 32];
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, m, d);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    const int anybad = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
        double b = 0.0;
        for (int i = 0; i < kQThreads / 32; ++i) b = red[i] > b ? red[i] : b;
        atomicMax(out, (unsigned long long)__double_as_longlong(b));
        if (anybad) atomicExch(nonfinite, 1);
    }
}

#ifndef DC_QUANT_MINB
#define DC_QUANT_MINB 4  // <= 64 registers: 4 CTAs per SM (fewer registers spill, measured slower)
#endif

// f32 product path for 8 elements: q bytes packed in (lo, hi), and whether any
// of them lies within 1e-4 of a half-integer (then the caller redoes the 8
// exactly).  Branch-free: one test per 8 elements instead of a convergence
// barrier per element.
__device__ __forceinline__ uint32_t q8_fast_byte(float wf, float cf, bool& near) {
    const float xf = wf * cf;
    const float a = fabsf(xf);
    const float t = __fadd_rn(a, 8388608.0f);  // 2^23: the nearest integer lands in the mantissa
    const float d = __fsub_rn(a, __fsub_rn(t, 8388608.0f));
    near |= fabsf(fabsf(d) - 0.5f) < 1e-4f;
    const int r = min((int)(__float_as_uint(t) & 0x7FFFFFu), 127);
    return (uint32_t)(uint8_t)(int8_t)(xf < 0.0f ? -r : r);
}

// q of 8 elements by the reference's exact f64 formula (re-reads w and s)
template <int T>
__device__ __noinline__ void exact8(const typename In<T>::type* __restrict__ w, const double* __restrict__ s, int64_t e,
                                    int64_t c, double w_scale, uint32_t& lo, uint32_t& hi) {
    Raw8<T> v;
    load_raw8<T>(w, e, v);
    double sc[8];
    load_s8(s, c, sc);
    lo = hi = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t b = (uint8_t)q_of(__dmul_rn(raw_at<T>(v, k), sc[k]), w_scale);
        if (k < 4)
            lo |= b << (8 * k);
        else
            hi |= b << (8 * (k - 4));
    }
}

template <int T>
__global__ void __launch_bounds__(kQThreads, DC_QUANT_MINB) k_quantize_v(const typename In<T>::type* __restrict__ w,
                                                           const double* __restrict__ s, int64_t rows, int64_t cols,
                                                           int64_t rows_par, double w_scale, int8_t* __restrict__ q) {
    const int64_t gpr = cols / 8, t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t cg = t % gpr, rp = t / gpr;
    {
        // only cf stays in registers (the f64 scales are re-read in the rare
        // exact path); kQR rows of raw loads are in flight per thread
        float cf[8];
        {
            double sc[8];
            load_s8(s, cg * 8, sc);
#pragma unroll
            for (int k = 0; k < 8; ++k) cf[k] = __double2float_rn(sc[k] / w_scale);
        }
#ifndef DC_QUANT_ROWS
#define DC_QUANT_ROWS 1
#endif
#ifndef DC_QUANT_PF
#define DC_QUANT_PF 1  // rows ahead whose warp span is bulk-prefetched into L2 (0: off)
#endif
#ifndef DC_QUANT_ROWS_H
#define DC_QUANT_ROWS_H 1  // rows in flight per thread for 2-byte inputs (bf16 / f16)
#endif
        constexpr int kQR = sizeof(typename In<T>::type) == 2 ? DC_QUANT_ROWS_H : DC_QUANT_ROWS;
        // the warp's 32 consecutive 8-column groups are one contiguous span of
        // a row (when they do not wrap): lane 0 bulk-prefetches the span
        // DC_QUANT_PF rows ahead into L2, so more bytes are in flight than the
        // registers of 4 resident CTAs can hold
        const int64_t cg0 = __shfl_sync(0xffffffffu, cg, 0);
        const bool span = DC_QUANT_PF > 0 && (threadIdx.x & 31) == 0 && cg0 + 32 <= gpr;
        constexpr uint32_t kSpan = 32 * 8 * sizeof(typename In<T>::type);
        for (int64_t r0 = rp; r0 < rows && rp < rows_par; r0 += kQR * rows_par) {
            if (span) {
                const int64_t rf = r0 + (int64_t)DC_QUANT_PF * kQR * rows_par;
                if (rf < rows)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(w + rf * cols + cg0 * 8), "r"(kSpan)
                                 : "memory");
            }
            Raw8<T> v[kQR];
#pragma unroll
            for (int j = 0; j < kQR; ++j) {
                const int64_t r = r0 + j * rows_par;
                if (r < rows) load_raw8<T>(w, r * cols + cg * 8, v[j]);
            }
#pragma unroll
            for (int j = 0; j < kQR; ++j) {
                const int64_t r = r0 + j * rows_par;
                if (r >= rows) break;
                uint32_t lo = 0, hi = 0;
                bool near = false;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t b = q8_fast_byte(raw_at_f32<T>(v[j], k), cf[k], near);
                    if (k < 4)
                        lo |= b << (8 * k);
                    else
                        hi |= b << (8 * (k - 4));
                }
                if (near)  // rare: the exact f64 rounding for these 8 (out of line)
                    exact8<T>(w, s, r * cols + cg * 8, cg * 8, w_scale, lo, hi);
                *reinterpret_cast<uint2*>(q + r * cols + cg * 8) = make_uint2(lo, hi);
            }
        }
    }
}

// ---- column-max absmax (f32 / bf16 / f16 inputs) ---------------------------
// max |W[r,c] * s[c]| over the tensor equals max over columns of
// RN(max_r |W[r,c]| * s[c]): IEEE rounding is monotone and s > 0.  So the
// pass over the tensor only keeps per-column maxima of the magnitude bits
// (integer max on |x|'s bit pattern, monotone for finite values, and inf /
// NaN patterns sort above every finite one), two 16-bit lanes per instruction
// for bf16 / f16 (max.u16x2); each CTA then forms the f64 products for the
// column maxima of its row block only and contributes one atomic max (the max
// of those over CTAs is the tensor's).  The tensor pass is a pure streaming read.
constexpr int kCmCols = 256;  // columns per CTA tile: 32 lanes x 8
constexpr int kCmRows = 4;    // rows in flight per warp iteration

template <int T>
__global__ void __launch_bounds__(kQThreads) k_absmax_cols(const typename In<T>::type* __restrict__ w,
                                                            const double* __restrict__ s, int64_t rows, int64_t cols,
                                                            int64_t rows_per_blk, unsigned long long* __restrict__ out,
                                                            int* __restrict__ nonfinite) {
    constexpr bool kHalf = sizeof(typename In<T>::type) == 2;
    constexpr int kWords = kHalf ? 4 : 8;  // 32-bit words per lane per row (8 columns)
    __shared__ uint32_t red[kQThreads / 32][kCmCols];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t c0 = (int64_t)blockIdx.x * kCmCols + lane * 8;
    const int64_t r_begin = (int64_t)blockIdx.y * rows_per_blk;
    const int64_t r_end = min(rows, r_begin + rows_per_blk);
    uint32_t m[kWords];
#pragma unroll
    for (int k = 0; k < kWords; ++k) m[k] = 0;
    if (c0 < cols) {
        const uint4* base = reinterpret_cast<const uint4*>(w + c0);
        const int64_t row_vec = cols * (int64_t)sizeof(typename In<T>::type) / 16;  // uint4 per row
        for (int64_t r0 = r_begin + warp; r0 < r_end; r0 += kCmRows * (kQThreads / 32)) {
            uint4 v[kCmRows][kWords / 4];
#pragma unroll
            for (int j = 0; j < kCmRows; ++j) {
                const int64_t r = r0 + j * (kQThreads / 32);
#pragma unroll
                for (int h = 0; h < kWords / 4; ++h)
                    v[j][h] = r < r_end ? __ldg(base + r * row_vec + h) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int j = 0; j < kCmRows; ++j) {
#pragma unroll
                for (int h = 0; h < kWords / 4; ++h) {
                    const uint32_t x[4] = {v[j][h].x, v[j][h].y, v[j][h].z, v[j][h].w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        if constexpr (kHalf) {
                            uint32_t a = x[k] & 0x7FFF7FFFu, d;
                            asm("max.u16x2 %0, %1, %2;" : "=r"(d) : "r"(m[4 * h + k]), "r"(a));
                            m[4 * h + k] = d;
                        } else {
                            m[4 * h + k] = max(m[4 * h + k], x[k] & 0x7FFFFFFFu);
                        }
                    }
                }
            }
        }
    }
    // column maxima of this warp -> shared, max over the CTA's warps, one atomic per column
#pragma unroll
    for (int k = 0; k < 8; ++k)
        red[warp][lane * 8 + k] = kHalf ? ((m[k >> 1] >> (16 * (k & 1))) & 0xFFFFu) : m[k];
    __syncthreads();
    // this CTA's column maxima (over its row block) -> RN(|x| * s[c]) -> CTA max
    // -> one atomic: the max over CTAs of these is the tensor's max|W*s|
    constexpr uint32_t kInf = T == kF32 ? 0x7F800000u : (T == kBF16 ? 0x7F80u : 0x7C00u);
    const int t = threadIdx.x;
    uint32_t b = 0;
#pragma unroll
    for (int q = 0; q < kQThreads / 32; ++q) b = max(b, red[q][t]);
    const int64_t c = (int64_t)blockIdx.x * kCmCols + t;
    double a = 0.0;
    const bool bad = c < cols && b >= kInf;
    if (c < cols && b && !bad) {
        double v;
        if constexpr (T == kF32) v = (double)__uint_as_float(b);
        else if constexpr (T == kBF16) v = (double)__uint_as_float(b << 16);
        else v = (double)__half2float(__ushort_as_half((uint16_t)b));
        a = s ? __dmul_rn(v, __ldg(s + c)) : v;
    }
    __shared__ double dred[kQThreads / 32];
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, a, d);
        a = o > a ? o : a;
    }
    if ((t & 31) == 0) dred[t >> 5] = a;
    const int anybad = __syncthreads_or(bad);
    if (t == 0) {
        double m = 0.0;
        for (int i = 0; i < kQThreads / 32; ++i) m = dred[i] > m ? dred[i] : m;
        if (m > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
        if (anybad) atomicExch(nonfinite, 1);
    }
}

static bool vec_ok(const void* w, const double* s, int64_t cols, const void* q) {
    return cols % 8 == 0 && (reinterpret_cast<uintptr_t>(w) & 15) == 0 && (reinterpret_cast<uintptr_t>(s) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(q) & 7) == 0;
}

// rows processed in parallel so that rows_par * (cols/8) threads ~ 8 CTAs per SM
static void vec_shape(int64_t rows, int64_t cols, int64_t& rows_par, unsigned& grid) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t cap = (int64_t)sms * 8 * kQThreads, gpr = cols / 8;
    rows_par = cap / gpr;
    if (rows_par < 1) rows_par = 1;
    if (rows_par > rows) rows_par = rows;
    grid = (unsigned)((rows_par * gpr + kQThreads - 1) / kQThreads);
}

// v = q * w_scale / s[c]   (scaling.py:114-117, dequantize)
__global__ void k_dequantize(const int8_t* __restrict__ q, double w_scale, const double* __restrict__ s,
                             int64_t rows, int64_t cols, double* __restrict__ out) {
    const int64_t n = rows * cols;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i % cols;
        out[i] = __ddiv_rn(__dmul_rn((double)q[i], w_scale), s[c]);
    }
}

// W' = W * s[c]  (scaling.py:78-81, scale_weights)
__global__ void k_scale(const double* __restrict__ w, const double* __restrict__ s, int64_t rows, int64_t cols,
                        double* __restrict__ out) {
    const int64_t n = rows * cols;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __dmul_rn(w[i], s[i % cols]);
}

static int64_t rows_per(int64_t rows, int64_t cols) {
    // ~64K elements per CTA, at least one row
    int64_t r = (65536 + cols - 1) / cols;
    return r < 1 ? 1 : r;
}

}  // namespace dc

using namespace dc;

namespace dc {
// Calibration statistics (exporter export.py:77-123): per input channel, the
// running max of |x| over every token that enters a linear layer.  x is
// [rows = tokens][cols = channels] in any of the input dtypes, widened to f64
// exactly.  Thread j of a CTA owns column c0 + j over a slab of rows (so
// loads are coalesced across the warp); one atomicMax per column per CTA on
// the f64 bit pattern (non-negative doubles order like their bits; a NaN
// propagates as the largest pattern, like torch's amax).
template <int T>
__global__ void __launch_bounds__(kQThreads) k_channel_absmax(const typename In<T>::type* __restrict__ x,
                                                               int64_t rows, int64_t cols, int64_t rows_per_cta,
                                                               unsigned long long* __restrict__ acc) {
    const int64_t c = (int64_t)blockIdx.y * kQThreads + threadIdx.x;
    if (c >= cols) return;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
    const int64_t r1 = min(rows, r0 + rows_per_cta);
    unsigned long long m = 0;
    for (int64_t r = r0; r < r1; ++r) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(fabs(In<T>::f64(x[r * cols + c])));
        m = b > m ? b : m;
    }
    if (r1 > r0) atomicMax(&acc[c], m);
}
}  // namespace dc

namespace dc {
// W8A8 activation prologue (scaling.py:143-149 applied to a decode step's
// activations): X' = X / s (per input channel, IEEE f64 division), one
// per-tensor symmetric quantization of X' exactly as the weights'
// (w_scale = max|X'| / 127, q = clip(sign * floor(|X'| / sx + 0.5))).  One
// CTA per activation tensor (decode-sized: ntok x K <= a few MB): a block
// max-reduction, then the quantize pass from the same (L1/L2-hot) data.
struct ActQ {
    const void* x;      // [ntok][k] in dtype
    const double* s;    // [k] channel scales (null = identity)
    int8_t* q;          // [ntok][k] out
    double* sx;         // out: per-tensor activation scale (0 when X' == 0)
    double* xp;         // scratch [ntok][k] f64: X' = X / s
    uint64_t* mbits;    // scratch: max|X'| as f64 bits (zeroed by the caller)
    int64_t k;
};

// pass 1 (grid x = tensors, y = slices): X' = X / s into the scratch, running max
template <int T>
__global__ void __launch_bounds__(256) k_act_scale(const ActQ* __restrict__ t, int64_t ntok,
                                                   int32_t* __restrict__ status) {
    const ActQ a = t[blockIdx.x];
    const auto* x = static_cast<const typename In<T>::type*>(a.x);
    const int64_t n = ntok * a.k;
    double m = 0.0;
    bool bad = false;
    for (int64_t i = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.y * blockDim.x) {
        const double v = In<T>::f64(x[i]);
        bad |= !isfinite(v);
        const double d = a.s ? __ddiv_rn(v, a.s[i % a.k]) : v;
        a.xp[i] = d;
        const double ad = fabs(d);
        m = ad > m ? ad : m;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        const double o = __shfl_xor_sync(0xffffffffu, m, d);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0 && m > 0.0) atomicMax((unsigned long long*)a.mbits, (unsigned long long)__double_as_longlong(m));
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicExch(&status[blockIdx.x], 1);  // non-finite activations
}

// pass 2: sx = max / 127 (scaling.py:102), q = round-half-away(X' / sx) clipped
__global__ void __launch_bounds__(256) k_act_round(const ActQ* __restrict__ t, int64_t ntok,
                                                   int32_t* __restrict__ status) {
    const ActQ a = t[blockIdx.x];
    const double sx = __longlong_as_double((long long)*a.mbits) / 127.0;
    const int64_t n = ntok * a.k;
    if (blockIdx.y == 0 && threadIdx.x == 0) {
        *a.sx = sx;
        if (sx == 0.0 && status[blockIdx.x] == 0) status[blockIdx.x] = 2;  // zero dynamic range (q = 0)
    }
    const double inv = sx == 0.0 ? 0.0 : 1.0 / sx;
    for (int64_t i = (int64_t)blockIdx.y * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.y * blockDim.x)
        a.q[i] = sx == 0.0 ? (int8_t)0 : q_of_fast(a.xp[i], sx, inv);
}
}  // namespace dc

extern "C" int dc_act_quant_bytes(void) { return (int)sizeof(ActQ); }

extern "C" int dc_act_quant(const void* tensors, int n_tensors, int dtype, int64_t ntok, int64_t max_k,
                            int32_t* status, void* stream) {
    if (n_tensors < 0 || ntok < 0 || max_k < 0 || dtype < 0 || dtype > 3) return DC_ERR_ARG;
    if (n_tensors == 0 || ntok == 0) return DC_OK;
    const auto* t = static_cast<const ActQ*>(tensors);
    cudaStream_t st = (cudaStream_t)stream;
    // slices per tensor: ~8 elements per thread per slice, grid <= 8 CTAs per SM in total
    int64_t slices = (ntok * max_k + 256 * 8 - 1) / (256 * 8);
    const int64_t cap = ((int64_t)sm_count() * 8 + n_tensors - 1) / n_tensors;
    slices = slices < 1 ? 1 : (slices > cap ? (cap < 1 ? 1 : cap) : slices);
    dim3 grid((unsigned)n_tensors, (unsigned)slices);
    switch (dtype) {
        case kF64: k_act_scale<kF64><<<grid, 256, 0, st>>>(t, ntok, status); break;
        case kF32: k_act_scale<kF32><<<grid, 256, 0, st>>>(t, ntok, status); break;
        case kBF16: k_act_scale<kBF16><<<grid, 256, 0, st>>>(t, ntok, status); break;
        default: k_act_scale<kF16><<<grid, 256, 0, st>>>(t, ntok, status); break;
    }
    DC_CHECK_LAUNCH("k_act_scale");
    k_act_round<<<grid, 256, 0, st>>>(t, ntok, status);
    DC_CHECK_LAUNCH("k_act_round");
    return DC_OK;
}

extern "C" int dc_channel_absmax(const void* x, int dtype, int64_t rows, int64_t cols, uint64_t* acc_bits,
                                 void* stream) {
    if (rows < 0 || cols < 0 || dtype < 0 || dtype > 3) return DC_ERR_ARG;
    if (rows == 0 || cols == 0) return DC_OK;
    const int64_t cblocks = (cols + kQThreads - 1) / kQThreads;
    int64_t rblocks = (int64_t)sm_count() * 8 / cblocks;
    rblocks = rblocks < 1 ? 1 : (rblocks > rows ? rows : rblocks);
    const int64_t per = (rows + rblocks - 1) / rblocks;
    dim3 grid((unsigned)((rows + per - 1) / per), (unsigned)cblocks);
    auto* a = reinterpret_cast<unsigned long long*>(acc_bits);
    cudaStream_t st = (cudaStream_t)stream;
    switch (dtype) {
        case kF64: k_channel_absmax<kF64><<<grid, kQThreads, 0, st>>>((const double*)x, rows, cols, per, a); break;
        case kF32: k_channel_absmax<kF32><<<grid, kQThreads, 0, st>>>((const float*)x, rows, cols, per, a); break;
        case kBF16:
            k_channel_absmax<kBF16><<<grid, kQThreads, 0, st>>>((const __nv_bfloat16*)x, rows, cols, per, a);
            break;
        default: k_channel_absmax<kF16><<<grid, kQThreads, 0, st>>>((const __half*)x, rows, cols, per, a); break;
    }
    DC_CHECK_LAUNCH("k_channel_absmax");
    return DC_OK;
}

extern "C" int dc_quant_absmax(const void* w, int dtype, const double* s, int64_t rows, int64_t cols,
                               unsigned long long* absmax_bits, int* nonfinite, void* stream) {
    if (rows < 0 || cols < 0 || dtype < 0 || dtype > 3) return DC_ERR_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(absmax_bits, 0, sizeof(unsigned long long), st);
    cudaMemsetAsync(nonfinite, 0, sizeof(int), st);
    if (rows == 0 || cols == 0) return DC_OK;
    if (dtype != kF64 && vec_ok(w, s, cols, nullptr)) {  // f32 / bf16 / f16: column-max streaming pass
        const int64_t tiles = (cols + kCmCols - 1) / kCmCols;
        int64_t blocks_y = ((int64_t)sm_count() * 8 + tiles - 1) / tiles;  // ~8 CTAs per SM
        if (blocks_y > rows) blocks_y = rows;
        const int64_t rows_per_blk = (rows + blocks_y - 1) / blocks_y;
        blocks_y = (rows + rows_per_blk - 1) / rows_per_blk;
        const dim3 grid((unsigned)tiles, (unsigned)blocks_y);
        switch (dtype) {
            case kF32: k_absmax_cols<kF32><<<grid, kQThreads, 0, st>>>((const float*)w, s, rows, cols, rows_per_blk, absmax_bits, nonfinite); break;
            case kBF16: k_absmax_cols<kBF16><<<grid, kQThreads, 0, st>>>((const __nv_bfloat16*)w, s, rows, cols, rows_per_blk, absmax_bits, nonfinite); break;
            default: k_absmax_cols<kF16><<<grid, kQThreads, 0, st>>>((const __half*)w, s, rows, cols, rows_per_blk, absmax_bits, nonfinite); break;
        }
        DC_CHECK_LAUNCH("k_absmax_cols");
        return DC_OK;
    }
    if (vec_ok(w, s, cols, nullptr)) {
        int64_t rp;
        unsigned g;
        vec_shape(rows, cols, rp, g);
        switch (dtype) {
            case kF64: k_absmax_v<kF64><<<g, kQThreads, 0, st>>>((const double*)w, s, rows, cols, rp, absmax_bits, nonfinite); break;
            case kF32: k_absmax_v<kF32><<<g, kQThreads, 0, st>>>((const float*)w, s, rows, cols, rp, absmax_bits, nonfinite); break;
            case kBF16: k_absmax_v<kBF16><<<g, kQThreads, 0, st>>>((const __nv_bfloat16*)w, s, rows, cols, rp, absmax_bits, nonfinite); break;
            default: k_absmax_v<kF16><<<g, kQThreads, 0, st>>>((const __half*)w, s, rows, cols, rp, absmax_bits, nonfinite); break;
        }
        DC_CHECK_LAUNCH("k_absmax_v");
        return DC_OK;
    }
    const int64_t rp = rows_per(rows, cols);
    const unsigned grid = (unsigned)((rows + rp - 1) / rp);
    switch (dtype) {
        case kF64: k_absmax<kF64><<<grid, kQThreads, 0, st>>>((const double*)w, s, rows, cols, rp, absmax_bits, nonfinite); break;
        case kF32: k_absmax<kF32><<<grid, kQThreads, 0, st>>>((const float*)w, s, rows, cols, rp, absmax_bits, nonfinite); break;
        case kBF16: k_absmax<kBF16><<<grid, kQThreads, 0, st>>>((const __nv_bfloat16*)w, s, rows, cols, rp, absmax_bits, nonfinite); break;
        default: k_absmax<kF16><<<grid, kQThreads, 0, st>>>((const __half*)w, s, rows, cols, rp, absmax_bits, nonfinite); break;
    }
    DC_CHECK_LAUNCH("k_absmax");
    return DC_OK;
}

extern "C" int dc_quantize(const void* w, int dtype, const double* s, int64_t rows, int64_t cols, double w_scale,
                           int8_t* q, void* stream) {
    if (rows < 0 || cols < 0 || dtype < 0 || dtype > 3 || !(w_scale > 0.0)) return DC_ERR_ARG;
    if (rows == 0 || cols == 0) return DC_OK;
    cudaStream_t st = (cudaStream_t)stream;
    if (vec_ok(w, s, cols, q)) {
        int64_t rp;
        unsigned g;
        vec_shape(rows, cols, rp, g);
        switch (dtype) {
            case kF64: k_quantize_v<kF64><<<g, kQThreads, 0, st>>>((const double*)w, s, rows, cols, rp, w_scale, q); break;
            case kF32: k_quantize_v<kF32><<<g, kQThreads, 0, st>>>((const float*)w, s, rows, cols, rp, w_scale, q); break;
            case kBF16: k_quantize_v<kBF16><<<g, kQThreads, 0, st>>>((const __nv_bfloat16*)w, s, rows, cols, rp, w_scale, q); break;
            default: k_quantize_v<kF16><<<g, kQThreads, 0, st>>>((const __half*)w, s, rows, cols, rp, w_scale, q); break;
        }
        DC_CHECK_LAUNCH("k_quantize_v");
        return DC_OK;
    }
    const int64_t rp = rows_per(rows, cols);
    const unsigned grid = (unsigned)((rows + rp - 1) / rp);
    switch (dtype) {
        case kF64: k_quantize<kF64><<<grid, kQThreads, 0, st>>>((const double*)w, s, rows, cols, rp, w_scale, q); break;
        case kF32: k_quantize<kF32><<<grid, kQThreads, 0, st>>>((const float*)w, s, rows, cols, rp, w_scale, q); break;
        case kBF16: k_quantize<kBF16><<<grid, kQThreads, 0, st>>>((const __nv_bfloat16*)w, s, rows, cols, rp, w_scale, q); break;
        default: k_quantize<kF16><<<grid, kQThreads, 0, st>>>((const __half*)w, s, rows, cols, rp, w_scale, q); break;
    }
    DC_CHECK_LAUNCH("k_quantize");
    return DC_OK;
}

extern "C" int dc_dequantize(const int8_t* q, double w_scale, const double* s, int64_t rows, int64_t cols,
                             double* out, void* stream) {
    if (rows < 0 || cols < 0) return DC_ERR_ARG;
    if (rows == 0 || cols == 0) return DC_OK;
    k_dequantize<<<1184, 256, 0, (cudaStream_t)stream>>>(q, w_scale, s, rows, cols, out);
    DC_CHECK_LAUNCH("k_dequantize");
    return DC_OK;
}

extern "C" int dc_scale_weights(const double* w, const double* s, int64_t rows, int64_t cols, double* out,
                                void* stream) {
    if (rows < 0 || cols < 0) return DC_ERR_ARG;
    if (rows == 0 || cols == 0) return DC_OK;
    k_scale<<<1184, 256, 0, (cudaStream_t)stream>>>(w, s, rows, cols, out);
    DC_CHECK_LAUNCH("k_scale");
    return DC_OK;
}
