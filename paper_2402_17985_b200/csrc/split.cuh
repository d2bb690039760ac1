// split.cuh — exact device restatement of the reference's per-element FP64
// decisions (smoothing.cpp:75, flatten.cpp:8-15,60-74, quantize.cpp:44-45),
// shared by the K1 kernels (flatten.cu, flatten16.cu) and K2/K3.
//
// Exactness. Every decision the reference makes in FP64 is reproduced bit for
// bit, with cheaper but provably identical operation sequences:
//  * x / s (smoothing.cpp:75) and piece / scale (quantize.cpp:44): one FMA
//    correction step of q0 = x * RN(1/s) (Markstein: with the correctly rounded
//    reciprocal and q0 within 1 ulp, fma(fma(-q0, s, x), r, q0) is the
//    correctly rounded quotient);
//  * fmod(a, T) and llround((a - rem) / T) (flatten.cpp:12-13): n = floor(a/T)
//    and rem = a - n*T exactly, via n0 = floor(a * RN(1/T)) (off by at most
//    one) and the exact FMA residual fma(-n0, T, a) with a +-1 fix-up; the
//    reference's count equals n because RN(n*T)/T rounds back to n.
// tools/verify_fast_split.c checks both against the IEEE operations on 8e8
// random cases; tests/test_gpu_parity.py checks the kernels end to end.
#pragma once
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>

namespace fqg {
namespace split {

// ------------------------------------------------------------ arithmetic
__device__ __forceinline__ double div_exact(double x, double s, double r) {
    const double q0 = __dmul_rn(x, r);
    const double e = __fma_rn(-q0, s, x);
    return __fma_rn(e, r, q0);
}

struct Split {
    int cnt;      // number of full +-T pieces (after the saturation clamp)
    double rem;   // remainder piece magnitude (0 when saturated)
    bool neg;     // sign = v < 0 ? -1 : +1 (flatten.cpp:62)
    bool sat;
};

// split_against_threshold + split_into_slots' capacity rule (flatten.cpp:8-15,
// :60-74) for capacity `cap` = E + 1 slots.
__device__ __forceinline__ Split split_elem(double v, double t, double rt, int cap) {
    Split r;
    r.neg = v < 0.0;
    const double a = fabs(v);
    const double t0 = __dmul_rn(a, rt);
    if (t0 >= static_cast<double>(cap + 2)) {  // count > cap for sure
        r.cnt = cap;
        r.rem = 0.0;
        r.sat = true;
        return r;
    }
    double n0 = floor(t0);
    double rem = __fma_rn(-n0, t, a);
    if (rem < 0.0) {
        n0 -= 1.0;
        rem = __fma_rn(-n0, t, a);
    } else if (rem >= t) {
        n0 += 1.0;
        rem = __fma_rn(-n0, t, a);
    }
    const int n = static_cast<int>(n0);
    r.sat = n > cap || (n == cap && rem > 0.0);
    r.cnt = r.sat ? cap : n;
    r.rem = r.sat ? 0.0 : rem;
    return r;
}

// quantize.cpp:44-45: clamp(round(v / s), -qmax, qmax), half away from zero.
__device__ __forceinline__ int quant(double piece, double scale, double rscale, double qmax) {
    double r = round(div_exact(piece, scale, rscale));
    r = r < -qmax ? -qmax : (qmax < r ? qmax : r);
    return static_cast<int>(r);
}

// Per-launch constants of the activation split.
struct SplitConsts {
    double t, rt;        // T_x and RN(1/T_x)
    double as, ras;      // s_x and RN(1/s_x)
    double qmax;
    float rt32, q32;     // RN32(1/T_x), RN32(T_x / s_x)
    float qmax32;
    int qT;              // q of a full piece, round(T_x / s_x) clamped
};

__device__ __forceinline__ SplitConsts make_consts(double t, double rt, double as, double qmax) {
    SplitConsts sc;
    sc.t = t;
    sc.rt = rt;
    sc.as = as;
    sc.ras = 1.0 / as;
    sc.qmax = qmax;
    sc.rt32 = static_cast<float>(rt);
    sc.q32 = static_cast<float>(t / as);
    sc.qmax32 = static_cast<float>(qmax);
    sc.qT = quant(t, as, sc.ras, qmax);
    return sc;
}

template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const T w = __shfl_xor_sync(0xffffffffu, v, o);
        v = v < w ? w : v;
    }
    return v;
}
__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double to_f64(double v) { return v; }
__device__ __forceinline__ double to_f64(float v) { return static_cast<double>(v); }
__device__ __forceinline__ double to_f64(__half v) { return static_cast<double>(__half2float(v)); }
__device__ __forceinline__ double to_f64(__nv_bfloat16 v) {
    return static_cast<double>(__bfloat162float(v));
}

// FP32 fast path of one element with a certified error margin
// (tools/verify_fp32_split.c): |v32 - v| <= 1.3e-7 |v| (bf16/f16/f32 inputs
// are exact in f32; f64 inputs add 2^-24), hence |u32 - a/T| <= 3e-7 u. When
// the fractional part of u (piece-count boundary) or of z = frac * T/s_x
// (rounding boundary of the remainder piece) lies within the margin, ok is
// false and the caller takes the exact FP64 sequence instead.
struct Fast {
    int cnt, qrem;
    bool neg, sat, ok;
};
__device__ __forceinline__ Fast fast_elem(float xf, float rs32, int cap, const SplitConsts& c) {
    Fast o;
    const float v = __fmul_rn(xf, rs32);
    o.neg = v < 0.0f;
    const float u = __fmul_rn(fabsf(v), c.rt32);
    const bool big = u >= static_cast<float>(cap + 2);
    const float fl = floorf(u);
    const float fr = __fsub_rn(u, fl);
    const float eu = __fadd_rn(__fmul_rn(u, 5e-7f), 1e-30f);
    const bool okn = fr > eu && fr < 1.0f - eu;
    const int n = big ? cap : static_cast<int>(fl);
    const float z = __fmul_rn(fr, c.q32);
    const float zf = floorf(z);
    const float d = __fsub_rn(__fsub_rn(z, zf), 0.5f);
    const float ez = __fadd_rn(__fmul_rn(__fmul_rn(eu, c.q32), 1.5f),
                               __fadd_rn(__fmul_rn(z, 2.5e-7f), 1e-30f));
    const bool okz = fabsf(d) > ez;
    const int qi = static_cast<int>(fminf(d > 0.0f ? zf + 1.0f : zf, c.qmax32));
    o.sat = big || (okn && n >= cap);
    o.cnt = o.sat ? cap : n;
    o.qrem = o.sat ? 0 : (o.neg ? -qi : qi);
    o.ok = big || (okn && (n >= cap || okz));
    return o;
}

// The exact FP64 sequence for one element (smoothing.cpp:75,
// flatten.cpp:8-15,60-74, quantize.cpp:44): packed cnt | qrem << 16 |
// neg << 32 | sat << 33. Out of line: it runs for ~0.1% of the elements and
// keeping it out of the unrolled fast loop keeps that loop in registers.
static __device__ __noinline__ uint64_t slow_elem(double x, const double* sp_, const double* rp_,
                                                  int cap, double t, double rt, double as,
                                                  double ras, double qmax) {
    const double v = div_exact(x, __ldg(sp_), __ldg(rp_));
    const Split sp = split_elem(v, t, rt, cap);
    const int qrem = sp.cnt < cap ? quant(sp.neg ? -sp.rem : sp.rem, as, ras, qmax) : 0;
    return static_cast<uint64_t>(sp.cnt) | (static_cast<uint64_t>(qrem & 0xFFFF) << 16) |
           (static_cast<uint64_t>(sp.neg) << 32) | (static_cast<uint64_t>(sp.sat) << 33);
}

// One element through the FP32 certified path, falling back to the exact
// FP64 sequence; same packing as slow_elem.
__device__ __forceinline__ uint64_t split_quant_elem(float xf, double xd, const double* sp_,
                                                     const double* rp_, float rs32, int cap,
                                                     const SplitConsts& c) {
    const Fast f = fast_elem(xf, rs32, cap, c);
    if (f.ok)
        return static_cast<uint64_t>(f.cnt) | (static_cast<uint64_t>(f.qrem & 0xFFFF) << 16) |
               (static_cast<uint64_t>(f.neg) << 32) | (static_cast<uint64_t>(f.sat) << 33);
    return slow_elem(xd, sp_, rp_, cap, c.t, c.rt, c.as, c.ras, c.qmax);
}

}  // namespace split
}  // namespace fqg
