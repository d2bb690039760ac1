// flatten.cu — the HBM-bound kernels of the hot path.
//
// K1 k_flatten_quant : divide_columns -> flatten_tensor(saturating) ->
//                      repeat_columns -> quantize_per_tensor(static scale)
//                      (smoothing.cpp:68-79, flatten.cpp:60-102,158-174,
//                      quantize.cpp:23-48), fused into one pass over x through
//                      the composite gather map (k' -> source channel j, piece p).
// K2 k_act_absmax    : per-tensor absmax of the flattened activations for the
//                      opt-in dynamic scale (quantize.cpp:34-40): warp shuffle ->
//                      block -> one atomicMax per block on the FP64 bit pattern.
// K3 k_weight_absmax / k_weight_quant : the offline weight tail of
//                      quantize_layer (pipeline.cpp:100,114-120,139-150):
//                      scale_rows, repeat_channels, strict flatten_rows, absmax
//                      -> s_w, round-to-nearest, K-major int8 / packed int4.
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
// Pieces equal to +-T quantize to +-round(T/scale) (once per CTA), zero
// pieces to 0, so only the remainder piece needs a division.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "fqg_internal.h"
#include "kernels.h"
#include "split.cuh"

namespace fqg {
namespace {

using namespace split;

// 8 consecutive activations -> f64 (exact conversions), 16-byte loads (bf16 is
// converted in place by the caller).
template <typename T>
__device__ __forceinline__ void load8(const T* p, bool vec, double (&o)[8]);
template <>
__device__ __forceinline__ void load8<__half>(const __half* p, bool vec, double (&o)[8]) {
    if (vec) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
        const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(h[i]);
            o[2 * i] = f.x;
            o[2 * i + 1] = f.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = static_cast<double>(__half2float(p[i]));
    }
}
template <>
__device__ __forceinline__ void load8<float>(const float* p, bool vec, double (&o)[8]) {
    if (vec) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(p));
        const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
        o[0] = a.x, o[1] = a.y, o[2] = a.z, o[3] = a.w;
        o[4] = b.x, o[5] = b.y, o[6] = b.z, o[7] = b.w;
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = p[i];
    }
}
template <>
__device__ __forceinline__ void load8<double>(const double* p, bool vec, double (&o)[8]) {
    if (vec) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double2 d = __ldg(reinterpret_cast<const double2*>(p) + i);
            o[2 * i] = d.x;
            o[2 * i + 1] = d.y;
        }
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) o[i] = p[i];
    }
}

// Static or dynamic activation scale.
__device__ __forceinline__ double act_scale_of(const double* scale, const unsigned long long* amax,
                                               double qmax) {
    if (amax == nullptr) return scale[0];
    // quantize.cpp:34-40: s = max|M| / qmax (a degenerate 0 yields zero outputs)
    return __ddiv_rn(__longlong_as_double(static_cast<long long>(*amax)), qmax);
}

// 8 consecutive activations as f32 (exact for bf16/f16/f32) + the f64 value
// (for non-f64 inputs d = f exactly; the conversion is only needed on the
// rare exact path).
template <typename T>
__device__ __forceinline__ void load8f(const T* p, bool vec, int nj, float (&f)[8],
                                       double (&d)[8]) {
    if constexpr (std::is_same<T, __nv_bfloat16>::value) {
        if (nj == 8 && vec) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
            const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                f[2 * i] = __uint_as_float(w[i] << 16);
                f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
            }
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) f[e] = e < nj ? __bfloat162float(p[e]) : 0.0f;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) d[e] = static_cast<double>(f[e]);
    } else {
        if (nj == 8) {
            load8<T>(p, vec, d);
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) d[e] = e < nj ? to_f64(p[e]) : 0.0;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = static_cast<float>(d[e]);
    }
}

// Packs 32 int8 (k 0..31 of a group) into 16 bytes of the FQG_I4 layout:
// byte i = q[i] & 15 | q[16 + i] << 4.
__device__ __forceinline__ uint4 pack_i4(uint4 lo, uint4 hi) {
    auto p = [](uint32_t a, uint32_t b) {
        return (a & 0x0F0F0F0Fu) | ((b << 4) & 0xF0F0F0F0u);
    };
    return make_uint4(p(lo.x, hi.x), p(lo.y, hi.y), p(lo.z, hi.z), p(lo.w, hi.w));
}

// One CTA = `rows` consecutive token rows; a shared-memory copy of each row's
// plan_x-flattened form flat[r][0..C1) (slot j, extension slots
// K + off_j + p - 1, zero padding; flatten.cpp:76-102) is built, then written.
// Phase 0: zero the extension/padding region [K, C1).
// Phase 1: every source element (i, j) is split once (thread owns 8
//   consecutive channels; tables reused across the CTA's rows). Tier 1 (every
//   element, ~20 instructions) handles |v| < T: no full piece, so slot j holds
//   the remainder q and every extension slot stays 0. Tier 2 (flagged elements
//   only) runs the general FP32-certified split with the exact FP64 fallback;
//   an element with pieces writes its single extension slot itself (E = 1) or
//   queues (row, channel, count, remainder) for a warp-parallel expansion.
// Phase 1b: warps expand queued elements, one lane per extension slot.
// Phase 2: columns [0, C1) of the final operand ARE the flattened row
//   (repeat_columns keeps column r at r, flatten.cpp:166) — 16-byte copies;
//   columns [C1, K') are plan_w copies of flat columns wsrc[k' - C1], gathered.
template <typename XT, bool PACK4>
__global__ void __launch_bounds__(256, 4)
    k_flatten_quant(const XT* __restrict__ x, int64_t ldx, int m, int k, int rows, int vec_ok,
                    const double* __restrict__ s, const double* __restrict__ rs,
                    const float* __restrict__ rs32, const int32_t* __restrict__ cap,
                    const int32_t* __restrict__ off, int qcap,
                    const int32_t* __restrict__ wsrc, int c1, int kp,
                    double t, double rt, double* __restrict__ scale,
                    const unsigned long long* __restrict__ amax, double qmax,
                    uint8_t* __restrict__ q, int64_t ldq, unsigned long long* __restrict__ sat_out) {
    extern __shared__ uint4 flat4[];  // [rows][c1] bytes, then the expansion queue
    int8_t* flat = reinterpret_cast<int8_t*>(flat4);
    uint2* queue = reinterpret_cast<uint2*>(flat + rows * c1);  // {code, r << 20 | j}
    __shared__ unsigned long long red[8];
    __shared__ int qlen;
    const int row0 = blockIdx.x * rows;
    const int nrows = min(rows, m - row0);
    const double as = act_scale_of(scale, amax, qmax);
    if (amax != nullptr && blockIdx.x == 0 && threadIdx.x == 0) scale[0] = as;
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
    const bool vec = vec_ok != 0;

    // ---- phase 0 ----
    if (threadIdx.x == 0) qlen = 0;
    {
        const int k4 = (k + 3) & ~3;  // c1 is a multiple of 32: words from k4, bytes before
        for (int r = 0; r < nrows; ++r) {
            if (threadIdx.x < k4 - k) flat[r * c1 + k + threadIdx.x] = 0;
            uint32_t* z = reinterpret_cast<uint32_t*>(flat + r * c1 + k4);
            for (int i = threadIdx.x; i < (c1 - k4) >> 2; i += blockDim.x) z[i] = 0u;
        }
    }
    __syncthreads();

    // ---- phase 1 ----
    // Tier 1: z = |x| * RN32(RN32(1/s_j) * RN32(1/s_x)) equals |v|/s_x = u*Q to
    // within 2.4e-7 relative. z < Q(1 - 4e-7) proves u < 1: no full pieces,
    // no saturation, slot j holds round(|v|/s_x) — accepted when z is also
    // clear of a rounding half-integer (tools/verify_fp32_split.c, tier 1).
    const float ras32 = static_cast<float>(sc.ras);
    const float qlo = sc.q32 * (1.0f - 4e-7f);
    const int qmaxi = static_cast<int>(sc.qmax);
    unsigned long long sat = 0;
    for (int j0 = threadIdx.x * 8; j0 < k; j0 += blockDim.x * 8) {
        const int nj = min(8, k - j0);
        float cz[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) cz[e] = __fmul_rn(__ldg(rs32 + min(j0 + e, k - 1)), ras32);
        for (int r = 0; r < nrows; ++r) {
            float xf[8];
            double xd[8];
            load8f<XT>(x + static_cast<int64_t>(row0 + r) * ldx + j0, vec, nj, xf, xd);
            int8_t* fr = flat + r * c1;
            uint32_t w0 = 0u, w1 = 0u;
            unsigned slow = 0;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float z = __fmul_rn(fabsf(xf[e]), cz[e]);
                const float tz = __fadd_rn(z, 0.5f);
                const float qf = floorf(tz);
                const float dd = fabsf(__fsub_rn(__fsub_rn(tz, qf), 0.5f));  // |frac - 1/2|
                const float lim = __fsub_rn(0.5f, __fadd_rn(__fmul_rn(z, 4e-7f), 1e-6f));
                const bool ok = z < qlo && dd < lim;
                // clamp (quantize.cpp:44-45): act_scale and T_x are independent recipe
                // fields, so z may exceed qmax when act_scale * qmax < T_x
                const int qi = min(static_cast<int>(qf), qmaxi);
                const uint32_t byte =
                    ok ? static_cast<uint32_t>((xf[e] < 0.0f ? -qi : qi) & 0xFF) : 0u;
                if (e < 4)
                    w0 |= byte << (8 * e);
                else
                    w1 |= byte << (8 * (e - 4));
                slow |= (!ok && e < nj) ? (1u << e) : 0u;
            }
            if (nj == 8) {
                *reinterpret_cast<uint2*>(fr + j0) = make_uint2(w0, w1);
            } else {
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    if (e < nj) fr[j0 + e] = static_cast<int8_t>((e < 4 ? w0 : w1) >> (8 * (e & 3)));
            }
            while (slow) {  // tier 2
                const int e = __ffs(slow) - 1;
                slow &= slow - 1;
                const int j = j0 + e;
                const int cap_e = __ldg(cap + j);
                const double xde = to_f64(x[static_cast<int64_t>(row0 + r) * ldx + j]);
                const Fast f = fast_elem(static_cast<float>(xde), __ldg(rs32 + j), cap_e, sc);
                uint64_t res;  // cnt | qrem << 16 | neg << 32 | sat << 33
                if (f.ok) {
                    res = static_cast<uint64_t>(f.cnt) |
                          (static_cast<uint64_t>(f.qrem & 0xFFFF) << 16) |
                          (static_cast<uint64_t>(f.neg) << 32) | (static_cast<uint64_t>(f.sat) << 33);
                } else {  // exact FP64 path
                    res = slow_elem(xde, s + j, rs + j, cap_e, sc.t, sc.rt, sc.as, sc.ras, sc.qmax);
                }
                const int ce = static_cast<int>(res & 0xFFFF);
                const int qe = static_cast<int>(static_cast<int16_t>(res >> 16));
                const bool ng = (res >> 32) & 1;
                const int full = ng ? -sc.qT : sc.qT;
                sat += (res >> 33) & 1;
                // slot j = piece 0: a full piece if cnt >= 1, else the remainder.
                fr[j] = static_cast<int8_t>(ce >= 1 ? full : qe);
                if (cap_e > 1 && ce >= 1) {  // extension slots carry pieces 1 .. E
                    const int ext0 = k + __ldg(off + j);
                    if (cap_e == 2) {
                        fr[ext0] = static_cast<int8_t>(1 < ce ? full : (1 == ce ? qe : 0));
                    } else {
                        const int slot = atomicAdd(&qlen, 1);
                        if (slot < qcap)
                            queue[slot] = make_uint2(static_cast<uint32_t>(ce) |
                                                         (static_cast<uint32_t>(qe & 0xFF) << 16) |
                                                         (static_cast<uint32_t>(ng) << 24),
                                                     (static_cast<uint32_t>(r) << 20) |
                                                         static_cast<uint32_t>(j));
                    }
                }
            }
        }
    }
    __syncthreads();
    // ---- phase 1b: warp-parallel expansion of queued elements ----
    {
        const int n_q = min(qlen, qcap);
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        for (int i = warp; i < n_q; i += blockDim.x >> 5) {
            const uint2 e = queue[i];
            const int j = static_cast<int>(e.y & 0xFFFFF), r = static_cast<int>(e.y >> 20);
            const int cnt = static_cast<int>(e.x & 0xFFFFu);
            const int qe = static_cast<int>(static_cast<int8_t>(e.x >> 16));
            const int full = (e.x >> 24) & 1 ? -sc.qT : sc.qT;
            const int ext = __ldg(cap + j) - 1;
            int8_t* dst = flat + r * c1 + k + __ldg(off + j) - 1;  // dst[p], p = 1 .. E
            for (int p = 1 + lane; p <= ext; p += 32)
                dst[p] = static_cast<int8_t>(p < cnt ? full : (p == cnt ? qe : 0));
        }
    }
    __syncthreads();

    // ---- phase 2 ----
    if constexpr (PACK4) {
        for (int c = threadIdx.x; c < c1 / 32; c += blockDim.x)
            for (int r = 0; r < nrows; ++r) {
                const uint4* f4 = reinterpret_cast<const uint4*>(flat + r * c1 + c * 32);
                *reinterpret_cast<uint4*>(q + static_cast<int64_t>(row0 + r) * ldq + c * 16) =
                    pack_i4(f4[0], f4[1]);
            }
    } else {
        for (int c = threadIdx.x; c < c1 / 16; c += blockDim.x)
            for (int r = 0; r < nrows; ++r)
                *reinterpret_cast<uint4*>(q + static_cast<int64_t>(row0 + r) * ldq + c * 16) =
                    *reinterpret_cast<const uint4*>(flat + r * c1 + c * 16);
    }
    constexpr int G = PACK4 ? 32 : 16;  // output columns per gathered chunk
    auto gather4 = [](const int8_t* fr, int4 s4) {
        const int sv[4] = {s4.x, s4.y, s4.z, s4.w};
        uint32_t acc = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b)
            acc |= (sv[b] < 0 ? 0u : static_cast<uint32_t>(static_cast<uint8_t>(fr[sv[b]])))
                   << (8 * b);
        return acc;
    };
    for (int c = threadIdx.x; c < (kp - c1) / G; c += blockDim.x) {
        const int4* src4 = reinterpret_cast<const int4*>(wsrc + c * G);
        for (int r = 0; r < nrows; ++r) {
            const int8_t* fr = flat + r * c1;
            uint32_t w[G / 4];
#pragma unroll
            for (int v = 0; v < G / 4; ++v) w[v] = gather4(fr, __ldg(src4 + v));
            uint8_t* qr = q + static_cast<int64_t>(row0 + r) * ldq;
            if constexpr (PACK4) {
                *reinterpret_cast<uint4*>(qr + (c1 + c * 32) / 2) =
                    pack_i4(make_uint4(w[0], w[1], w[2], w[3]), make_uint4(w[4], w[5], w[6], w[7]));
            } else {
                *reinterpret_cast<uint4*>(qr + c1 + c * 16) = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
    }

    // Saturation events: warp shuffle -> block -> one atomic per CTA.
    if (sat_out != nullptr) {
        sat = warp_sum(sat);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sat;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long tot = 0;
            for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += red[w];
            if (tot) atomicAdd(sat_out, tot);
        }
    }
}

// ------------------------------------------------------------------ K2
// max over the flattened tensor = max over source elements of the largest
// piece: T when at least one full piece exists, else the remainder.
template <typename XT>
__global__ void __launch_bounds__(256)
    k_act_absmax(const XT* __restrict__ x, int64_t ldx, int m, int k,
                 const double* __restrict__ s, const double* __restrict__ rs,
                 const int32_t* __restrict__ cap, double t, double rt,
                 unsigned long long* __restrict__ amax) {
    __shared__ double red[8];
    double mx = 0.0;
    const int64_t total = static_cast<int64_t>(m) * k;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(idx / k), j = static_cast<int>(idx % k);
        const double xv = to_f64(x[static_cast<int64_t>(i) * ldx + j]);
        const double v = div_exact(xv, s[j], rs[j]);
        const Split sp = split_elem(v, t, rt, cap[j]);
        const double piece = sp.cnt >= 1 ? t : sp.rem;
        mx = mx < piece ? piece : mx;
    }
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) mx = mx < red[w] ? red[w] : mx;
        // Non-negative doubles order like their bit patterns.
        atomicMax(amax, static_cast<unsigned long long>(__double_as_longlong(mx)));
    }
}

// ------------------------------------------------------------------ K3
// Pass 1: global max |W_flat| over ALL columns (the per-tensor s_w must be
// the unsharded one) + strict-capacity check (flatten.cpp:116-119).
__global__ void __launch_bounds__(256)
    k_weight_absmax(const double* __restrict__ w, int k, int64_t ncols,
                    const double* __restrict__ s, const int32_t* __restrict__ capw_src,
                    double t_w, double rt_w, unsigned long long* __restrict__ amax,
                    unsigned int* __restrict__ overflow) {
    __shared__ double red[8];
    double mx = 0.0;
    bool over = false;
    const int64_t total = static_cast<int64_t>(k) * ncols;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(idx / ncols);
        const double v = __dmul_rn(w[idx], s[j]);  // scale_rows, smoothing.cpp:88
        const Split sp = split_elem(v, t_w, rt_w, capw_src[j]);
        over |= sp.sat;
        const double piece = sp.cnt >= 1 ? t_w : sp.rem;
        mx = mx < piece ? piece : mx;
    }
    if (__any_sync(0xffffffffu, over) && (threadIdx.x & 31) == 0) atomicOr(overflow, 1u);
    mx = warp_max(mx);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w8 = 1; w8 < static_cast<int>(blockDim.x >> 5); ++w8)
            mx = mx < red[w8] ? red[w8] : mx;
        atomicMax(amax, static_cast<unsigned long long>(__double_as_longlong(mx)));
    }
}

// Pass 2: q_w[n][k'] (K-major) for the shard's columns. Tile: 32 output
// columns (threadIdx.x, coalesced 256-byte reads of W rows) x 128 k' (the
// composite weight map: k' -> source row j, piece p_w, capacity).
constexpr int WQ_TK = 128;
template <bool PACK4>
__global__ void __launch_bounds__(256)
    k_weight_quant(const double* __restrict__ w, int64_t ldw, int64_t n_begin, int n,
                   const double* __restrict__ s, const int32_t* __restrict__ wmap,
                   const int32_t* __restrict__ wcap, int kp, double t_w, double rt_w, double s_w,
                   double rs_w, double qmax, uint8_t* __restrict__ wq, int64_t ldq) {
    __shared__ int8_t tile[32][WQ_TK + 4];
    const int n0 = blockIdx.x * 32, k0 = blockIdx.y * WQ_TK;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int col = n0 + tx;
    for (int kk = ty; kk < WQ_TK; kk += 8) {
        const int kq = k0 + kk;
        int qv = 0;
        if (kq < kp && col < n) {
            const int32_t mp = wmap[kq];
            if (mp >= 0) {
                const int j = mp >> 12, p = mp & 0xFFF;
                const double v = __dmul_rn(w[static_cast<int64_t>(j) * ldw + n_begin + col], s[j]);
                const Split sp = split_elem(v, t_w, rt_w, wcap[kq]);
                double piece = 0.0;
                if (p < sp.cnt)
                    piece = sp.neg ? -t_w : t_w;
                else if (p == sp.cnt)
                    piece = sp.neg ? -sp.rem : sp.rem;
                qv = quant(piece, s_w, rs_w, qmax);
            }
        }
        tile[tx][kk] = static_cast<int8_t>(qv);
    }
    __syncthreads();
    // Write: each warp writes rows n0+ty, n0+ty+8, ...; lane covers 4 k' values
    // (int8) or 4 packed bytes (FQG_I4: per 32-k group, byte i = q[i] | q[16+i] << 4).
    for (int r = ty; r < 32; r += 8) {
        const int nn = n0 + r;
        if (nn >= n) continue;
        if constexpr (PACK4) {
            if (tx >= 16) continue;
            const int g = tx >> 2, i = (tx & 3) * 4;  // group of 32 k, first byte
            if (k0 + 32 * g >= kp) continue;
            const int8_t* lo = &tile[r][32 * g + i];
            const int8_t* hi = lo + 16;
            uint32_t b = 0;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                // biased nibbles q + 8 (FQG_I4_BIASED, the layer's weight storage)
                b |= static_cast<uint32_t>(((lo[e] + 8) & 0xF) | (((hi[e] + 8) & 0xF) << 4)) << (8 * e);
            *reinterpret_cast<uint32_t*>(wq + nn * ldq + k0 / 2 + 16 * g + i) = b;
        } else {
            const int kk = tx * 4;
            if (k0 + kk >= kp) continue;
            const int8_t* src = &tile[r][kk];
            const uint32_t b = static_cast<uint32_t>(static_cast<uint8_t>(src[0])) |
                               (static_cast<uint32_t>(static_cast<uint8_t>(src[1])) << 8) |
                               (static_cast<uint32_t>(static_cast<uint8_t>(src[2])) << 16) |
                               (static_cast<uint32_t>(static_cast<uint8_t>(src[3])) << 24);
            *reinterpret_cast<uint32_t*>(wq + nn * ldq + k0 + kk) = b;
        }
    }
}

// Sum of each operand row (int8, or signed nibbles of packed int4): the row
// sums the biased-int4 GEMM epilogue needs when K1 took the general path.
__global__ void __launch_bounds__(256)
    k_rowsum(const uint8_t* __restrict__ q, int64_t ldq, int m, int nbytes, bool pack4,
             int32_t* __restrict__ out) {
    const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row >= m) return;
    const uint4* r = reinterpret_cast<const uint4*>(q + row * ldq);
    int acc = 0;
    for (int i = lane; i < (nbytes >> 4); i += 32) {
        const uint4 v = r[i];
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if (pack4) {  // sum of (nibble ^ 8) = sum of (q + 8), 8 nibbles per word
                acc += static_cast<int>(__dp4a((w[e] & 0x0F0F0F0Fu) ^ 0x08080808u, 0x01010101u, 0u));
                acc += static_cast<int>(__dp4a(((w[e] >> 4) & 0x0F0F0F0Fu) ^ 0x08080808u, 0x01010101u, 0u));
                acc -= 64;
            } else {
                acc = __dp4a(static_cast<int>(w[e]), 0x01010101, acc);
            }
        }
    }
    acc = static_cast<int>(warp_sum(static_cast<unsigned long long>(static_cast<int64_t>(acc))));
    if (lane == 0) out[row] = acc;
}

template <typename XT>
void launch_flatten_t(const FlattenArgs& a, cudaStream_t st) {
    const double rt = 1.0 / a.t;
    if (a.amax != nullptr) {
        const int64_t total = a.m * a.k;
        const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, a.num_sms * 8));
        k_act_absmax<XT><<<grid, 256, 0, st>>>(static_cast<const XT*>(a.x), a.ldx,
                                                static_cast<int>(a.m), static_cast<int>(a.k), a.s,
                                                a.rs, a.cap, a.t, rt, a.amax);
        FQG_CUDA(cudaGetLastError());
    }
    // flattened row + room to queue every channel with >= 2 extension slots
    const int64_t row_bytes = a.c1 + 8 * a.n_ext2;
    // Rows per CTA: several rows amortize the table/map loads; keep >= ~4 CTAs per SM.
    int rows = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(8, (48 * 1024) / row_bytes)));
    while (rows > 1 && (a.m + rows - 1) / rows < 4 * a.num_sms) rows >>= 1;
    const int64_t smem = (rows * a.c1 + 15) / 16 * 16 + rows * 8 * a.n_ext2;
    require(smem <= 200 * 1024, "flatten: plan_x width too large for the shared-memory row");
    const int grid = static_cast<int>((a.m + rows - 1) / rows);
    const bool vec = (reinterpret_cast<uintptr_t>(a.x) % 16 == 0) &&
                     ((a.ldx * static_cast<int64_t>(sizeof(XT))) % 16 == 0);
    auto run = [&](auto kern) {
        FQG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        kern<<<grid, 256, smem, st>>>(static_cast<const XT*>(a.x), a.ldx, static_cast<int>(a.m),
                                      static_cast<int>(a.k), rows, vec ? 1 : 0, a.s, a.rs, a.rs32,
                                      a.cap, a.off, static_cast<int>(rows * a.n_ext2), a.wsrc,
                                      static_cast<int>(a.c1), static_cast<int>(a.kp), a.t, rt,
                                      a.scale, a.amax, a.qmax, a.q, a.ldq, a.sat);
    };
    if (a.pack4)
        run(k_flatten_quant<XT, true>);
    else
        run(k_flatten_quant<XT, false>);
    FQG_CUDA(cudaGetLastError());
}

}  // namespace

void flatten_quant(const FlattenArgs& a, cudaStream_t st) {
    require(a.kp % 32 == 0, "flatten: K' must be a multiple of 32");
    require(a.m >= 1 && a.k >= 1, "flatten: empty input");
    if (flatten16(a, st)) return;
    switch (a.x_dtype) {
        case FQG_F64: launch_flatten_t<double>(a, st); break;
        case FQG_F32: launch_flatten_t<float>(a, st); break;
        case FQG_F16: launch_flatten_t<__half>(a, st); break;
        case FQG_BF16: launch_flatten_t<__nv_bfloat16>(a, st); break;
        default: throw Error(FQG_ERR_INVALID, "flatten: unsupported activation dtype");
    }
    if (a.rowsum != nullptr) operand_rowsum(a.q, a.ldq, a.m, a.kp, a.pack4, a.rowsum, st);
}

void operand_rowsum(const uint8_t* q, int64_t ldq, int64_t m, int64_t kp, bool pack4,
                    int32_t* out, cudaStream_t st) {
    require(ldq % 16 == 0 && reinterpret_cast<uintptr_t>(q) % 16 == 0,
            "rowsum: operand rows must be 16-byte aligned");
    k_rowsum<<<static_cast<unsigned>((m + 7) / 8), 256, 0, st>>>(
        q, ldq, static_cast<int>(m), static_cast<int>(pack4 ? kp / 2 : kp), pack4, out);
    FQG_CUDA(cudaGetLastError());
}

void weight_absmax(const double* w, int64_t k, int64_t ncols, const double* s,
                   const int32_t* capw_src, double t_w, unsigned long long* amax,
                   unsigned int* overflow, int num_sms, cudaStream_t st) {
    const int64_t total = k * ncols;
    const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, num_sms * 8));
    k_weight_absmax<<<grid, 256, 0, st>>>(w, static_cast<int>(k), ncols, s, capw_src, t_w,
                                          1.0 / t_w, amax, overflow);
    FQG_CUDA(cudaGetLastError());
}

void weight_quant(const double* w, int64_t ldw, int64_t n_begin, int64_t n, const double* s,
                  const int32_t* wmap, const int32_t* wcap, int64_t kp, double t_w, double s_w,
                  double qmax, bool pack4, uint8_t* wq, int64_t ldq, cudaStream_t st) {
    dim3 grid(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((kp + WQ_TK - 1) / WQ_TK));
    auto run = [&](auto kern) {
        kern<<<grid, 256, 0, st>>>(w, ldw, n_begin, static_cast<int>(n), s, wmap, wcap,
                                   static_cast<int>(kp), t_w, 1.0 / t_w, s_w, 1.0 / s_w, qmax, wq,
                                   ldq);
    };
    if (pack4)
        run(k_weight_quant<true>);
    else
        run(k_weight_quant<false>);
    FQG_CUDA(cudaGetLastError());
}

}  // namespace fqg
