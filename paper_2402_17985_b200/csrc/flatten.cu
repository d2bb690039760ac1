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
// Exactness. Every decision the reference makes in FP64 is made here on the
// same operands with the same IEEE operations: the divide x/s_j, fmod, the
// divide (a - rem)/T, llround, the divide piece/scale and round-half-away.
// CUDA's double '/', fmod, llround and round are correctly rounded / exact;
// the explicit __d*_rn intrinsics keep nvcc from contracting anything into
// an FMA. Pieces equal to +-T quantize to +-round(T/scale) (computed once),
// pieces that are 0 quantize to 0, so only the remainder piece needs a divide.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include "fqg_internal.h"
#include "kernels.h"

namespace fqg {
namespace {

template <typename T>
__device__ __forceinline__ double to_f64(T v);
template <>
__device__ __forceinline__ double to_f64<double>(double v) { return v; }
template <>
__device__ __forceinline__ double to_f64<float>(float v) { return static_cast<double>(v); }
template <>
__device__ __forceinline__ double to_f64<__half>(__half v) {
    return static_cast<double>(__half2float(v));
}
template <>
__device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 v) {
    return static_cast<double>(__bfloat162float(v));
}

// Split of one element against T with plan capacity `cap` slots
// (flatten.cpp:8-15 + split_into_slots :60-74). Returns the saturated flag.
struct Split {
    long long cnt;  // number of full +-T pieces (after saturation clamp)
    double rem;     // remainder piece magnitude (0 when saturated)
    double sign;
    bool sat;
};

__device__ __forceinline__ Split split_elem(double v, double t, long long cap) {
    Split r;
    r.sign = v < 0.0 ? -1.0 : 1.0;
    const double a = fabs(v);
    r.rem = fmod(a, t);
    r.cnt = llround(__ddiv_rn(__dsub_rn(a, r.rem), t));
    r.sat = r.cnt > cap || (r.cnt == cap && r.rem > 0.0);
    if (r.sat) {
        r.cnt = cap;
        r.rem = 0.0;
    }
    return r;
}

// quantize.cpp:44-45: clamp(round(v / s), -qmax, qmax), half away from zero.
__device__ __forceinline__ int quant(double piece, double scale, double qmax) {
    double r = round(__ddiv_rn(piece, scale));
    r = r < -qmax ? -qmax : (qmax < r ? qmax : r);
    return static_cast<int>(r);
}

// Per-source-element code: [0,16) piece count, [16,24) q of the remainder
// piece, [24,32) q of a full piece (sign included).
__device__ __forceinline__ uint32_t make_code(long long cnt, int qrem, int qfull) {
    return static_cast<uint32_t>(cnt) | (static_cast<uint32_t>(qrem & 0xFF) << 16) |
           (static_cast<uint32_t>(qfull & 0xFF) << 24);
}
__device__ __forceinline__ int decode(uint32_t code, int p) {
    const int cnt = static_cast<int>(code & 0xFFFFu);
    if (p < cnt) return static_cast<int>(static_cast<int8_t>(code >> 24));
    if (p == cnt) return static_cast<int>(static_cast<int8_t>(code >> 16));
    return 0;
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

// Static or dynamic activation scale -> (scale, q of a full +-T piece).
__device__ __forceinline__ double act_scale_of(const double* scale, const unsigned long long* amax,
                                               double qmax) {
    if (amax == nullptr) return scale[0];
    // quantize.cpp:34-40: s = max|M| / qmax (degenerate 0 is flagged by the host)
    return __ddiv_rn(__longlong_as_double(static_cast<long long>(*amax)), qmax);
}

// ------------------------------------------------------------------ K1
template <typename XT, bool PACK4>
__global__ void __launch_bounds__(256)
    k_flatten_quant(const XT* __restrict__ x, int64_t ldx, int m, int k, int rows_per_cta,
                    const double* __restrict__ s, const int32_t* __restrict__ cap,
                    const int32_t* __restrict__ amap, int kp, double t,
                    double* __restrict__ scale, const unsigned long long* __restrict__ amax,
                    double qmax, uint8_t* __restrict__ q, int64_t ldq,
                    unsigned long long* __restrict__ sat_out) {
    extern __shared__ uint32_t codes[];  // [rows_per_cta][k]
    __shared__ unsigned long long red[8];
    const int row0 = blockIdx.x * rows_per_cta;
    const int nrows = min(rows_per_cta, m - row0);
    const double as = act_scale_of(scale, amax, qmax);
    if (amax != nullptr && blockIdx.x == 0 && threadIdx.x == 0) scale[0] = as;
    const int qT = quant(t, as, qmax);

    // Phase 1: one split per source element (i, j).
    unsigned long long sat = 0;
    for (int r = 0; r < nrows; ++r) {
        const XT* xr = x + static_cast<int64_t>(row0 + r) * ldx;
        uint32_t* cr = codes + static_cast<int64_t>(r) * k;
        for (int j = threadIdx.x; j < k; j += blockDim.x) {
            const double v = __ddiv_rn(to_f64<XT>(xr[j]), s[j]);  // smoothing.cpp:75
            const long long cp = cap[j];
            const Split sp = split_elem(v, t, cp);
            sat += sp.sat ? 1ull : 0ull;
            const int qrem = sp.cnt < cp ? quant(sp.sign * sp.rem, as, qmax) : 0;
            cr[j] = make_code(sp.cnt, qrem, sp.sign < 0.0 ? -qT : qT);
        }
    }
    __syncthreads();

    // Phase 2: gather 16 output columns per thread through the composite map.
    const int chunks = kp / 16;
    for (int c = threadIdx.x; c < chunks; c += blockDim.x) {
        int32_t mp[16];
        const int4* m4 = reinterpret_cast<const int4*>(amap + c * 16);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int4 w = __ldg(m4 + v);
            mp[4 * v] = w.x;
            mp[4 * v + 1] = w.y;
            mp[4 * v + 2] = w.z;
            mp[4 * v + 3] = w.w;
        }
        for (int r = 0; r < nrows; ++r) {
            const uint32_t* cr = codes + static_cast<int64_t>(r) * k;
            int qv[16];
#pragma unroll
            for (int e = 0; e < 16; ++e)
                qv[e] = mp[e] < 0 ? 0 : decode(cr[mp[e] >> 12], mp[e] & 0xFFF);
            uint8_t* qr = q + static_cast<int64_t>(row0 + r) * ldq;
            if constexpr (PACK4) {
                uint32_t w0 = 0, w1 = 0;
#pragma unroll
                for (int e = 0; e < 8; ++e) w0 |= static_cast<uint32_t>(qv[e] & 0xF) << (4 * e);
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    w1 |= static_cast<uint32_t>(qv[8 + e] & 0xF) << (4 * e);
                *reinterpret_cast<uint2*>(qr + c * 8) = make_uint2(w0, w1);
            } else {
                uint32_t w[4];
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    w[v] = (static_cast<uint32_t>(qv[4 * v] & 0xFF)) |
                           (static_cast<uint32_t>(qv[4 * v + 1] & 0xFF) << 8) |
                           (static_cast<uint32_t>(qv[4 * v + 2] & 0xFF) << 16) |
                           (static_cast<uint32_t>(qv[4 * v + 3] & 0xFF) << 24);
                *reinterpret_cast<uint4*>(qr + c * 16) = make_uint4(w[0], w[1], w[2], w[3]);
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
                 const double* __restrict__ s, const int32_t* __restrict__ cap, double t,
                 unsigned long long* __restrict__ amax) {
    __shared__ double red[8];
    double mx = 0.0;
    const int64_t total = static_cast<int64_t>(m) * k;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(idx / k), j = static_cast<int>(idx % k);
        const double v = __ddiv_rn(to_f64<XT>(x[static_cast<int64_t>(i) * ldx + j]), s[j]);
        const Split sp = split_elem(v, t, cap[j]);
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
                    double t_w, unsigned long long* __restrict__ amax,
                    unsigned int* __restrict__ overflow) {
    __shared__ double red[8];
    double mx = 0.0;
    bool over = false;
    const int64_t total = static_cast<int64_t>(k) * ncols;
    for (int64_t idx = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; idx < total;
         idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(idx / ncols);
        const double v = __dmul_rn(w[idx], s[j]);  // scale_rows, smoothing.cpp:88
        const Split sp = split_elem(v, t_w, capw_src[j]);
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
                   const int32_t* __restrict__ wcap, int kp, double t_w, double s_w, double qmax,
                   uint8_t* __restrict__ wq, int64_t ldq) {
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
                const Split sp = split_elem(v, t_w, wcap[kq]);
                double piece = 0.0;
                if (p < sp.cnt)
                    piece = sp.sign * t_w;
                else if (p == sp.cnt)
                    piece = sp.sign * sp.rem;
                qv = quant(piece, s_w, qmax);
            }
        }
        tile[tx][kk] = static_cast<int8_t>(qv);
    }
    __syncthreads();
    // Write: each warp writes rows n0+ty, n0+ty+8, ...; lane covers 4 k' values.
    for (int r = ty; r < 32; r += 8) {
        const int nn = n0 + r;
        if (nn >= n) continue;
        const int kk = tx * 4;
        if (k0 + kk >= kp) continue;
        const int8_t* src = &tile[r][kk];
        if constexpr (PACK4) {
            const uint16_t b = static_cast<uint16_t>((src[0] & 0xF) | ((src[1] & 0xF) << 4) |
                                                     ((src[2] & 0xF) << 8) | ((src[3] & 0xF) << 12));
            *reinterpret_cast<uint16_t*>(wq + nn * ldq + (k0 + kk) / 2) = b;
        } else {
            const uint32_t b = static_cast<uint32_t>(static_cast<uint8_t>(src[0])) |
                               (static_cast<uint32_t>(static_cast<uint8_t>(src[1])) << 8) |
                               (static_cast<uint32_t>(static_cast<uint8_t>(src[2])) << 16) |
                               (static_cast<uint32_t>(static_cast<uint8_t>(src[3])) << 24);
            *reinterpret_cast<uint32_t*>(wq + nn * ldq + k0 + kk) = b;
        }
    }
}

template <typename XT>
void launch_flatten_t(const FlattenArgs& a, cudaStream_t st) {
    const int dev_sm = a.num_sms;
    if (a.amax != nullptr) {
        const int64_t total = a.m * a.k;
        const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, dev_sm * 8));
        k_act_absmax<XT><<<grid, 256, 0, st>>>(static_cast<const XT*>(a.x), a.ldx,
                                                static_cast<int>(a.m), static_cast<int>(a.k), a.s,
                                                a.cap, a.t, a.amax);
        FQG_CUDA(cudaGetLastError());
    }
    const int64_t row_bytes = a.k * 4;
    int rows = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(8, (96 * 1024) / row_bytes)));
    // keep at least ~2 waves of CTAs
    while (rows > 1 && (a.m + rows - 1) / rows < 2 * dev_sm) rows >>= 1;
    const int64_t smem = rows * row_bytes;
    require(smem <= 200 * 1024, "flatten: K too large for the shared-memory code buffer");
    const int grid = static_cast<int>((a.m + rows - 1) / rows);
    if (a.pack4) {
        auto kern = k_flatten_quant<XT, true>;
        FQG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        kern<<<grid, 256, smem, st>>>(static_cast<const XT*>(a.x), a.ldx, static_cast<int>(a.m),
                                      static_cast<int>(a.k), rows, a.s, a.cap, a.amap,
                                      static_cast<int>(a.kp), a.t, a.scale, a.amax, a.qmax, a.q,
                                      a.ldq, a.sat);
    } else {
        auto kern = k_flatten_quant<XT, false>;
        FQG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        kern<<<grid, 256, smem, st>>>(static_cast<const XT*>(a.x), a.ldx, static_cast<int>(a.m),
                                      static_cast<int>(a.k), rows, a.s, a.cap, a.amap,
                                      static_cast<int>(a.kp), a.t, a.scale, a.amax, a.qmax, a.q,
                                      a.ldq, a.sat);
    }
    FQG_CUDA(cudaGetLastError());
}

}  // namespace

void flatten_quant(const FlattenArgs& a, cudaStream_t st) {
    require(a.kp % 32 == 0, "flatten: K' must be a multiple of 32");
    require(a.m >= 1 && a.k >= 1, "flatten: empty input");
    switch (a.x_dtype) {
        case FQG_F64: return launch_flatten_t<double>(a, st);
        case FQG_F32: return launch_flatten_t<float>(a, st);
        case FQG_F16: return launch_flatten_t<__half>(a, st);
        case FQG_BF16: return launch_flatten_t<__nv_bfloat16>(a, st);
        default: throw Error(FQG_ERR_INVALID, "flatten: unsupported activation dtype");
    }
}

void weight_absmax(const double* w, int64_t k, int64_t ncols, const double* s,
                   const int32_t* capw_src, double t_w, unsigned long long* amax,
                   unsigned int* overflow, int num_sms, cudaStream_t st) {
    const int64_t total = k * ncols;
    const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, num_sms * 8));
    k_weight_absmax<<<grid, 256, 0, st>>>(w, static_cast<int>(k), ncols, s, capw_src, t_w, amax,
                                          overflow);
    FQG_CUDA(cudaGetLastError());
}

void weight_quant(const double* w, int64_t ldw, int64_t n_begin, int64_t n, const double* s,
                  const int32_t* wmap, const int32_t* wcap, int64_t kp, double t_w, double s_w,
                  double qmax, bool pack4, uint8_t* wq, int64_t ldq, cudaStream_t st) {
    dim3 grid(static_cast<unsigned>((n + 31) / 32), static_cast<unsigned>((kp + WQ_TK - 1) / WQ_TK));
    if (pack4)
        k_weight_quant<true><<<grid, 256, 0, st>>>(w, ldw, n_begin, static_cast<int>(n), s, wmap,
                                                   wcap, static_cast<int>(kp), t_w, s_w, qmax, wq,
                                                   ldq);
    else
        k_weight_quant<false><<<grid, 256, 0, st>>>(w, ldw, n_begin, static_cast<int>(n), s, wmap,
                                                    wcap, static_cast<int>(kp), t_w, s_w, qmax, wq,
                                                    ldq);
    FQG_CUDA(cudaGetLastError());
}

}  // namespace fqg
