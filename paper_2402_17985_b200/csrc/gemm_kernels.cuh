// gemm_kernels.cuh — K4: the flattened low-bit GEMM on 5th-gen tensor cores.
// Included by the gemm_*.cu translation units (one per operand-format pair, so
// the ~100 kernel instantiations compile in parallel); gemm.cu holds the plan.
//
//   Y[M,N] = epi( sum_k A[M,k] * B[N,k] ),  A,B int8 K-major, INT32 accumulate
//
// replaces fq::int_matmul_raw + fq::int_matmul (quantize.cpp:166-198). The
// accumulators are exact int32 (|acc| <= K' * qmax^2 < 2^31 for K' <= 133144,
// checked by the host), so the result is bit-identical to the reference's
// int64 sums; the epilogue then forms y = double(acc) * (s_x * s_w) exactly as
// quantize.cpp:193-196 does and rounds once to the output type.
//
// Structure (one CTA per SM, persistent over output tiles, 256 threads):
//   warp 0 lane 0 : TMA producer — A tile 128x128B and B tile BNx128B per stage,
//                   128-byte swizzle, OOB rows/cols zero-filled by the TMA unit
//   warp 1        : TMEM allocator (2*BN columns: double-buffered accumulator);
//                   lane 0 issues tcgen05.mma.cta_group::1.kind::i8 128xBNx32
//   warps 4..7    : epilogue — tcgen05.ld 32x32b, dequant + bias, convert, store
// Pipelines: smem ring full/empty mbarriers (TMA <-> MMA, tcgen05.commit frees a
// slot), TMEM full/empty mbarriers (MMA <-> epilogue), so the epilogue of tile
// i overlaps the main loop of tile i+1.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#pragma once
#include "fqg_internal.h"
#include "ptx.cuh"

namespace fqg {
namespace {

constexpr int BM = 128;       // UMMA M (cta_group::1)
// Operand formats inside the kernels: int8 bytes, signed packed int4 (FQG_I4),
// or biased packed int4 (stored nibble = q + 8, the layer's weight format: it
// unpacks with one AND per 4 values and is fed to the MMA as UNSIGNED int8;
// the epilogue subtracts 8 * rowsum(A) per output row, exact in int32).
constexpr int F8 = 0, FS4 = 1, FU4 = 2;
constexpr int BK = 128;       // K bytes per stage = one 128B swizzle row
constexpr int UK = 32;        // K per tcgen05.mma kind::i8

// Shared-memory plan. The "raw" ring is what the TMA writes: int8 operands in
// the 128B-swizzled UMMA layout, packed int4 operands as plain 64-byte rows.
// With a packed operand, unpack warps expand it into the "unpacked" ring
// (int8, 128B-swizzled) before the MMA reads it.
template <int BN, int STAGES, bool APK, bool BPK>
struct Layout {
    static constexpr bool packed = APK || BPK;
    static constexpr int a_raw = APK ? BM * BK / 2 : BM * BK;
    static constexpr int b_raw = BPK ? BN * BK / 2 : BN * BK;
    static constexpr int raw_stage = a_raw + b_raw;  // multiple of 1024
    static constexpr int USTAGES = packed ? 2 : 0;
    static constexpr int a_unp = APK ? BM * BK : 0;
    static constexpr int b_unp = BPK ? BN * BK : 0;
    static constexpr int unp_stage = a_unp + b_unp;
    static constexpr int unp_off = STAGES * raw_stage;
    static constexpr int bar_off = unp_off + USTAGES * unp_stage;
    static constexpr int n_bars = 2 * STAGES + 2 * USTAGES + 4;
    static constexpr int total = bar_off + n_bars * 8 + 16 + 1024;  // + alignment slack
    static constexpr int unpack_warps = packed ? 8 : 0;
    static constexpr int threads = 256 + 32 * unpack_warps;
    // Arrivals that free a raw stage: the MMA commit if it reads an int8
    // operand straight from the raw stage, plus one per unpack warp.
    // Unpack warps form two teams that take alternate k-blocks (two stages in
    // flight); a stage is read by one team.
    static constexpr int team_warps = unpack_warps / 2;
    static constexpr int raw_release = (APK && BPK ? 0 : 1) + team_warps;
};

// FQG_I4 layout: per group of 32 k, byte i (0..15) = q[i] & 15 | q[16 + i] << 4.
// 16 packed bytes -> the group's 32 int8: low nibbles are k 0..15 in order,
// high nibbles k 16..31. Per nibble v: ((v ^ 8) + 0x78) ^ 0x80 is v
// sign-extended to 8 bits with no carry between byte lanes ((v ^ 8) + 0x78
// <= 0x87); the AND and first XOR fuse into one LOP3.
__device__ __forceinline__ uint32_t sext4x4(uint32_t nib) {
    return ((nib ^ 0x08080808u) + 0x78787878u) ^ 0x80808080u;
}
__device__ __forceinline__ void unpack16(uint4 p, uint4& o0, uint4& o1) {
    o0 = make_uint4(sext4x4(p.x & 0x0F0F0F0Fu), sext4x4(p.y & 0x0F0F0F0Fu),
                    sext4x4(p.z & 0x0F0F0F0Fu), sext4x4(p.w & 0x0F0F0F0Fu));
    o1 = make_uint4(sext4x4((p.x >> 4) & 0x0F0F0F0Fu), sext4x4((p.y >> 4) & 0x0F0F0F0Fu),
                    sext4x4((p.z >> 4) & 0x0F0F0F0Fu), sext4x4((p.w >> 4) & 0x0F0F0F0Fu));
}

// Biased nibbles u = q + 8 in [0, 15] -> unsigned bytes: one AND (low) and
// SHIFT + AND (high) per 4 values.
__device__ __forceinline__ void unpack16_biased(uint4 p, uint4& o0, uint4& o1) {
    o0 = make_uint4(p.x & 0x0F0F0F0Fu, p.y & 0x0F0F0F0Fu, p.z & 0x0F0F0F0Fu, p.w & 0x0F0F0F0Fu);
    o1 = make_uint4((p.x >> 4) & 0x0F0F0F0Fu, (p.y >> 4) & 0x0F0F0F0Fu, (p.z >> 4) & 0x0F0F0F0Fu,
                    (p.w >> 4) & 0x0F0F0F0Fu);
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

// Expand `rows` x 64 packed bytes (plain rows) into rows x 128 int8 in the
// 128B-swizzle K-major layout: 16-byte chunk c of row r at r*128 + ((c ^ r%8) * 16).
// Shared-window 32-bit addresses (ld/st.shared), so no generic-address math.
template <int FMT>
__device__ __forceinline__ void unpack_tile(const uint8_t* src, uint8_t* dst, int rows, int tid,
                                            int nthreads) {
    const uint32_t s0 = ptx::smem_u32(src), d0 = ptx::smem_u32(dst);
#pragma unroll 4
    for (int u = tid; u < rows * 4; u += nthreads) {
        const int r = u >> 2, pc = u & 3;
        const uint4 p = lds128(s0 + static_cast<uint32_t>(u) * 16);  // == r * 64 + pc * 16
        uint4 o0, o1;
        if constexpr (FMT == FU4)
            unpack16_biased(p, o0, o1);
        else
            unpack16(p, o0, o1);
        const uint32_t row = d0 + static_cast<uint32_t>(r) * 128;
        const int sw = r & 7;
        sts128(row + (((2 * pc) ^ sw) << 4), o0);
        sts128(row + (((2 * pc + 1) ^ sw) << 4), o1);
    }
}

// Exact int32 -> double without the quarter-rate I2F.F64 conversion: the
// double with high word 0x43300000 and low word acc ^ 2^31 is 2^52 + acc + 2^31;
// one DADD (full FP64 rate) removes the offset exactly.
__device__ __forceinline__ double i2d_exact(int32_t acc) {
    return __dsub_rn(__hiloint2double(0x43300000, acc ^ static_cast<int32_t>(0x80000000u)),
                     4503601774854144.0);  // 2^52 + 2^31
}

// cvt16_certified mode bits from the kernel's accumulator bound and S.
__device__ __forceinline__ int cvt_mode(int small_acc, float s32) {
    return (small_acc != 0 ? 1 : 0) | (s32 >= 6.103515625e-05f ? 2 : 0);
}

__device__ __forceinline__ double load_bias(const void* bias, int dt, int col) {
    switch (dt) {
        case FQG_F32: return static_cast<double>(static_cast<const float*>(bias)[col]);
        case FQG_F64: return static_cast<const double*>(bias)[col];
        case FQG_F16: return static_cast<double>(__half2float(static_cast<const __half*>(bias)[col]));
        case FQG_BF16:
            return static_cast<double>(__bfloat162float(static_cast<const __nv_bfloat16*>(bias)[col]));
        default: return 0.0;
    }
}

template <int OUT>
__device__ __forceinline__ void store_one(void* y, int64_t idx, int32_t acc, double s, double b) {
    if constexpr (OUT == FQG_I32) {
        static_cast<int32_t*>(y)[idx] = acc;
    } else {
        // quantize.cpp:196: out = double(acc) * (s_x * s_w); + bias extension
        // (rounded separately: the reference output plus the bias, no FMA).
        const double v = __dadd_rn(__dmul_rn(i2d_exact(acc), s), b);
        if constexpr (OUT == FQG_F64) static_cast<double*>(y)[idx] = v;
        if constexpr (OUT == FQG_F32) static_cast<float*>(y)[idx] = static_cast<float>(v);
        if constexpr (OUT == FQG_F16) static_cast<__half*>(y)[idx] = __double2half(v);
        if constexpr (OUT == FQG_BF16) static_cast<__nv_bfloat16*>(y)[idx] = __double2bfloat16(v);
    }
}

// 2-byte outputs, certified FP32 path: y = RN16(double(acc) * S) (quantize.cpp:193-196,
// rounded once) computed as RN32(RN32(acc) * RN32(S)), whose error is below 3
// fp32 ulps (RN32(acc) is exact for |acc| < 2^24). The FP32 value rounds to the
// same 16-bit value as the exact product unless it lies within 4 fp32 ulps of a
// 16-bit rounding midpoint (low 13 mantissa bits 0x1000 for fp16, low 16 bits
// 0x8000 for bf16) or in the 16-bit subnormal range; those elements (~0.1%)
// take the exact FP64 path. Everything runs on the full-rate FP32/ALU pipes
// instead of the quarter-rate FP64 conversions.
template <int OUT, int NV>
__device__ __forceinline__ void cvt16_certified(const uint32_t (&r)[NV], int32_t corr, float s32,
                                                double s, int mode, uint32_t (&packed)[NV / 2]) {
    // mode bit 0: |acc - corr| < 2^22 (one-add int -> float); bit 1: S >= 2^-14, so
    // only an exact zero can land in the 16-bit subnormal range (no range check).
    const bool small_acc = (mode & 1) != 0, no_tiny = (mode & 2) != 0;
    float v[NV];
    // t = (bits + 4 - midpoint) << (32 - mantissa bits dropped): t <= 8 << shift
    // <=> within 4 fp32 ulps of a 16-bit midpoint; one IMAD (FMA pipe) per
    // element, tracked as a running minimum (one IMNMX). Per element: IADD3,
    // FADD, FMUL, IMAD, IMNMX: 3 ops on the FMA pipe, 2 on the ALU pipe.
    constexpr uint32_t kMul = OUT == FQG_F16 ? (1u << 19) : (1u << 16);
    constexpr uint32_t kAdd = (OUT == FQG_F16 ? (4u - 0x1000u) : (4u - 0x8000u)) * kMul;
    uint32_t tmin = 0xFFFFFFFFu;
    float vmin = 3.0e38f;
    const int32_t mag0 = 0x4B400000 - corr;  // 1.5 * 2^23 magic, row correction folded in
#pragma unroll
    for (int e = 0; e < NV; ++e) {
        float xf;
        if (small_acc) {  // |acc - corr| < 2^22: exact by the magic number
            xf = __fsub_rn(__int_as_float(mag0 + static_cast<int32_t>(r[e])), 12582912.0f);
        } else {  // a = hi * 2^16 + lo, both exact; one rounding in the FMA
            const int32_t a = static_cast<int32_t>(r[e]) - corr;
            const float fh = __fsub_rn(__int_as_float(0x4B400000 + (a >> 16)), 12582912.0f);
            const float fl = __fsub_rn(__int_as_float(0x4B000000 | (a & 0xFFFF)), 8388608.0f);
            xf = __fmaf_rn(fh, 65536.0f, fl);
        }
        const float yv = __fmul_rn(xf, s32);
        v[e] = yv;
        tmin = min(tmin, __float_as_uint(yv) * kMul + kAdd);
        if (!no_tiny) vmin = fminf(vmin, fabsf(yv));
    }
#pragma unroll
    for (int q = 0; q < NV / 2; ++q) {
        if constexpr (OUT == FQG_F16) {
            __half2 h = __floats2half2_rn(v[2 * q], v[2 * q + 1]);
            packed[q] = *reinterpret_cast<uint32_t*>(&h);
        } else {
            __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * q], v[2 * q + 1]);
            packed[q] = *reinterpret_cast<uint32_t*>(&h);
        }
    }
    constexpr uint32_t kNear = 8u * kMul;
    const float kTiny = OUT == FQG_F16 ? 6.103515625e-05f : 2.3509887e-38f;  // 2^-14, 2^-125
    if (tmin <= kNear || vmin < kTiny) {
        // some element may round differently from the exact product: redo the
        // chunk's uncertain elements on the exact FP64 path (static indices: a
        // dynamic r[e] / packed[q] would move the arrays to local memory)
#pragma unroll
        for (int e = 0; e < NV; ++e) {
            if (__float_as_uint(v[e]) * kMul + kAdd <= kNear || fabsf(v[e]) < kTiny) {
                const double vd = __dmul_rn(i2d_exact(static_cast<int32_t>(r[e]) - corr), s);
                uint32_t hb;
                if constexpr (OUT == FQG_F16)
                    hb = __half_as_ushort(__double2half(vd));
                else
                    hb = __bfloat16_as_ushort(__double2bfloat16(vd));
                packed[e >> 1] = (packed[e >> 1] & ~(0xFFFFu << ((e & 1) * 16))) |
                                 (hb << ((e & 1) * 16));
            }
        }
    }
}

// 32-byte store (one full sector per lane): st.global.v8.b32 (sm_100).
__device__ __forceinline__ void stg256(void* p, const uint32_t (&v)[8]) {
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

// 32 consecutive columns of one row, from 32 accumulator registers.
template <int OUT>
__device__ __forceinline__ void store_row_chunk(void* y, int64_t base, uint32_t (&r)[32],
                                                double s, const void* bias, int bias_dt, int col0,
                                                int ncols, bool vec, int32_t corr, float s32 = 0.0f,
                                                int cvt_mode = 0) {
    if constexpr (OUT == FQG_F16 || OUT == FQG_BF16) {
        if (vec && ncols == 32 && bias == nullptr) {
            uint32_t packed[16];
            cvt16_certified<OUT, 32>(r, corr, s32, s, cvt_mode, packed);
            uint4* p = reinterpret_cast<uint4*>(static_cast<uint16_t*>(y) + base);
#pragma unroll
            for (int q = 0; q < 4; ++q)  // streaming stores: the output is not re-read here
                __stcs(p + q, make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2],
                                         packed[4 * q + 3]));
            return;
        }
    }
    if (corr != 0) {
#pragma unroll
        for (int c = 0; c < 32; ++c) r[c] = static_cast<uint32_t>(static_cast<int32_t>(r[c]) - corr);
    }
    if (vec && ncols == 32) {
        if constexpr (OUT == FQG_I32) {
            int4* p = reinterpret_cast<int4*>(static_cast<int32_t*>(y) + base);
#pragma unroll
            for (int q = 0; q < 8; ++q)
                p[q] = make_int4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]);
            return;
        } else if constexpr (OUT == FQG_F16 || OUT == FQG_BF16) {
            uint32_t packed[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                double v0 = __dmul_rn(i2d_exact(static_cast<int32_t>(r[2 * q])), s);
                double v1 = __dmul_rn(i2d_exact(static_cast<int32_t>(r[2 * q + 1])), s);
                if (bias) {
                    v0 = __dadd_rn(v0, load_bias(bias, bias_dt, col0 + 2 * q));
                    v1 = __dadd_rn(v1, load_bias(bias, bias_dt, col0 + 2 * q + 1));
                }
                if constexpr (OUT == FQG_F16) {
                    __half2 h = __halves2half2(__double2half(v0), __double2half(v1));
                    packed[q] = *reinterpret_cast<uint32_t*>(&h);
                } else {
                    __nv_bfloat162 h;
                    h.x = __double2bfloat16(v0);
                    h.y = __double2bfloat16(v1);
                    packed[q] = *reinterpret_cast<uint32_t*>(&h);
                }
            }
            uint4* p = reinterpret_cast<uint4*>(static_cast<uint16_t*>(y) + base);
#pragma unroll
            for (int q = 0; q < 4; ++q)  // streaming stores: the output is not re-read here
                __stcs(p + q, make_uint4(packed[4 * q], packed[4 * q + 1], packed[4 * q + 2],
                                         packed[4 * q + 3]));
            return;
        }
    }
#pragma unroll
    for (int c = 0; c < 32; ++c) {
        if (c < ncols) {
            const double b = bias ? load_bias(bias, bias_dt, col0 + c) : 0.0;
            store_one<OUT>(y, base + c, static_cast<int32_t>(r[c]), s, b);
        }
    }
}

template <int OUT>
struct OutT;
template <> struct OutT<FQG_I32> { using T = int32_t; };
template <> struct OutT<FQG_F64> { using T = double; };
template <> struct OutT<FQG_F32> { using T = float; };
template <> struct OutT<FQG_F16> { using T = __half; };
template <> struct OutT<FQG_BF16> { using T = __nv_bfloat16; };

template <int OUT>
__device__ __forceinline__ typename OutT<OUT>::T convert_out(int32_t acc, double s, double b) {
    if constexpr (OUT == FQG_I32) {
        return acc;
    } else {
        const double v = __dadd_rn(__dmul_rn(i2d_exact(acc), s), b);  // quantize.cpp:196 (+ bias)
        if constexpr (OUT == FQG_F64) return v;
        if constexpr (OUT == FQG_F32) return static_cast<float>(v);
        if constexpr (OUT == FQG_F16) return __double2half(v);
        if constexpr (OUT == FQG_BF16) return __double2bfloat16(v);
    }
}

template <int BN, int STAGES, int OUT, int AF, int BF>
__global__ void __launch_bounds__(Layout<BN, STAGES, AF != F8, BF != F8>::threads, 1)
    k_gemm_i8(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              void* __restrict__ y, int64_t ldy, int m, int n, int num_kb,
              const double* __restrict__ scale, const void* __restrict__ bias, int bias_dt,
              int vec_ok, const int32_t* __restrict__ rowsum, int small_acc) {
    constexpr bool APK = AF != F8, BPK = BF != F8;
    using L = Layout<BN, STAGES, APK, BPK>;
    constexpr int U = L::USTAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::bar_off);
    uint64_t* empty = full + STAGES;
    uint64_t* ufull = empty + STAGES;   // [U] unpacked stage ready
    uint64_t* uempty = ufull + U;       // [U] unpacked stage consumed by the MMA
    uint64_t* tfull = uempty + U;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int num_m = (m + BM - 1) / BM;
    const int num_n = (n + BN - 1) / BN;
    const int num_tiles = num_m * num_n;

    if (threadIdx.x == 0) {
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], L::raw_release);
        }
        for (int u = 0; u < U; ++u) {
            ptx::mbar_init(&ufull[u], L::team_warps);
            ptx::mbar_init(&uempty[u], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 4);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 1) {
        ptx::tmem_alloc(tmem_holder, 2 * BN);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer ----------------
        const uint64_t keep = ptx::policy_evict_last();
        int stage = 0;
        uint32_t phase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            const int m_blk = tile % num_m, n_blk = tile / num_m;
            for (int kb = 0; kb < num_kb; ++kb) {
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* sa = smem + stage * L::raw_stage;
                uint8_t* sb = sa + L::a_raw;
                ptx::mbar_arrive_expect_tx(&full[stage], L::raw_stage);
                ptx::tma_load_2d_hint(sa, &tmA, &full[stage], kb * (APK ? BK / 2 : BK), m_blk * BM,
                                      keep);
                ptx::tma_load_2d_hint(sb, &tmB, &full[stage], kb * (BPK ? BK / 2 : BK), n_blk * BN,
                                      keep);
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer ----------------
        constexpr uint32_t idesc = ptx::idesc_i8(BM, BN, BF == FU4);
        int stage = 0, us = 0;
        uint32_t phase = 0, uphase = 0;
        int it = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
            ptx::tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * BN;
            for (int kb = 0; kb < num_kb; ++kb) {
                ptx::mbar_wait(&full[stage], phase);
                if constexpr (L::packed) ptx::mbar_wait(&ufull[us], uphase);
                ptx::tc_fence_after();
                const uint32_t raw = ptx::smem_u32(smem + stage * L::raw_stage);
                const uint32_t unp = ptx::smem_u32(smem + L::unp_off + us * L::unp_stage);
                const uint32_t a_addr = APK ? unp : raw;
                const uint32_t b_addr = BPK ? unp + L::a_unp : raw + L::a_raw;
#pragma unroll
                for (int k = 0; k < BK / UK; ++k) {
                    ptx::mma_i8(d_tmem, ptx::smem_desc_sw128_kmajor(a_addr + k * UK),
                                ptx::smem_desc_sw128_kmajor(b_addr + k * UK), idesc,
                                (kb | k) != 0 ? 1u : 0u);
                }
                if constexpr (!(APK && BPK)) ptx::mma_commit(&empty[stage]);
                if constexpr (L::packed) {
                    ptx::mma_commit(&uempty[us]);
                    if (++us == U) {
                        us = 0;
                        uphase ^= 1;
                    }
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            ptx::mma_commit(&tfull[acc]);
        }
    } else if (warp >= 4 && warp < 8) {
        // ---------------- epilogue ----------------
        const int ew = warp - 4;  // TMEM lane quarter this warp may access
        // quantize.cpp:193: the product s_x * s_w formed once in FP64.
        const double s = OUT == FQG_I32 ? 1.0 : __dmul_rn(scale[0], scale[1]);
        const float s32 = __double2float_rn(s);
        int it = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
            const int m_blk = tile % num_m, n_blk = tile / num_m;
            const int acc = it & 1;
            const uint32_t acc_phase = (it >> 1) & 1;
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            const int row = m_blk * BM + ew * 32 + lane;
            const int32_t corr = (BF == FU4 && row < m) ? 8 * rowsum[row] : 0;
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t r[32];
                ptx::tmem_ld_32x32b_x32(t_row + c * 32, r);
                ptx::tmem_wait_ld();
                const int col0 = n_blk * BN + c * 32;
                if (row < m && col0 < n) {
                    const int ncols = min(32, n - col0);
                    store_row_chunk<OUT>(y, static_cast<int64_t>(row) * ldy + col0, r, s, bias,
                                         bias_dt, col0, ncols, vec_ok != 0, corr, s32,
                                         cvt_mode(small_acc, s32));
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
        }
    } else if (L::packed && warp >= 8) {
        // ---------------- int4 -> int8 unpack warps ----------------
        const int team = (warp - 8) / (L::team_warps > 0 ? L::team_warps : 1);
        const int utid = threadIdx.x - 256 - 32 * L::team_warps * team, nut = 32 * L::team_warps;
        int stage = 0, us = 0, step = 0;
        uint32_t phase = 0, uphase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            for (int kb = 0; kb < num_kb; ++kb, ++step) {
                if ((step & 1) != team) {
                    if (++us == U) {
                        us = 0;
                        uphase ^= 1;
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                    continue;
                }
                ptx::mbar_wait(&full[stage], phase);
                ptx::mbar_wait(&uempty[us], uphase ^ 1);
                const uint8_t* raw = smem + stage * L::raw_stage;
                uint8_t* unp = smem + L::unp_off + us * L::unp_stage;
                if constexpr (APK) unpack_tile<AF>(raw, unp, BM, utid, nut);
                if constexpr (BPK) unpack_tile<BF>(raw + L::a_raw, unp + L::a_unp, BN, utid, nut);
                // generic-proxy smem writes -> visible to the tensor core (async proxy)
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive(&ufull[us]);
                    ptx::mbar_arrive(&empty[stage]);
                }
                if (++us == U) {
                    us = 0;
                    uphase ^= 1;
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        __syncwarp();
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, 2 * BN);
    }
}

// Developer instrumentation (FQG_GEMM_DEBUG=1): per-CTA cycles spent in each
// role's barrier waits. Off by default (one predicated branch per wait).
__device__ unsigned long long g_dbg[296][8];
__device__ unsigned long long g_dbg3[296][8];  // arrival (ns after start) at the final sync per warp role
__device__ __align__(16) double g_sink[32 * 32];  // FQG_GEMM_DEBUG bit 16
__device__ unsigned long long g_dbg2[296][8];  // pair packed path: see launch_pair
#define FQG_TWAIT2(slot, ...)                                                  \
    do {                                                                       \
        const long long t0_ = dbg ? clock64() : 0;                             \
        __VA_ARGS__;                                                           \
        if (dbg) atomicAdd(&g_dbg2[blockIdx.x % 296][slot], clock64() - t0_);  \
    } while (0)
#define FQG_TWAIT(slot, ...)                                                   \
    do {                                                                       \
        const long long t0_ = dbg ? clock64() : 0;                             \
        __VA_ARGS__;                                                           \
        if (dbg) atomicAdd(&g_dbg[blockIdx.x % 296][slot], clock64() - t0_);   \
    } while (0)

// ------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of 2 CTAs on one TPC computes a
// 256 x 256 output tile with tcgen05.mma.cta_group::2 (M = 256, N = 256,
// K = 32). Each CTA stages its own 128 rows of A and 128 of the 256 rows of
// B, so per SM the smem/L2 operand traffic per MMA drops from 48 KB to 32 KB
// per 128-deep k-block versus the 1-CTA 128 x 256 tile. The even CTA issues
// the MMAs; commits multicast to both CTAs' barriers; each CTA's epilogue
// drains its own TMEM half (its 128 rows x 256 columns).
//   int8 operands: 2-SM TMA (completion counted on the leader's barrier);
//   packed int4 operands: 1-SM TMA into this CTA's raw ring, local unpack
//   warps expand to int8 and signal the leader.
// NB = 256-column blocks of B per tile: NB = 1 -> 256 x 256 tiles with a
// double-buffered accumulator; NB = 2 -> 256 x 512 tiles, two accumulators
// filling TMEM (no double buffer): the A tile is read once per two MMAs, so
// L2 -> SMEM bytes per MAC drop by a quarter (the kernel is TMA-throughput bound).
// NB = 3 encodes 512 x 256 tiles (MB = 2 row sub-tiles, one 256-column B block):
// two MMAs per K step with different A and the same B, so the expanded B tile
// (the costly one with packed weights: TMA write, unpack read, unpack write,
// MMA read) is half as large per MAC as with 256 x 512, at the price of a
// second A sub-tile; shared-memory traffic per k-block and CTA drops from 144 KB
// to 128 KB for int8 A / packed B (the int4 main loop is SMEM-bandwidth bound).
template <int STAGES, bool APK, bool BPK, int NB = 1, int EPIB = 0>
struct PairLayout {
    static constexpr int BN = 256;
    static constexpr int NBS = NB == 3 ? 1 : NB;   // 256-column B blocks per tile
    static constexpr int MBS = NB == 3 ? 2 : 1;    // 256-row A sub-tiles per tile
    static constexpr int NACC = NBS * MBS == 1 ? 2 : 1;  // accumulator buffers
    static constexpr bool packed = APK || BPK;
    static constexpr int a_raw = MBS * (APK ? BM * BK / 2 : BM * BK);  // own 128 rows per sub-tile
    static constexpr int b_raw = NBS * (BPK ? (BN / 2) * BK / 2 : (BN / 2) * BK);  // own halves of B
    static constexpr int raw_stage = a_raw + b_raw;
    static constexpr int direct_bytes = (APK ? 0 : a_raw) + (BPK ? 0 : b_raw);
    static constexpr int packed_bytes = (APK ? a_raw : 0) + (BPK ? b_raw : 0);
    static constexpr int USTAGES = packed ? (NB == 1 ? 4 : 3) : 0;
    static constexpr int a_unp = APK ? MBS * BM * BK : 0;
    static constexpr int b_unp = BPK ? NBS * (BN / 2) * BK : 0;
    static constexpr int unp_stage = a_unp + b_unp;
    static constexpr int unp_off = STAGES * raw_stage;
    // epilogue staging: per epilogue warp 2 buffers of a 32 x 32 output block
    // (the box of a TMA tensor store); EPIB = bytes of one block, 0 = direct stores
    static constexpr int epi_off = unp_off + USTAGES * unp_stage;
    static constexpr int bar_off = epi_off + 4 * 2 * EPIB;
    static constexpr int n_bars = 3 * STAGES + 2 * USTAGES + 4;
    static constexpr int total = bar_off + n_bars * 8 + 16 + 1024;
    static constexpr int unpack_warps = packed ? 8 : 0;
    // epilogue warp groups (4 warps each): NB = 2 drains its single accumulator
    // after the main loop with the unpack warps (or 4 spare warps) joining in
    // (4-byte outputs keep one group and the staged TMA-store epilogue instead)
    // (3 groups: 512 threads keep 128 registers per thread; a 4th group of spare
    // warps for int8 operands spilled the 16-bit drain at 640 threads)
    static constexpr int epi_groups = (NBS * MBS == 2 && EPIB != 32 * 32 * 4) ? 3 : 1;
    // spare warps (after the unpack warps, if any) that only run epilogue groups
    static constexpr int spare_warps = (epi_groups - 1) * 4 - (packed && epi_groups > 1 ? unpack_warps : 0);
    static constexpr int threads = 256 + 32 * (unpack_warps + spare_warps);
    static constexpr int tmem_cols = NACC == 2 ? 2 * BN : NBS * MBS * BN;
    // Arrivals freeing a raw stage in each CTA: the leader's multicast MMA
    // commit when an operand is read straight from the raw stage, plus one per
    // local unpack warp that reads it.
    static constexpr int team_warps = unpack_warps / 2;  // alternate k-blocks, as in Layout
    static constexpr int raw_release = (direct_bytes > 0 ? 1 : 0) + (packed_bytes > 0 ? team_warps : 0);
    static_assert(tmem_cols <= 512, "TMEM budget");
};

// Staged TMA-store epilogue for 4-byte outputs (f32 at 2048x4096: 97 -> 71 us);
// 2-byte outputs keep direct 16-byte stores (measured faster: 60 vs 66 us),
// f64 keeps direct stores (the staging would not fit next to the rings).
template <int OUT>
constexpr int epi_block_bytes() {
    return (OUT == FQG_F32 || OUT == FQG_I32) ? 32 * 32 * 4 : 0;
}

template <int STAGES, int OUT, int AF, int BF, int NB>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(
    PairLayout<STAGES, AF != F8, BF != F8, NB, epi_block_bytes<OUT>()>::threads, 1)
    k_gemm_i8_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   void* __restrict__ y, int64_t ldy, int m, int n, int num_kb,
                   const double* __restrict__ scale, const void* __restrict__ bias, int bias_dt,
                   int vec_ok, int dbg, const int32_t* __restrict__ rowsum, int sk,
                   int32_t* __restrict__ ws,
                   const __grid_constant__ CUtensorMap tmY, int tma_y, int small_acc) {
    constexpr bool APK = AF != F8, BPK = BF != F8;
    constexpr int EPIB = epi_block_bytes<OUT>();
    using L = PairLayout<STAGES, APK, BPK, NB, EPIB>;
    using OT = typename OutT<OUT>::T;
    constexpr int NACC = L::NACC;
    constexpr int NG = L::epi_groups;
    constexpr int NBS = L::NBS, MBS = L::MBS;
    constexpr int TN = NBS * L::BN;     // tile columns
    constexpr int TM = MBS * 2 * BM;    // tile rows
    const long long t_start = clock64();
    unsigned long long gstart = 0;
    if (dbg) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gstart));
    constexpr int BN = L::BN;
    constexpr int U = L::USTAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    uint64_t* full_mma = reinterpret_cast<uint64_t*>(smem + L::bar_off);  // leader: direct operands
    uint64_t* full_unp = full_mma + STAGES;  // own: packed operands landed
    uint64_t* empty = full_unp + STAGES;     // own: raw stage free
    uint64_t* ufull = empty + STAGES;        // leader: unpacked stage ready (both CTAs)
    uint64_t* uempty = ufull + U;            // own: unpacked stage consumed
    uint64_t* tfull = uempty + U;            // own: accumulator ready
    uint64_t* tempty = tfull + 2;            // leader: accumulator drained (both CTAs)
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);
    __shared__ uint32_t s_fixup;  // split-K: the chunks this CTA claimed

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const int num_m = (m + TM - 1) / TM;
    const int num_n = (n + TN - 1) / TN;
    const int num_tiles = num_m * num_n;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    // Work of this cluster as segments (tile, kb0, kb1, split).
    //  sk == 0: data-parallel, whole tiles round robin (split = -1).
    //  sk >= 2: split-K by sk (small M): cluster cid takes split s = cid % sk of
    //    tile cid / sk. Split s owns the 32-column chunks c = s, s + sk, ...: it
    //    writes the chunks it does not own as raw INT32 partials to its workspace
    //    slot (coalesced [chunk][v][row][4] layout), counts itself in and waits
    //    for the tile's other splits (the grid is at most one CTA per SM, so they
    //    normally run together), then sums their partials of its own chunks into
    //    its accumulator before the epilogue. The wait is bounded (~20 us): a
    //    split whose peers are not resident (SMs held by other work, an SM-
    //    limited context) writes its own chunks too, marks them orphaned and
    //    leaves; the split that arrives last finishes orphaned chunks. Nothing
    //    waits on a CTA that has not arrived. No second kernel, no full planes.
    // Integer partial sums: exact and order-free. Split-K only exists in the
    // NB = 1 instantiation (small M); the 256 x 512 kernel is data-parallel.
    constexpr bool SPLITS = NB == 1;
    static_assert(!SPLITS || NG == 1, "split-K fix-up barrier counts the 4 epilogue warps");
    auto for_each_seg = [&](auto&& f) {
        if (SPLITS && sk >= 2) {
            if (cid < num_tiles * sk) {
                const int tile = cid / sk, sp = cid % sk;
                const int kb0 = sp * num_kb / sk, kb1 = (sp + 1) * num_kb / sk;
                f(tile, kb0, kb1, sp);
            }
        } else {
            for (int tile = cid; tile < num_tiles; tile += ncl) f(tile, 0, num_kb, -1);
        }
    };

    if (threadIdx.x == 0) {
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            ptx::mbar_init(&full_mma[s], 1);
            ptx::mbar_init(&full_unp[s], 1);
            ptx::mbar_init(&empty[s], L::raw_release);
        }
        for (int u = 0; u < U; ++u) {
            ptx::mbar_init(&ufull[u], 2 * L::team_warps);  // one team's warps in both CTAs
            ptx::mbar_init(&uempty[u], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 8 * (L::packed ? 1 : NG));
        }
        ptx::fence_barrier_init();
    }
    if (warp == 1) {
        ptx::tmem_alloc_pair(tmem_holder, L::tmem_cols);
        ptx::tmem_relinquish_pair();
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    // Launched as a programmatic dependent of K1: everything above overlapped
    // K1's tail; A, the row sums and y are touched only after this.
    ptx::griddep_wait();

    // ---------------- epilogue (both CTAs: own 128 rows) ----------------
    // Lane quarter ew of TMEM; group grp of NG takes chunks grp, grp + NG, ...
    // (with one accumulator, NB = 2, the unpack warps / spare warps join after
    // the main loop so the exposed drain is split NG ways).
    // Helpers (grp > 0): with packed operands the unpack warps only reach the
    // epilogue after their whole loop, so they help on the cluster's LAST tile
    // and never arrive on tempty (nothing reuses the accumulator after it);
    // spare warps (int8 operands) help on every tile and arrive.
    constexpr bool HELP_ALL = !L::packed;
    auto run_epilogue = [&](const int ew, const int grp) {
        const double s = OUT == FQG_I32 ? 1.0 : __dmul_rn(scale[0], scale[1]);
        const float s32 = __double2float_rn(s);
        int it = 0, echunk = 0;
        if (EPIB > 0 && tma_y && lane == 0) ptx::tma_prefetch_desc(&tmY);
        for_each_seg([&](int tile, int, int, int split) {
            const bool last = tile + ncl >= num_tiles || (SPLITS && sk != 0);
            const int ng = (HELP_ALL || last) ? NG : 1;  // groups sharing this tile's chunks
            if (grp >= ng) {  // a helper skips this tile (keeps the phase count)
                // Spare warps are idle, so they must observe every tfull phase in
                // order (a parity wait two phases ahead would alias); the unpack
                // warps only get here after all earlier phases completed.
                if (warp >= 8 + L::unpack_warps) ptx::mbar_wait(&tfull[it % NACC], (it / NACC) & 1);
                ++it;
                return;
            }
            const int m_blk = tile % num_m, n_blk = tile / num_m;
            const int acc = it % NACC;
            const uint32_t acc_phase = (it / NACC) & 1;
            const bool plane = SPLITS && split >= 0;  // split-K: this split fixes up through the workspace
            ptx::mbar_wait(&tfull[acc], acc_phase);
            ptx::tc_fence_after();
            unsigned long long ge0 = 0;
            if (dbg && lane == 0 && ew == 0 && grp == 0) {
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ge0));
                atomicAdd(&g_dbg2[blockIdx.x % 296][6], ge0 - gstart);  // tfull reached (ns)
            }
#pragma unroll 1
            for (int sub = 0; sub < MBS; ++sub) {  // 256-row sub-tiles (NB = 3: two)
            const int rloc = rank * BM + ew * 32 + lane;  // row within the 256-row sub-tile
            const int row = m_blk * TM + sub * 2 * BM + rloc;
            const int32_t corr = (BF == FU4 && row < m) ? 8 * rowsum[row] : 0;
            const uint32_t t_row =
                tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN + sub * BN;
            // 2-byte outputs, no bias, full tile: 16-column chunks with the next
            // chunk's TMEM load in flight while this one is converted and stored
            constexpr bool OUT16 = OUT == FQG_F16 || OUT == FQG_BF16;
            if (OUT16 && !plane && bias == nullptr && (vec_ok & 2) && !(dbg & 12) &&
                (n_blk + 1) * TN <= n) {
                // one pipelined stream over the chunks of every sub-tile: chunk cc is
                // sub-tile cc / NCH (whose accumulator columns follow contiguously)
                if (sub > 0) continue;
                const int mode = cvt_mode(small_acc, s32);
                constexpr int NCH = TN / 16;
                constexpr int NCHT = MBS * NCH;
                static_assert(MBS == 1 || TN == BN, "sub-tile accumulators must be contiguous");
                // row-sum corrections of this lane's rows in sub-tiles 0 and 1
                const int32_t corr1 = (MBS > 1 && BF == FU4 && row + 2 * BM < m)
                                          ? 8 * rowsum[row + 2 * BM] : 0;
                uint32_t dsink = 0;  // debug bits 32/64 (drain anatomy experiments)
                auto emit = [&](uint32_t (&rr)[16], int cc) {
                    const int sb = MBS == 1 ? 0 : cc / NCH, c = MBS == 1 ? cc : cc % NCH;
                    const int rs = row + sb * 2 * BM;
                    uint32_t pk[8];
                    if (dbg & 32) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) pk[q] = rr[2 * q] ^ (rr[2 * q + 1] << 1);
                    } else {
                        cvt16_certified<OUT, 16>(rr, sb ? corr1 : corr, s32, s, mode, pk);
                    }
                    if (dbg & 64) {
#pragma unroll
                        for (int q = 0; q < 8; ++q) dsink ^= pk[q];
                    } else if (rs < m) {  // 32 contiguous bytes: one full sector per lane
                        stg256(static_cast<uint16_t*>(y) + static_cast<int64_t>(rs) * ldy +
                                   n_blk * TN + c * 16,
                               pk);
                    }
                };
                uint32_t ra[16], rb[16];
                int c = grp;
                if (c < NCHT) ptx::tmem_ld_32x32b_x16(t_row + c * 16, ra);
                ptx::tmem_wait_ld_r(ra);
#pragma unroll 1
                while (c < NCHT) {
                    const int c1 = c + ng;
                    if (c1 < NCHT) ptx::tmem_ld_32x32b_x16(t_row + c1 * 16, rb);
                    emit(ra, c);
                    ptx::tmem_wait_ld_r(rb);
                    if (c1 >= NCHT) break;
                    const int c2 = c1 + ng;
                    if (c2 < NCHT) ptx::tmem_ld_32x32b_x16(t_row + c2 * 16, ra);
                    emit(rb, c1);
                    ptx::tmem_wait_ld_r(ra);
                    c = c2;
                }
                if ((dbg & 64) && dsink == 0x9E3779B9u) g_sink[lane] = 1.0;
            } else
#pragma unroll 1
            for (int c = grp; c < TN / 32; c += ng) {
                // split-K partials only for lane quarters that hold rows < M (decode-size
                // M: most of the 256-row tile is empty)
                if constexpr (SPLITS)
                    if (plane && m_blk * TM + sub * 2 * BM + rank * BM + ew * 32 >= m) break;
                uint32_t r[32];
                if (!(dbg & 8)) {
                    ptx::tmem_ld_32x32b_x32(t_row + c * 32, r);
                    ptx::tmem_wait_ld();
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) r[e] = static_cast<uint32_t>(c + e);
                }
                if (plane) {  // chunks owned by another split -> slot (512-byte warp stores)
                    if (c % sk == split) continue;
                    int4* slot = reinterpret_cast<int4*>(ws) +
                                 ((static_cast<int64_t>(tile * 2 + rank) * sk + split) * (TN / 32) + c) *
                                     8 * BM + ew * 32 + lane;
#pragma unroll
                    for (int v = 0; v < 8; ++v)
                        slot[v * BM] = make_int4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
                    continue;
                }
                const int col0 = n_blk * TN + c * 32;
                if constexpr (EPIB > 0) {
                    if (tma_y) {  // convert, stage the 32 x 32 block, one TMA tensor store
                        uint8_t* ep = smem + L::epi_off + (ew * 2 + (echunk & 1)) * EPIB;
                        ++echunk;
                        if (lane == 0) ptx::bulk_wait_read_allbut1();
                        __syncwarp();
                        constexpr int ESZ = static_cast<int>(sizeof(OT));
                        uint32_t wv[32 * ESZ / 4];
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            const double bv =
                                bias != nullptr ? load_bias(bias, bias_dt, min(col0 + e, n - 1)) : 0.0;
                            const OT v = convert_out<OUT>(static_cast<int32_t>(r[e]) - corr, s, bv);
                            if constexpr (ESZ == 4) {
                                wv[e] = *reinterpret_cast<const uint32_t*>(&v);
                            } else {
                                const uint32_t h = *reinterpret_cast<const uint16_t*>(&v);
                                wv[e >> 1] = (e & 1) ? (wv[e >> 1] | (h << 16)) : h;
                            }
                        }
                        uint4* dst = reinterpret_cast<uint4*>(ep + lane * 32 * ESZ);
#pragma unroll
                        for (int v = 0; v < 8 * ESZ / 4; ++v)
                            dst[v] = make_uint4(wv[4 * v], wv[4 * v + 1], wv[4 * v + 2], wv[4 * v + 3]);
                        ptx::fence_proxy_async_smem();
                        __syncwarp();
                        if (lane == 0) {
                            ptx::tma_store_2d(&tmY, ep, col0,
                                              m_blk * TM + sub * 2 * BM + rank * BM + ew * 32);
                            ptx::bulk_commit();
                        }
                        continue;
                    }
                }
                if (row < m && col0 < n && !(dbg & 4)) {
                    const int ncols = min(32, n - col0);
                    // debug bit 16: convert, but store into a tiny L2-resident sink
                    const bool sink = (dbg & 16) != 0;
                    store_row_chunk<OUT>(sink ? static_cast<void*>(g_sink) : y,
                                         sink ? static_cast<int64_t>(lane) * 32
                                              : static_cast<int64_t>(row) * ldy + col0,
                                         r, s, bias, bias_dt, col0, ncols, sink || vec_ok != 0,
                                         corr, s32, cvt_mode(small_acc, s32));
                }
            }
            }  // sub-tiles
            if constexpr (SPLITS) if (plane) {
                // count this split in (release: every writer fences, one thread adds).
                // One word per (tile, CTA): arrivals in bits 0-7, chunks orphaned by a
                // split that stopped waiting in bits 8 + c.
                __threadfence();
                asm volatile("bar.sync 1, 128;" ::: "memory");
                unsigned int* const ctl = reinterpret_cast<unsigned int*>(
                                              ws + static_cast<int64_t>(num_tiles) * 2 * sk * BM * TN) +
                                          (tile * 2 + rank);
                if (ew == 0 && lane == 0) {
                    const unsigned int old = atomicAdd(ctl, 1u);
                    const bool last = (old & 0xFFu) == static_cast<unsigned int>(sk - 1);
                    bool all_in = last;
                    // (debug bit 128: never wait, every split but the last orphans)
                    if (!last && !(dbg & 128)) {  // wait for the other splits, at most ~20 us
                        unsigned long long t0, t1;
                        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                        for (;;) {
                            unsigned int v;
                            asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(ctl) : "memory");
                            if ((v & 0xFFu) >= static_cast<unsigned int>(sk)) {
                                all_in = true;
                                break;
                            }
                            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
                            if (t1 - t0 > 20000ull) break;
                        }
                    }
                    if (all_in) __threadfence();  // acquire side for the slot reads below
                    // bit 0: reduce own chunks; bit 1: wrote own chunks, decide after;
                    // bits 8..: orphaned chunks this (last) split must also reduce
                    s_fixup = (all_in ? 1u : 2u) | (last ? (old & 0xFF00u) : 0u);
                }
                asm volatile("bar.sync 1, 128;" ::: "memory");
                uint32_t mode = s_fixup;
                const int rloc = rank * BM + ew * 32 + lane;
                const int row = m_blk * TM + rloc;
                const int32_t corr = (BF == FU4 && row < m) ? 8 * rowsum[row] : 0;
                const uint32_t t_row = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN;
                const int4* const slots = reinterpret_cast<const int4*>(ws) +
                                          static_cast<int64_t>(tile * 2 + rank) * sk * (TN / 32) * 8 * BM +
                                          ew * 32 + lane;
                // accumulator chunk c plus the other splits' partials -> y
                const bool quarter_live = m_blk * TM + rank * BM + ew * 32 < m;  // (MBS = 1)
                auto reduce_chunk = [&](int c) {
                    if (!quarter_live) return;
                    uint32_t r[32];
                    ptx::tmem_ld_32x32b_x32(t_row + c * 32, r);
                    ptx::tmem_wait_ld();
#pragma unroll 1
                    for (int sp = 0; sp < sk; sp += 2) {  // two partials in flight
                        const bool u0 = sp != split, u1 = sp + 1 < sk && sp + 1 != split;
                        const int4* p0 = slots + (static_cast<int64_t>(sp) * (TN / 32) + c) * 8 * BM;
                        const int4* p1 = p0 + (TN / 32) * 8 * BM;
                        int4 a0[8], a1[8];
#pragma unroll
                        for (int v = 0; v < 8; ++v) {
                            a0[v] = u0 ? __ldcg(p0 + v * BM) : make_int4(0, 0, 0, 0);
                            a1[v] = u1 ? __ldcg(p1 + v * BM) : make_int4(0, 0, 0, 0);
                        }
#pragma unroll
                        for (int v = 0; v < 8; ++v) {
                            r[4 * v] += a0[v].x + a1[v].x, r[4 * v + 1] += a0[v].y + a1[v].y;
                            r[4 * v + 2] += a0[v].z + a1[v].z, r[4 * v + 3] += a0[v].w + a1[v].w;
                        }
                    }
                    const int col0 = n_blk * TN + c * 32;
                    if (row < m && col0 < n)
                        store_row_chunk<OUT>(y, static_cast<int64_t>(row) * ldy + col0, r, s, bias,
                                             bias_dt, col0, min(32, n - col0), vec_ok != 0, corr, s32,
                                             cvt_mode(small_acc, s32));
                };
                if (mode & 2u) {  // stopped waiting: own chunks -> slot as well, then orphan them
#pragma unroll 1
                    for (int c = split; quarter_live && c < TN / 32; c += sk) {
                        uint32_t r[32];
                        ptx::tmem_ld_32x32b_x32(t_row + c * 32, r);
                        ptx::tmem_wait_ld();
                        int4* slot = reinterpret_cast<int4*>(ws) +
                                     ((static_cast<int64_t>(tile * 2 + rank) * sk + split) * (TN / 32) + c) *
                                         8 * BM + ew * 32 + lane;
#pragma unroll
                        for (int v = 0; v < 8; ++v)
                            slot[v * BM] = make_int4(r[4 * v], r[4 * v + 1], r[4 * v + 2], r[4 * v + 3]);
                    }
                    __threadfence();
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    if (ew == 0 && lane == 0) {
                        unsigned int own = 0;
                        for (int c = split; c < TN / 32; c += sk) own |= 1u << (8 + c);
                        // if the last split has arrived meanwhile it will not look at
                        // these bits: every partial is in, so reduce them here
                        const unsigned int old = atomicOr(ctl, own);
                        const bool done_in = (old & 0xFFu) >= static_cast<unsigned int>(sk);
                        if (done_in) __threadfence();
                        s_fixup = done_in ? 1u : 0u;
                    }
                    asm volatile("bar.sync 1, 128;" ::: "memory");
                    mode = s_fixup;
                }
                if (mode & 1u) {
#pragma unroll 1
                    for (int c = split; c < TN / 32; c += sk) reduce_chunk(c);
                }
#pragma unroll 1
                for (int c = 0; c < TN / 32; ++c)  // orphans seen at the last arrival
                    if ((mode >> (8 + c)) & 1u) reduce_chunk(c);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0 && (HELP_ALL || grp == 0))
                ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
            if (dbg && lane == 0 && ew == 0 && grp == 0) {
                unsigned long long ge1;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ge1));
                atomicAdd(&g_dbg[blockIdx.x % 296][1], ge1 - ge0);
                atomicAdd(&g_dbg[blockIdx.x % 296][2], 1ull);
                atomicAdd(&g_dbg2[blockIdx.x % 296][7], ge1 - gstart);  // epilogue done (ns)
            }
            ++it;
        });
        if (EPIB > 0 && tma_y && lane == 0) ptx::bulk_wait_all();  // staged output stores
    };

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer (both CTAs) ----------------
        const uint64_t keep = ptx::policy_evict_last();
        int stage = 0;
        uint32_t phase = 0;
        for_each_seg([&](int tile, int kb0, int kb1, int) {
            const int m_blk = tile % num_m, n_blk = tile / num_m;
            const int a_row = m_blk * TM + rank * BM;         // + mb * 2 BM per sub-tile
            const int b_row = n_blk * TN + rank * (BN / 2);  // + nb * BN per block
            for (int kb = kb0; kb < kb1; ++kb) {
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* sa = smem + stage * L::raw_stage;
                uint8_t* sb = sa + L::a_raw;
                const uint32_t lead_full = ptx::mapa(ptx::smem_u32(&full_mma[stage]), 0);
                if constexpr (L::direct_bytes > 0) {
                    if (leader) ptx::mbar_arrive_expect_tx(&full_mma[stage], 2 * L::direct_bytes);
                }
                if constexpr (L::packed_bytes > 0)
                    ptx::mbar_arrive_expect_tx(&full_unp[stage], L::packed_bytes);
#pragma unroll
                for (int mb = 0; mb < MBS; ++mb) {
                    if constexpr (APK)
                        ptx::tma_load_2d_hint(sa + mb * (L::a_raw / MBS), &tmA, &full_unp[stage],
                                              kb * BK / 2, a_row + mb * 2 * BM, keep);
                    else
                        ptx::tma_load_2d_2sm(sa + mb * (L::a_raw / MBS), &tmA, lead_full, kb * BK,
                                             a_row + mb * 2 * BM, keep);
                }
#pragma unroll
                for (int nb = 0; nb < NBS; ++nb) {
                    if constexpr (BPK)
                        ptx::tma_load_2d_hint(sb + nb * (L::b_raw / NBS), &tmB, &full_unp[stage],
                                              kb * BK / 2, b_row + nb * BN, keep);
                    else
                        ptx::tma_load_2d_2sm(sb + nb * (L::b_raw / NBS), &tmB, lead_full, kb * BK,
                                             b_row + nb * BN, keep);
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        });
    } else if (warp == 1 && lane == 0 && leader) {
        // ---------------- MMA issuer (leader CTA) ----------------
        constexpr uint32_t idesc = ptx::idesc_i8(2 * BM, BN, BF == FU4);
        int stage = 0, us = 0;
        uint32_t phase = 0, uphase = 0;
        int it = 0;
        const long long t_mma0 = clock64();
        unsigned long long g0;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
        long long nkb_done = 0;
        for_each_seg([&](int, int kb0, int kb1, int) {
            const int acc = it % NACC;
            const uint32_t acc_phase = (it / NACC) & 1;
            FQG_TWAIT(2, ptx::mbar_wait(&tempty[acc], acc_phase ^ 1));
            ptx::tc_fence_after();
            const uint32_t d_tmem = tmem_base + acc * BN;
            for (int kb = kb0; kb < kb1; ++kb) {
                if constexpr (L::direct_bytes > 0) FQG_TWAIT2(1, ptx::mbar_wait(&full_mma[stage], phase));
                if constexpr (L::packed) FQG_TWAIT2(0, ptx::mbar_wait(&ufull[us], uphase));
                ptx::tc_fence_after();
                const uint32_t raw = ptx::smem_u32(smem + stage * L::raw_stage);
                const uint32_t unp = ptx::smem_u32(smem + L::unp_off + us * L::unp_stage);
                const uint32_t a_addr = APK ? unp : raw;
                const uint32_t b_addr = BPK ? unp + L::a_unp : raw + L::a_raw;
#pragma unroll
                for (int k = 0; k < BK / UK; ++k) {
#pragma unroll
                    for (int mb = 0; mb < MBS; ++mb)
#pragma unroll
                        for (int nb = 0; nb < NBS; ++nb)
                            ptx::mma_i8_pair(d_tmem + (mb * NBS + nb) * BN,
                                             ptx::smem_desc_sw128_kmajor(a_addr + mb * (BM * BK) + k * UK),
                                             ptx::smem_desc_sw128_kmajor(b_addr + nb * ((BN / 2) * BK) + k * UK),
                                             idesc, (kb != kb0 || k != 0) ? 1u : 0u);
                }
                if constexpr (L::direct_bytes > 0) ptx::mma_commit_pair(&empty[stage], 0x3);
                if constexpr (L::packed) {
                    ptx::mma_commit_pair(&uempty[us], 0x3);
                    if (++us == U) {
                        us = 0;
                        uphase ^= 1;
                    }
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            ptx::mma_commit_pair(&tfull[acc], 0x3);
            nkb_done += kb1 - kb0;
            ++it;
        });
        if (dbg) {
            atomicAdd(&g_dbg[blockIdx.x % 296][5], clock64() - t_mma0);
            atomicAdd(&g_dbg[blockIdx.x % 296][6], static_cast<unsigned long long>(nkb_done));
            atomicAdd(&g_dbg[blockIdx.x % 296][7], t_mma0 - t_start);
            unsigned long long g1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
            atomicAdd(&g_dbg[blockIdx.x % 296][4], g1 - g0);  // ns of the MMA loop
        }
    } else if (warp >= 4 && warp < 8) {
        run_epilogue(warp - 4, 0);
    } else if (L::packed && warp >= 8 && warp < 8 + L::unpack_warps) {
        // ---------------- int4 -> int8 unpack warps (both CTAs) ----------------
        const int team = (warp - 8) / (L::team_warps > 0 ? L::team_warps : 1);
        const int utid = threadIdx.x - 256 - 32 * L::team_warps * team, nut = 32 * L::team_warps;
        int stage = 0, us = 0, step = 0;
        uint32_t phase = 0, uphase = 0;
        for_each_seg([&](int, int kb0, int kb1, int) {
            for (int kb = kb0; kb < kb1; ++kb, ++step) {
                if ((step & 1) != team) {
                    if (++us == U) {
                        us = 0;
                        uphase ^= 1;
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                    continue;
                }
                const bool d0 = dbg && utid == 0;
                long long tw0 = d0 ? clock64() : 0;
                ptx::mbar_wait(&full_unp[stage], phase);
                long long tw1 = d0 ? clock64() : 0;
                ptx::mbar_wait(&uempty[us], uphase ^ 1);
                long long tw2 = d0 ? clock64() : 0;
                const uint8_t* raw = smem + stage * L::raw_stage;
                uint8_t* unp = smem + L::unp_off + us * L::unp_stage;
                if constexpr (APK) unpack_tile<AF>(raw, unp, MBS * BM, utid, nut);
                if constexpr (BPK)
                    unpack_tile<BF>(raw + L::a_raw, unp + L::a_unp, NBS * (BN / 2), utid, nut);
                if (d0) {
                    atomicAdd(&g_dbg2[blockIdx.x % 296][2], tw1 - tw0);
                    atomicAdd(&g_dbg2[blockIdx.x % 296][3], tw2 - tw1);
                    atomicAdd(&g_dbg2[blockIdx.x % 296][4], clock64() - tw2);
                    atomicAdd(&g_dbg2[blockIdx.x % 296][5], 1ull);
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&ufull[us]), 0));
                    ptx::mbar_arrive(&empty[stage]);
                }
                if (++us == U) {
                    us = 0;
                    uphase ^= 1;
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        });
        if constexpr (NG > 1) run_epilogue(warp & 3, 1 + (warp - 8) / 4);
    } else if (NG > 1 && warp >= 8) {  // spare warps: epilogue groups only
        run_epilogue(warp & 3, 1 + (warp - 8) / 4);
    }
    if (dbg && lane == 0) {
        unsigned long long ga;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ga));
        const int role = warp < 4 ? warp : (warp < 8 ? 4 : (warp < 8 + L::unpack_warps ? 5 : 6));
        atomicMax(&g_dbg3[blockIdx.x % 296][role], ga - gstart);
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (dbg && threadIdx.x == 32) {
        unsigned long long gs;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gs));
        g_dbg3[blockIdx.x % 296][7] = gs - gstart;
    }
    if (warp == 1) {
        __syncwarp();
        ptx::tc_fence_after();
        ptx::tmem_dealloc_pair(tmem_base, L::tmem_cols);
    }
    if (dbg && threadIdx.x == 32) {
        unsigned long long gend;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gend));
        g_dbg[blockIdx.x % 296][0] = gstart;
        g_dbg[blockIdx.x % 296][3] = gend;
    }
}

// |acc - corr| < 2^22 for every output (the epilogue's one-FADD int -> float):
// K' * max|a| * max|b| from the operand value bounds (the layer passes its qmax).
bool small_acc(const GemmArgs& g) {
    const int64_t qa = g.qmax_a > 0 ? g.qmax_a : (g.a_fmt == FQG_I8 ? 128 : 8);
    const int64_t qb = g.qmax_b > 0 ? g.qmax_b : (g.b_fmt == FQG_I8 ? 128 : 8);
    return g.kp * qa * qb < (int64_t{1} << 22);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw Error(FQG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
    return fn;
}

template <int BN, int STAGES, int OUT, int AF, int BF>
void launch(const GemmArgs& g, cudaStream_t stream) {
    constexpr bool APK = AF != F8, BPK = BF != F8;
    using L = Layout<BN, STAGES, APK, BPK>;
    static_assert(L::total <= 227 * 1024, "shared memory budget");
    CUtensorMap ta, tb;
    // Logical K extent in bytes: the TMA zero-fills K' .. ceil(K', 128).
    make_tmap_2d_u8(&ta, g.a, static_cast<uint64_t>(APK ? g.kp / 2 : g.kp),
                    static_cast<uint64_t>(g.m), static_cast<uint64_t>(g.lda), APK ? BK / 2 : BK,
                    BM, APK ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B);
    make_tmap_2d_u8(&tb, g.b, static_cast<uint64_t>(BPK ? g.kp / 2 : g.kp),
                    static_cast<uint64_t>(g.n), static_cast<uint64_t>(g.ldb), BPK ? BK / 2 : BK,
                    BN, BPK ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B);
    auto kern = k_gemm_i8<BN, STAGES, OUT, AF, BF>;
    ensure_smem_attr<k_gemm_i8<BN, STAGES, OUT, AF, BF>>(L::total);
    int dev = 0;
    FQG_CUDA(cudaGetDevice(&dev));
    const int num_tiles = static_cast<int>(((g.m + BM - 1) / BM) * ((g.n + BN - 1) / BN));
    const int grid = std::max(1, std::min(num_tiles, num_sms(dev)));
    const int esz = dtype_size(g.y_dtype);
    const bool vec = (reinterpret_cast<uintptr_t>(g.y) % 16 == 0) && ((g.ldy * esz) % 16 == 0);
    const int num_kb = static_cast<int>((g.kp + BK - 1) / BK);
    kern<<<grid, L::threads, L::total, stream>>>(ta, tb, g.y, g.ldy, static_cast<int>(g.m),
                                                 static_cast<int>(g.n), num_kb, g.scale, g.bias,
                                                 g.bias_dtype, vec ? 1 : 0, g.rowsum,
                                                 small_acc(g) ? 1 : 0);
    FQG_CUDA(cudaGetLastError());
}

template <int STAGES, int OUT, int AF, int BF, int NB>
void launch_pair(const GemmArgs& g, const GemmPlan& p, cudaStream_t stream) {
    constexpr bool APK = AF != F8, BPK = BF != F8;
    using L = PairLayout<STAGES, APK, BPK, NB, epi_block_bytes<OUT>()>;
    static_assert(L::total <= 227 * 1024, "shared memory budget");
    CUtensorMap ta, tb;
    make_tmap_2d_u8(&ta, g.a, static_cast<uint64_t>(APK ? g.kp / 2 : g.kp),
                    static_cast<uint64_t>(g.m), static_cast<uint64_t>(g.lda), APK ? BK / 2 : BK,
                    BM, APK ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B);
    make_tmap_2d_u8(&tb, g.b, static_cast<uint64_t>(BPK ? g.kp / 2 : g.kp),
                    static_cast<uint64_t>(g.n), static_cast<uint64_t>(g.ldb), BPK ? BK / 2 : BK,
                    L::BN / 2, BPK ? CU_TENSOR_MAP_SWIZZLE_NONE : CU_TENSOR_MAP_SWIZZLE_128B);
    auto kern = k_gemm_i8_pair<STAGES, OUT, AF, BF, NB>;
    ensure_smem_attr<k_gemm_i8_pair<STAGES, OUT, AF, BF, NB>>(L::total);
    int dev = 0;
    FQG_CUDA(cudaGetDevice(&dev));
    const int esz = dtype_size(g.y_dtype);
    const bool vec = (reinterpret_cast<uintptr_t>(g.y) % 16 == 0) && ((g.ldy * esz) % 16 == 0);
    // 32-byte row stores (st.global.v8) of the 16-column drain need 32-byte rows
    const bool vec32 = (reinterpret_cast<uintptr_t>(g.y) % 32 == 0) && ((g.ldy * esz) % 32 == 0);
    const int num_kb = static_cast<int>((g.kp + BK - 1) / BK);
    static const int dbg = [] {
        const char* e = std::getenv("FQG_GEMM_DEBUG");
        return e ? std::atoi(e) : 0;
    }();
    if (dbg) {
        static unsigned long long zeros[296][8] = {};
        FQG_CUDA(cudaMemcpyToSymbol(g_dbg, zeros, sizeof(zeros)));
        FQG_CUDA(cudaMemcpyToSymbol(g_dbg3, zeros, sizeof(zeros)));
        FQG_CUDA(cudaMemcpyToSymbol(g_dbg2, zeros, sizeof(zeros)));
    }
    const int sk = p.splits;  // 0, or >= 2 split-K ways (plan_gemm)
    const int nclusters = p.ctas / 2;
    int32_t* ws = nullptr;
    if (sk >= 2) {  // per (tile, CTA): sk slots of 128 x tile_n INT32, then the counters
        const int64_t tiles = ((g.m + L::MBS * 2 * BM - 1) / (L::MBS * 2 * BM)) *
                              ((g.n + L::NBS * L::BN - 1) / (L::NBS * L::BN));
        const size_t slot_bytes = static_cast<size_t>(tiles) * 2 * sk * BM * L::NBS * L::BN * 4;
        static_assert(NB != 1 || L::NBS * L::BN / 32 <= 8, "split-K control word: 8 chunk bits");
        const size_t ctl_bytes = static_cast<size_t>(tiles) * 2 * 4;
        FQG_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), slot_bytes + ctl_bytes, stream));
        FQG_CUDA(cudaMemsetAsync(reinterpret_cast<uint8_t*>(ws) + slot_bytes, 0, ctl_bytes, stream));
    }
    CUtensorMap ty;
    std::memset(&ty, 0, sizeof(ty));
    const bool tma_y = epi_block_bytes<OUT>() > 0 && vec && sk < 2 && L::epi_groups == 1;
    if (tma_y) {
        const CUtensorMapDataType dt =
            esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT16;
        const cuuint64_t dims[2] = {static_cast<cuuint64_t>(g.n), static_cast<cuuint64_t>(g.m)};
        const cuuint64_t strides[1] = {static_cast<cuuint64_t>(g.ldy * esz)};
        const cuuint32_t box[2] = {32, 32};
        const cuuint32_t estr[2] = {1, 1};
        const CUresult r = encode_fn()(&ty, dt, 2, g.y, dims, strides, box, estr,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                       CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            throw Error(FQG_ERR_CUDA, "cuTensorMapEncodeTiled (y) failed (" + std::to_string(r) + ")");
    }
    static const bool pdl = [] {
        const char* e = std::getenv("FQG_PDL");
        return !(e && std::atoi(e) == 0);
    }();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * nclusters);
    cfg.blockDim = dim3(L::threads);
    cfg.dynamicSmemBytes = L::total;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaError_t le = cudaLaunchKernelEx(
        &cfg, kern, ta, tb, g.y, g.ldy, static_cast<int>(g.m), static_cast<int>(g.n), num_kb,
        g.scale, g.bias, g.bias_dtype, (vec ? 1 : 0) | (vec32 ? 2 : 0), dbg, g.rowsum, sk, ws, ty,
        tma_y ? 1 : 0,
        small_acc(g) ? 1 : 0);
    if (le == cudaSuccess) le = cudaGetLastError();
    if (ws) cudaFreeAsync(ws, stream);
    FQG_CUDA(le);
    if (dbg) {
        unsigned long long h[296][8];
        FQG_CUDA(cudaDeviceSynchronize());
        FQG_CUDA(cudaMemcpyFromSymbol(h, g_dbg, sizeof(h)));
        double acc[8] = {0};
        const int nc = 2 * nclusters;
        for (int c = 0; c < nc; ++c)
            for (int i = 0; i < 8; ++i) acc[i] += static_cast<double>(h[c][i]) / nc;
        // leader-only slots are averaged over both CTAs of a pair: x2
        std::fprintf(stderr,
                     "[fqg gemm pair] per leader: mma loop %.0f cyc for %.0f k-blocks (%.0f "
                     "cyc/kb), start %.0f | mma wait-full %.0f wait-tempty %.0f | producer "
                     "wait-empty %.0f | epi(thread) wait-tfull %.0f\n",
                     acc[5] * 2, acc[6] * 2, acc[6] > 0 ? acc[5] / acc[6] : 0.0, acc[7] * 2,
                     acc[1] * 2, acc[2] * 2, acc[0], acc[3] / 128);
        std::fprintf(stderr, "[fqg gemm pair] SM clock during the MMA loop: %.0f MHz\n",
                     acc[4] > 0 ? acc[5] / acc[4] * 1e3 : 0.0);
        unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
        for (int c = 0; c < nc; ++c) {
            s0 = std::min<unsigned long long>(s0, h[c][0]);
            s1 = std::max<unsigned long long>(s1, h[c][0]);
            e0 = std::min<unsigned long long>(e0, h[c][3]);
            e1 = std::max<unsigned long long>(e1, h[c][3]);
        }
        std::fprintf(stderr,
                     "[fqg gemm pair] CTA start spread %.1f us, end spread %.1f..%.1f us after "
                     "first start; per-leader mma loop %.1f us avg\n",
                     (s1 - s0) * 1e-3, (e0 - s0) * 1e-3, (e1 - s0) * 1e-3, acc[4] * 2e-3);
        for (int c = 0; c < nc; ++c)
            if (h[c][3] - s0 > (e1 - s0) * 0.8 || (c >= 112 && c < 128))
                std::fprintf(stderr,
                             "[fqg gemm pair]   slow CTA %d (cluster %d, rank %d): start %.1f end %.1f us; "
                             "mma loop %llu ns; epi %llu ns over %llu tiles\n",
                             c, c / 2, c % 2, (h[c][0] - s0) * 1e-3, (h[c][3] - s0) * 1e-3, h[c][4],
                             h[c][1], h[c][2]);
        std::fprintf(stderr, "[fqg gemm pair] epilogue per tile (warp 0 of 4): %.2f us\n",
                     acc[2] > 0 ? acc[1] / acc[2] * 1e-3 : 0.0);
        unsigned long long h2[296][8];
        FQG_CUDA(cudaMemcpyFromSymbol(h2, g_dbg2, sizeof(h2)));
        double a2[8] = {0};
        for (int c = 0; c < nc; ++c)
            for (int i = 0; i < 8; ++i) a2[i] += static_cast<double>(h2[c][i]) / nc;
        std::fprintf(stderr, "[fqg gemm pair] epilogue: accumulator ready at %.1f us, done at %.1f us (avg per CTA, summed over its tiles)\n",
                     a2[6] * 1e-3, a2[7] * 1e-3);
        {
            unsigned long long h3[296][8];
            FQG_CUDA(cudaMemcpyFromSymbol(h3, g_dbg3, sizeof(h3)));
            double a3[8] = {0}, m3[8] = {0};
            for (int c = 0; c < nc; ++c)
                for (int i = 0; i < 8; ++i) {
                    a3[i] += static_cast<double>(h3[c][i]) / nc;
                    m3[i] = std::max(m3[i], static_cast<double>(h3[c][i]));
                }
            std::fprintf(stderr,
                         "[fqg gemm pair] final-sync arrival avg/max us: producer %.1f/%.1f mma %.1f/%.1f "
                         "w2 %.1f w3 %.1f epi %.1f/%.1f unpack %.1f/%.1f spare %.1f/%.1f | past sync %.1f/%.1f\n",
                         a3[0] * 1e-3, m3[0] * 1e-3, a3[1] * 1e-3, m3[1] * 1e-3, a3[2] * 1e-3,
                         a3[3] * 1e-3, a3[4] * 1e-3, m3[4] * 1e-3, a3[5] * 1e-3, m3[5] * 1e-3,
                         a3[6] * 1e-3, m3[6] * 1e-3, a3[7] * 1e-3, m3[7] * 1e-3);
        }
        std::fprintf(stderr,
                     "[fqg gemm pair] per CTA: mma wait ufull %.0f, wait full_mma %.0f | unpack "
                     "(thread 0): wait full_unp %.0f, wait uempty %.0f, work %.0f cyc over %.0f "
                     "k-blocks\n",
                     a2[0] * 2, a2[1] * 2, a2[2], a2[3], a2[4], a2[5]);
    }
}

// Largest raw-ring depth (<= maxst) that fits the shared-memory budget.
template <bool APK, bool BPK, int NB, int EPIB>
constexpr int fit_stages(int maxst) {
    using L1 = PairLayout<1, APK, BPK, NB, EPIB>;
    const int fixed = L1::USTAGES * L1::unp_stage + 4 * 2 * EPIB + 1024 + 64 * 8 + 16;
    const int st = (227 * 1024 - fixed) / L1::raw_stage;
    return st < maxst ? st : maxst;
}

template <int AF, int BF, int NB, int OUT>
void launch_pair_fit(const GemmArgs& g, const GemmPlan& p, cudaStream_t s) {
    constexpr int ST = fit_stages<AF != F8, BF != F8, NB, epi_block_bytes<OUT>()>(6);
    static_assert(ST >= 2, "pipeline depth");
    launch_pair<ST, OUT, AF, BF, NB>(g, p, s);
}

template <int AF, int BF>
void dispatch_pair(const GemmArgs& g, const GemmPlan& p, cudaStream_t s) {
    auto go = [&](auto nbc) {
        constexpr int NB = decltype(nbc)::value;
        switch (g.y_dtype) {
            case FQG_I32: return launch_pair_fit<AF, BF, NB, FQG_I32>(g, p, s);
            case FQG_F64: return launch_pair_fit<AF, BF, NB, FQG_F64>(g, p, s);
            case FQG_F32: return launch_pair_fit<AF, BF, NB, FQG_F32>(g, p, s);
            case FQG_F16: return launch_pair_fit<AF, BF, NB, FQG_F16>(g, p, s);
            case FQG_BF16: return launch_pair_fit<AF, BF, NB, FQG_BF16>(g, p, s);
            default: throw Error(FQG_ERR_INVALID, "gemm: unsupported output dtype");
        }
    };
    if (p.tile_m == 512) return go(std::integral_constant<int, 3>{});
    if (p.tile_n == 512) return go(std::integral_constant<int, 2>{});
    return go(std::integral_constant<int, 1>{});
}

template <int BN, int AF, int BF>
void dispatch_out(const GemmArgs& g, cudaStream_t s) {
    constexpr int ST = 4;
    switch (g.y_dtype) {
        case FQG_I32: return launch<BN, ST, FQG_I32, AF, BF>(g, s);
        case FQG_F64: return launch<BN, ST, FQG_F64, AF, BF>(g, s);
        case FQG_F32: return launch<BN, ST, FQG_F32, AF, BF>(g, s);
        case FQG_F16: return launch<BN, ST, FQG_F16, AF, BF>(g, s);
        case FQG_BF16: return launch<BN, ST, FQG_BF16, AF, BF>(g, s);
        default: throw Error(FQG_ERR_INVALID, "gemm: unsupported output dtype");
    }
}


constexpr int kfmt(int f) { return f == FQG_I8 ? F8 : (f == FQG_I4 ? FS4 : FU4); }

}  // namespace
}  // namespace fqg
