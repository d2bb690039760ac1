// flatten16.cu — K1 for 16-bit activations (bf16 / f16) under the static
// activation scale: the same fused divide_columns -> flatten_tensor(saturating)
// -> repeat_columns -> quantize_per_tensor pass as flatten.cu
// (smoothing.cpp:68-79, flatten.cpp:60-102,158-174, quantize.cpp:23-48), with
// the per-element work cut to a handful of instructions by an exhaustive
// per-channel certificate computed once per layer.
//
// Certificate (k_tier1_tables). A 16-bit input has at most 32640 finite
// magnitudes. For channel j the reference maps a magnitude u with
// |RN(u / s_j)| < T_x ("tier 1": no full +-T piece, fmod(a, T) = a) to the
// single slot value q = clamp(round(RN(RN(u / s_j) / s_x)), +-qmax) and zeros in
// every extension slot. The kernel checks, for every u of every channel, that
// the low byte of RN32(u * c_j + 1.5 * 2^23) (one FFMA; the magic constant
// leaves round-to-nearest(u * c_j) as a two's-complement integer in the low
// mantissa bits) equals that q, for five fp32 candidates c_j around
// 1 / (s_j * s_x), and keeps the candidate with the largest verified prefix
// [0, H_j). The sign is symmetric on both sides (RN(-v) = -RN(v)). Elements
// with |x| < H_j (compared as integer bit patterns, two per 32-bit word) take
// the one-FFMA path; every other element (tier 2: full pieces, saturation,
// a certificate gap, inf/NaN) is queued and runs the exact split of
// split.cuh. The result is therefore bit-identical to the reference for
// every input, with no statistical argument.
//
// Data movement (k_flatten16). Persistent CTAs walk blocks of R token rows;
// x rows arrive by 1-D bulk copies (cp.async.bulk, mbarrier completion,
// double-buffered so block b+1 streams in while block b is computed); the
// final operand rows are assembled in shared memory and leave by bulk stores.
// Per block:
//   zero    the plan_x extension slots [K, C1) (16-byte stores);
//   tier 1  every element: slot j = low byte of one FFMA; tier-2 elements
//           (outside the certificate) are queued;
//   tier 2  "hot" channels (calibrated maximum >= 4 T_x, full pieces on most
//           rows) on every row plus the queued elements: the exact split, slot j
//           and its extension pieces (long runs written by the whole warp);
//   copies  plan_w copies [C1, K'): byte gathers from the flattened row;
//   pack    (int4 output) and per-row operand sums (biased int4 GEMM epilogue);
//   store   bulk stores of the finished rows.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <vector>
#include <type_traits>
#include <cstdio>
#include <cstdlib>
#include <cmath>

#include "fqg_internal.h"
#include "kernels.h"
#include "ptx.cuh"
#include "split.cuh"

namespace fqg {
namespace {

using namespace split;

constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
constexpr int kCand = 5;

template <bool F16>
__device__ __forceinline__ float mag_to_f32(uint32_t u) {
    if constexpr (F16)
        return __half2float(__ushort_as_half(static_cast<unsigned short>(u)));
    else
        return __uint_as_float(u << 16);
}

// One CTA per channel: the verified prefix H_j and multiplier c_j.
template <bool F16>
__global__ void __launch_bounds__(256)
    k_tier1_tables(const double* __restrict__ s, int k, double sx, double t, double qmax,
                   float* __restrict__ cj, uint16_t* __restrict__ pj) {
    constexpr uint32_t kEnd = F16 ? 0x7C00u : 0x7F80u;  // first non-finite magnitude
    __shared__ uint32_t red[8][kCand];
    const int j = blockIdx.x;
    const double sj = s[j];
    const float c0 = static_cast<float>(1.0 / (sj * sx));
    float c[kCand];
#pragma unroll
    for (int i = 0; i < kCand; ++i) c[i] = __int_as_float(__float_as_int(c0) + (i - kCand / 2));
    uint32_t h[kCand];
#pragma unroll
    for (int i = 0; i < kCand; ++i) h[i] = kEnd;
    for (uint32_t u = threadIdx.x; u < kEnd; u += blockDim.x) {
        const float xf = mag_to_f32<F16>(u);
        const double v = __ddiv_rn(static_cast<double>(xf), sj);  // smoothing.cpp:75
        if (!(fabs(v) < t)) {  // a full piece exists (flatten.cpp:12-13): tier 2
#pragma unroll
            for (int i = 0; i < kCand; ++i) h[i] = min(h[i], u);
            continue;
        }
        // tier 1: piece = sign * fmod(|v|, T) = v (flatten.cpp:62-72), quantize.cpp:44-45
        double r = round(__ddiv_rn(v, sx));
        r = r < -qmax ? -qmax : (qmax < r ? qmax : r);
        const int qr = static_cast<int>(r);
#pragma unroll
        for (int i = 0; i < kCand; ++i) {
            const uint32_t b = __float_as_uint(__fmaf_rn(xf, c[i], kMagic));
            const int qf = static_cast<int>(static_cast<int8_t>(b & 0xFFu));
            if (qf != qr) h[i] = min(h[i], u);
        }
    }
#pragma unroll
    for (int i = 0; i < kCand; ++i) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) h[i] = min(h[i], __shfl_xor_sync(0xffffffffu, h[i], o));
    }
    if ((threadIdx.x & 31) == 0)
        for (int i = 0; i < kCand; ++i) red[threadIdx.x >> 5][i] = h[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        int best = kCand / 2;
        uint32_t hb = 0;
        for (int i = 0; i < kCand; ++i) {
            uint32_t hi = kEnd;
            for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) hi = min(hi, red[w][i]);
            if (hi > hb || (hi == hb && i == kCand / 2)) {
                hb = hi;
                best = i;
            }
        }
        cj[j] = c[best];
        pj[j] = static_cast<uint16_t>(0x7FFFu + hb);  // tier 1 <=> P - |x| has bit 15 set
    }
}

// Two 16-bit activations of one 32-bit word -> fp32 (exact).
template <bool F16>
__device__ __forceinline__ float2 word_to_f32x2(uint32_t w) {
    if constexpr (F16) {
        __half2 h;
        *reinterpret_cast<uint32_t*>(&h) = w;
        return __half22float2(h);
    } else {
        return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
    }
}

__device__ __forceinline__ uint32_t pack_lowbytes(uint32_t b0, uint32_t b1, uint32_t b2,
                                                  uint32_t b3) {
    return __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
}

__device__ __forceinline__ uint32_t pack_i4_word(uint32_t lo, uint32_t hi) {
    return (lo & 0x0F0F0F0Fu) | ((hi << 4) & 0xF0F0F0F0u);
}

// K1 layout: a CTA of 256 threads owns a block of R token rows (R in {1, 2,
// 4, 8}, chosen from M so that every SM holds several blocks at once). Every
// phase spreads the block's elements over all threads, so no thread carries a
// row's whole dependency chain:
//   1. tier 1   thread t takes channel groups g = t, t + 256, ... (8 channels,
//               one 16-byte x load per row, the R rows' loads in flight
//               together); certificate c_j / P_j loaded once per group and
//               reused for the R rows; slot bytes go to the row buffers in SMEM.
//               Tier-2 elements are queued (warp-aggregated SMEM atomics).
//   2. splits   the "hot" channels (calibrated maximum >= 4 T_x: exact path on
//               every row, from a per-layer list) and the queued elements run
//               the exact split of split.cuh: piece 0 into slot j and the run of
//               extension pieces (count full +-q(T) pieces, then q(rem);
//               flatten.cpp:71-72) into the channel's slots K + off_j ...
//               (the slots [K, C1) are zeroed at block start).
//   3. copies   plan_w copies [C1, K') (repeat_columns, flatten.cpp:158-174):
//               byte gathers from the finished row.
//   4. store    int4 packing in place (packed activations), then one bulk copy
//               per row to HBM.
// The per-row operand sums (biased-int4 GEMM epilogue) are accumulated on the
// way (dp4a of the tier-1 words and copy words, corrections and extension
// pieces of the splits) instead of by a re-read of the rows.
constexpr int kThreads = 256;
constexpr int kMaxHot = 128;  // hot channels (layer.cu caps the list)
constexpr int kListCap = 1024;  // compacted tier-2 elements per block

struct K16Params {
    const void* x;
    int64_t ldx;
    int m, k, kp, c1, ldf, nhot;
    const float* cj;
    const uint16_t* pj;
    const int32_t* hotm;   // [nhot] {j, cap, off, rs32 bits}
    const int32_t* off;    // [k] plan_x ext_offset
    const int32_t* wsrc;   // [kp - c1] flat column of each plan_w copy (padding -> kp, a zero byte)
    const double* s;
    const double* rs;
    const int32_t* cap;
    const float* rs32;
    SplitConsts sc;        // host-computed (identical IEEE arithmetic)
    uint8_t* q;
    int64_t ldq;
    unsigned long long* sat;
    int32_t* rowsum;
    long long* dbg;        // FQG_K1_DEBUG: per block {start, zero, tier1, splits, copies, pack, end}
};

// Extension pieces 1 .. last of one element into d[0 .. last): full pieces
// (value fv) for p < ce, the remainder qe at p == ce (flatten.cpp:71-72);
// word stores for the aligned middle of the full-piece run.
__device__ __forceinline__ void fill_pieces(int8_t* d, int last, int ce, int fv, int qe) {
    const int nfull = min(ce - 1, last);
    const uint32_t word = (static_cast<uint32_t>(fv) & 0xFFu) * 0x01010101u;
    int p = 0;
    for (; p < nfull && (reinterpret_cast<uintptr_t>(d + p) & 3u) != 0u; ++p)
        d[p] = static_cast<int8_t>(fv);
    for (; p + 4 <= nfull; p += 4) *reinterpret_cast<uint32_t*>(d + p) = word;
    for (; p < nfull; ++p) d[p] = static_cast<int8_t>(fv);
    if (ce <= last) d[ce - 1] = static_cast<int8_t>(qe);
}

template <bool F16, bool PACK4, int R>
__global__ void __launch_bounds__(kThreads, R >= 8 ? 2 : 4) k_flatten16(const __grid_constant__ K16Params p) {
    ptx::griddep_launch_dependents();  // K4 may start its prologue (it waits for our stores)
    extern __shared__ __align__(16) uint8_t sm[];
    const int tid = threadIdx.x;
    if (p.dbg && tid == 0) {
        p.dbg[blockIdx.x * 10LL] = clock64();
        unsigned long long g;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
        p.dbg[blockIdx.x * 10LL + 8] = static_cast<long long>(g);
    }
    const int k = p.k, kp = p.kp, c1 = p.c1, ldf = p.ldf;
    const int ngrp = k >> 3;  // channel groups of 8
    const int row0 = blockIdx.x * R;
    const int nrow = min(R, p.m - row0);
    const SplitConsts& sc = p.sc;
    int8_t* const rows = reinterpret_cast<int8_t*>(sm);                     // [R][ldf]
    __shared__ uint32_t list[kListCap];  // compacted tier-2 elements: r << 24 | j
    __shared__ int rsum_s[R];
    __shared__ int qlen;
    if (tid < R) rsum_s[tid] = 0;
    if (tid == 0) qlen = 0;
    {  // zero the plan_x extension slots [K, C1) and the byte at K' (plan_w padding
       // copies read it)
        const int z0 = (k + 15) & ~15;
#pragma unroll
        for (int r = 0; r < R; ++r)
            for (int u = tid; u < ((c1 - z0) >> 4); u += kThreads)
                *reinterpret_cast<uint4*>(rows + r * ldf + z0 + 16 * u) = make_uint4(0u, 0u, 0u, 0u);
        if (tid < R) {
            if (z0 != k) *reinterpret_cast<uint2*>(rows + tid * ldf + k) = make_uint2(0u, 0u);
            rows[tid * ldf + kp] = 0;
        }
    }
    __syncthreads();
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 10LL + 1] = clock64();

    const bool want_rs = p.rowsum != nullptr;
    int rs[R];
#pragma unroll
    for (int r = 0; r < R; ++r) rs[r] = 0;

    unsigned long long sat = 0;
    const uint16_t* x16 = static_cast<const uint16_t*>(p.x);
    // piece 0 into slot j (replacing the tier-1 byte), pieces 1 .. E_j into the
    // channel's extension slots; returns the change of the row sum
    auto split_store = [&](int r, int j, int cap_e, int off_j, float rs32_j) -> int {
        const uint32_t xb = __ldg(x16 + static_cast<int64_t>(row0 + r) * p.ldx + j);
        const float xf = mag_to_f32<F16>(xb & 0x7FFFu) * ((xb & 0x8000u) ? -1.0f : 1.0f);
        const uint64_t res = split_quant_elem(xf, static_cast<double>(xf), p.s + j, p.rs + j,
                                              rs32_j, cap_e, sc);
        const int ce = static_cast<int>(res & 0xFFFF);
        const int qe = static_cast<int>(static_cast<int16_t>(res >> 16));
        const int fv = (res >> 32) & 1 ? -sc.qT : sc.qT;
        sat += (res >> 33) & 1;
        const int v0 = ce >= 1 ? fv : qe;
        int8_t* fr = rows + r * ldf;
        int d = v0 - fr[j];
        fr[j] = static_cast<int8_t>(v0);
        if (ce >= 1 && cap_e > 1) {
            const int last = min(ce, cap_e - 1);
            fill_pieces(fr + k + off_j, last, ce, fv, qe);
            d += min(ce - 1, last) * fv + (ce <= last ? qe : 0);
        }
        return d;
    };
    // ---- 1. tier 1: one FFMA per element; tier-2 elements are queued ----
    // the block's rows as 32-bit offsets from its first row (rows past M read row
    // M - 1 and are never stored)
    const uint4* const xr0 = static_cast<const uint4*>(p.x) + static_cast<int64_t>(row0) * (p.ldx >> 3);
    uint32_t xoff[R];
#pragma unroll
    for (int r = 0; r < R; ++r)
        xoff[r] = static_cast<uint32_t>((min(row0 + r, p.m - 1) - row0) * (p.ldx >> 3));
    const float4* const cj4 = reinterpret_cast<const float4*>(p.cj);
    const uint4* const pj4 = reinterpret_cast<const uint4*>(p.pj);
    for (int g = tid; g < ngrp; g += kThreads) {
        uint4 xw[R];
#pragma unroll
        for (int r = 0; r < R; ++r) xw[r] = __ldg(xr0 + xoff[r] + g);
        const float4 ca = __ldg(cj4 + 2 * g);
        const float4 cb = __ldg(cj4 + 2 * g + 1);
        const uint4 pw = __ldg(pj4 + g);
        const float cc[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
        const uint32_t pv[4] = {pw.x, pw.y, pw.z, pw.w};
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t w[4] = {xw[r].x, xw[r].y, xw[r].z, xw[r].w};
            uint32_t tw[4], bq[8];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                tw[e] = pv[e] - (w[e] & 0x7FFF7FFFu);
                const float2 f = word_to_f32x2<F16>(w[e]);
                bq[2 * e] = __float_as_uint(__fmaf_rn(f.x, cc[2 * e], kMagic));
                bq[2 * e + 1] = __float_as_uint(__fmaf_rn(f.y, cc[2 * e + 1], kMagic));
            }
            const uint32_t wlo = pack_lowbytes(bq[0], bq[1], bq[2], bq[3]);
            const uint32_t whi = pack_lowbytes(bq[4], bq[5], bq[6], bq[7]);
            *reinterpret_cast<uint2*>(rows + r * ldf + 8 * g) = make_uint2(wlo, whi);
            // row sums unconditionally (two dp4a are cheaper than the branch)
            rs[r] = __dp4a(static_cast<int>(wlo), 0x01010101, rs[r]);
            rs[r] = __dp4a(static_cast<int>(whi), 0x01010101, rs[r]);
            const uint32_t all = tw[0] & tw[1] & tw[2] & tw[3] & 0x80008000u;
            if (all != 0x80008000u && row0 + r < p.m) {  // outside the certificate: tier 2
                uint32_t msk = ((~tw[0] >> 15) & 1u) | ((~tw[0] >> 30) & 2u) |
                               ((~tw[1] >> 13) & 4u) | ((~tw[1] >> 28) & 8u) |
                               ((~tw[2] >> 11) & 16u) | ((~tw[2] >> 26) & 32u) |
                               ((~tw[3] >> 9) & 64u) | ((~tw[3] >> 24) & 128u);
                while (msk != 0u) {  // (the compiler aggregates the SMEM atomics per warp)
                    const int e = __ffs(static_cast<int>(msk)) - 1;
                    msk &= msk - 1u;
                    const int j = 8 * g + e;
                    const int slot = atomicAdd(&qlen, 1);
                    if (slot < kListCap)
                        list[slot] = static_cast<uint32_t>(r << 24 | j);
                    else  // pathological input: run it here (this thread owns the group's bytes)
                        rs[r] += split_store(r, j, __ldg(p.cap + j), __ldg(p.off + j),
                                             __ldg(p.rs32 + j));
                }
            }
        }
    }
    __syncthreads();
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 10LL + 2] = clock64();

    // ---- 2. exact splits: hot channels on every row, then the queued elements ----
    const int nhot_items = nrow * p.nhot;
    const int nlist = min(qlen, kListCap);
    for (int i = tid; i < nhot_items + nlist; i += kThreads) {
        int r, j, cap_e, off_j;
        float rs32_j;
        if (i < nhot_items) {
            r = i / p.nhot;
            const int4 hm = __ldg(reinterpret_cast<const int4*>(p.hotm) + (i - r * p.nhot));
            j = hm.x, cap_e = hm.y, off_j = hm.z, rs32_j = __int_as_float(hm.w);
        } else {
            const uint32_t e = list[i - nhot_items];
            r = static_cast<int>(e >> 24), j = static_cast<int>(e & 0xFFFFFFu);
            cap_e = __ldg(p.cap + j), off_j = __ldg(p.off + j), rs32_j = __ldg(p.rs32 + j);
        }
        const int d = split_store(r, j, cap_e, off_j, rs32_j);
#pragma unroll
        for (int rr = 0; rr < R; ++rr) rs[rr] += rr == r ? d : 0;
    }
    __syncthreads();
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 10LL + 3] = clock64();

    // ---- 3. plan_w copies [C1, K') ----
    for (int u = tid; u < ((kp - c1) >> 2); u += kThreads) {
        const int4 sv = __ldg(reinterpret_cast<const int4*>(p.wsrc) + u);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint8_t* fr = reinterpret_cast<const uint8_t*>(rows + r * ldf);
            const uint32_t wv =
                static_cast<uint32_t>(fr[sv.x]) | (static_cast<uint32_t>(fr[sv.y]) << 8) |
                (static_cast<uint32_t>(fr[sv.z]) << 16) | (static_cast<uint32_t>(fr[sv.w]) << 24);
            *reinterpret_cast<uint32_t*>(rows + r * ldf + c1 + 4 * u) = wv;
            if (want_rs) rs[r] = __dp4a(static_cast<int>(wv), 0x01010101, rs[r]);
        }
    }
    if (want_rs) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            int v = rs[r];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if ((tid & 31) == 0 && v != 0) atomicAdd(&rsum_s[r], v);
        }
    }
    __syncthreads();
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 10LL + 4] = clock64();

    // ---- 4. int4 packing in place, then one bulk copy per row ----
    if constexpr (PACK4) {  // byte i = q[i] & 15 | q[16 + i] << 4 per group of 32
        // group u reads bytes [32u, 32u + 32) and writes [16u, 16u + 16): a barrier
        // between the reads and the writes of each pass keeps it race-free
#pragma unroll
        for (int r = 0; r < R; ++r) {
            int8_t* fr = rows + r * ldf;
            for (int u0 = 0; u0 < (kp >> 5); u0 += kThreads) {
                const int u = u0 + tid;
                uint4 o = make_uint4(0u, 0u, 0u, 0u);
                if (u < (kp >> 5)) {
                    const uint4 lo = *reinterpret_cast<const uint4*>(fr + 32 * u);
                    const uint4 hi = *reinterpret_cast<const uint4*>(fr + 32 * u + 16);
                    o = make_uint4(pack_i4_word(lo.x, hi.x), pack_i4_word(lo.y, hi.y),
                                   pack_i4_word(lo.z, hi.z), pack_i4_word(lo.w, hi.w));
                }
                __syncthreads();
                if (u < (kp >> 5)) *reinterpret_cast<uint4*>(fr + 16 * u) = o;
            }
        }
    }
    ptx::fence_proxy_async_smem();  // generic-proxy SMEM writes -> visible to the bulk copies
    __syncthreads();
    if (p.dbg && tid == 0) p.dbg[blockIdx.x * 10LL + 5] = clock64();
    if (tid < nrow) {
        ptx::bulk_store(p.q + static_cast<int64_t>(row0 + tid) * p.ldq, rows + tid * ldf,
                        PACK4 ? static_cast<uint32_t>(kp >> 1) : static_cast<uint32_t>(kp));
        ptx::bulk_commit();
        if (want_rs) p.rowsum[row0 + tid] = rsum_s[tid];
    }
    if (p.sat != nullptr) {
        sat = warp_sum(sat);
        if ((tid & 31) == 0 && sat) atomicAdd(p.sat, sat);
    }
    if (tid < nrow) ptx::bulk_wait_all();
    if (p.dbg && tid == 0) {
        long long* d = p.dbg + static_cast<int64_t>(blockIdx.x) * 10;
        d[6] = clock64();
        unsigned long long g_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
        d[7] = static_cast<long long>(g_end) - d[8];  // ns: the SM clock of the block
        d[9] = static_cast<long long>(g_end);
    }
}

}  // namespace

void tier1_tables(const double* s, int64_t k, double act_scale, double t, double qmax, bool f16,
                  float* cj, uint16_t* pj, cudaStream_t st) {
    auto kern = f16 ? k_tier1_tables<true> : k_tier1_tables<false>;
    kern<<<static_cast<unsigned>(k), 256, 0, st>>>(s, static_cast<int>(k), act_scale, t, qmax, cj,
                                                   pj);
    FQG_CUDA(cudaGetLastError());
}

bool flatten16(const FlattenArgs& a, cudaStream_t st) {
    if (a.cj == nullptr || a.pj == nullptr || a.wsrc16 == nullptr || a.amax != nullptr)
        return false;
    if (a.x_dtype != FQG_BF16 && a.x_dtype != FQG_F16) return false;
    if (a.k % 8 != 0 || a.k >= (1 << 24) || a.ldx % 8 != 0 || a.nhot > kMaxHot ||
        reinterpret_cast<uintptr_t>(a.x) % 16 != 0)
        return false;
    if (reinterpret_cast<uintptr_t>(a.q) % 16 != 0 || a.ldq % 16 != 0) return false;
    // rows per block: the largest of 8/4/2/1 that still gives >= 3 blocks per SM
    int rb = 8;
    while (rb > 1 && (a.m + rb - 1) / rb < 3 * a.num_sms) rb >>= 1;
    static const int rb_env = [] {  // tuning override: FQG_K1_ROWS = 1, 2, 4 or 8
        const char* e = std::getenv("FQG_K1_ROWS");
        return e ? std::atoi(e) : 0;
    }();
    if (rb_env == 1 || rb_env == 2 || rb_env == 4 || rb_env == 8) rb = rb_env;
    const int ldf = static_cast<int>((a.kp + 16 + 15) / 16 * 16);
    auto smem_of = [&](int r) {
        return static_cast<size_t>(r) * ldf;
    };
    while (rb > 1 && smem_of(rb) > 200 * 1024) rb >>= 1;
    const size_t smem = smem_of(rb);
    if (smem > 220 * 1024) return false;
    K16Params p{};
    p.x = a.x;
    p.ldx = a.ldx;
    p.m = static_cast<int>(a.m);
    p.k = static_cast<int>(a.k);
    p.kp = static_cast<int>(a.kp);
    p.c1 = static_cast<int>(a.c1);
    p.ldf = ldf;
    p.nhot = static_cast<int>(a.nhot);
    p.cj = a.cj;
    p.pj = a.pj;
    p.hotm = a.hotm;
    p.off = a.off;
    p.wsrc = a.wsrc16;
    p.s = a.s;
    p.rs = a.rs;
    p.cap = a.cap;
    p.rs32 = a.rs32;
    {  // SplitConsts on the host: the same IEEE double arithmetic as make_consts
        SplitConsts& c = p.sc;
        c.t = a.t;
        c.rt = 1.0 / a.t;
        c.as = a.act_scale;
        c.ras = 1.0 / a.act_scale;
        c.qmax = a.qmax;
        c.rt32 = static_cast<float>(c.rt);
        c.q32 = static_cast<float>(a.t / a.act_scale);
        c.qmax32 = static_cast<float>(a.qmax);
        double qt = std::round(a.t / a.act_scale);  // quantize.cpp:44-45, half away from zero
        qt = qt < -a.qmax ? -a.qmax : (a.qmax < qt ? a.qmax : qt);
        c.qT = static_cast<int>(qt);
    }
    p.q = a.q;
    p.ldq = a.ldq;
    p.sat = a.sat;
    p.rowsum = a.rowsum;
    static const bool k1_dbg = std::getenv("FQG_K1_DEBUG") != nullptr;
    long long* dbg_buf = nullptr;
    const int64_t nblk_dbg = (a.m + rb - 1) / rb;
    if (k1_dbg) {
        FQG_CUDA(cudaMalloc(&dbg_buf, nblk_dbg * 10 * sizeof(long long)));
        p.dbg = dbg_buf;
    }
    const bool f16 = a.x_dtype == FQG_F16;
    const unsigned grid = static_cast<unsigned>((a.m + rb - 1) / rb);
    auto go = [&](auto rc) {
        constexpr int R = decltype(rc)::value;
        auto run = [&](auto kern) {
            kern<<<grid, kThreads, smem, st>>>(p);
            FQG_CUDA(cudaGetLastError());
        };
        if (f16 && a.pack4) {
            ensure_smem_attr<k_flatten16<true, true, R>>(220 * 1024);
            run(k_flatten16<true, true, R>);
        } else if (f16) {
            ensure_smem_attr<k_flatten16<true, false, R>>(220 * 1024);
            run(k_flatten16<true, false, R>);
        } else if (a.pack4) {
            ensure_smem_attr<k_flatten16<false, true, R>>(220 * 1024);
            run(k_flatten16<false, true, R>);
        } else {
            ensure_smem_attr<k_flatten16<false, false, R>>(220 * 1024);
            run(k_flatten16<false, false, R>);
        }
    };
    switch (rb) {
        case 8: go(std::integral_constant<int, 8>{}); break;
        case 4: go(std::integral_constant<int, 4>{}); break;
        case 2: go(std::integral_constant<int, 2>{}); break;
        default: go(std::integral_constant<int, 1>{}); break;
    }
    if (k1_dbg) {  // developer instrumentation: mean cycles per phase, per-SM spread
        std::vector<long long> h(nblk_dbg * 10);
        FQG_CUDA(cudaStreamSynchronize(st));
        FQG_CUDA(cudaMemcpy(h.data(), dbg_buf, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
        cudaFree(dbg_buf);
        double ph[6] = {0};
        for (int64_t b = 0; b < nblk_dbg; ++b)
            for (int i = 0; i < 6; ++i) ph[i] += static_cast<double>(h[b * 10 + i + 1] - h[b * 10 + i]) / nblk_dbg;
        double cyc = 0, ns = 0;
        for (int64_t b = 0; b < nblk_dbg; ++b) {
            cyc += static_cast<double>(h[b * 10 + 6] - h[b * 10]);
            ns += static_cast<double>(h[b * 10 + 7]);
        }
        long long s0 = h[8], s1 = h[8], e1 = h[9];
        int late = 0;
        for (int64_t b = 0; b < nblk_dbg; ++b) {
            s0 = std::min(s0, h[b * 10 + 8]);
            s1 = std::max(s1, h[b * 10 + 8]);
            e1 = std::max(e1, h[b * 10 + 9]);
        }
        for (int64_t b = 0; b < nblk_dbg; ++b) late += h[b * 10 + 8] - s0 > 2000;
        std::fprintf(stderr, "[fqg k1] block starts spread %.1f us (%d blocks start > 2 us late), last end %.1f us\n",
                     (s1 - s0) * 1e-3, late, (e1 - s0) * 1e-3);
        std::fprintf(stderr, "[fqg k1] R=%d blocks=%lld mean cycles: zero %.0f tier1 %.0f splits %.0f copies %.0f pack %.0f store %.0f | block %.1f us at %.0f MHz\n",
                     rb, static_cast<long long>(nblk_dbg), ph[0], ph[1], ph[2], ph[3], ph[4], ph[5],
                     ns / nblk_dbg * 1e-3, ns > 0 ? cyc / ns * 1e3 : 0.0);
    }
    return true;
}

}  // namespace fqg
