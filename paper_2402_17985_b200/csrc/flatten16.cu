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

// K1 layout: a CTA of kWarps warps forms row teams of TW threads (TW / 32
// warps, synchronised by a named barrier); each team streams its own token
// rows. The CTA shares the per-channel certificate in shared memory; each team
// owns its final operand row (+ a zero byte at column K' for padding copies),
// its int4 packing, a tier-2 queue and a long-run list. x streams straight
// into registers (16-byte loads, the next chunk in flight while the current
// one is computed); finished rows leave by bulk stores. Splitting a row over
// several warps shortens the per-row dependency chain, which (with all rows
// in flight at once) is what bounds this kernel.
constexpr int kWarps = 8;     // warps per CTA
constexpr int kCh = 8;        // 16-byte x loads per thread per chunk (= 8 channel groups)
constexpr int kInline = 6;    // extension runs up to this long are written by their thread
constexpr int kRunCap = 32;   // longer runs are listed and written by the whole team
constexpr int kQCap = 128;    // tier-2 queue entries per team
constexpr int kMaxHot = 128;  // hot channels (layer.cu caps the list)

struct K1Smem {
    uint32_t cj, pj, wsrc, hotm, hotg, tbar, per_team0, fl, pk, queue, runs, hotx, per_team, total;
    uint32_t hotg_bytes;
    int ldf;
};
K1Smem k1_smem(int k, int kp, int c1, bool pack4, int teams) {
    K1Smem w{};
    uint32_t o = 0;
    auto take = [&](uint32_t& at, uint32_t bytes) {
        at = o;
        o = (o + bytes + 15) & ~15u;
    };
    take(w.cj, static_cast<uint32_t>(k) * 4);
    take(w.pj, static_cast<uint32_t>(k) * 2);
    take(w.wsrc, static_cast<uint32_t>(kp - c1) * 4);
    take(w.hotm, kMaxHot * 16);
    w.hotg_bytes = static_cast<uint32_t>((k / 8 + 3) / 4 * 16);
    take(w.hotg, w.hotg_bytes);
    take(w.tbar, 16);
    w.per_team0 = o;
    w.ldf = kp + 16;
    o = 0;
    take(w.fl, static_cast<uint32_t>(w.ldf));
    take(w.pk, pack4 ? static_cast<uint32_t>(kp) / 2 : 0u);
    take(w.queue, kQCap * 8);
    take(w.runs, kRunCap * 16);
    take(w.hotx, kMaxHot * 2);
    w.per_team = o;
    w.total = w.per_team0 + teams * w.per_team;
    return w;
}

struct K16Params {
    const void* x;
    int64_t ldx;
    int m, k, kp, c1, ldf, nhot;
    uint32_t s_cj, s_pj, s_wsrc, s_hotm, s_hotg, s_tbar, hotg_bytes, per_team0, fl, pk, queue, runs,
        hotx, per_team;
    const float* cj;
    const uint16_t* pj;
    const int32_t* hot;   // channels taking the exact path on every row (P_j = 0xFFFF)
    const int32_t* hotm;  // [nhot] {j, cap, off, rs32 bits}
    const int32_t* hotg;  // [k / 8] group hot mask | first hot index << 8
    const int32_t* off;   // [k] plan_x ext_offset
    const int32_t* wsrc;  // [kp - c1] flat column of each plan_w copy (padding -> kp, a zero byte)
    const double* s;
    const double* rs;
    const float* rs32;
    const int32_t* cap;
    SplitConsts sc;       // host-computed (identical IEEE arithmetic)
    uint8_t* q;
    int64_t ldq;
    unsigned long long* sat;
    int32_t* rowsum;
    int dbg;
};

__device__ unsigned long long g_k1dbg[16];

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
}  // FQG_K1_DEBUG: summed phase end times (cycles)

template <int TW>
__device__ __forceinline__ void team_sync(int team) {
    if constexpr (TW == 32)
        __syncwarp();
    else
        asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "n"(TW) : "memory");
}

template <bool F16, bool PACK4, int TW>
__global__ void __launch_bounds__(kWarps * 32, 2) k_flatten16(const __grid_constant__ K16Params p) {
    constexpr int TEAMS = kWarps * 32 / TW;
    const long long t_start = clock64();
    ptx::griddep_launch_dependents();  // K4 may start its prologue (it waits for our stores)
    auto mark = [&](int slot) {
        if (p.dbg && (threadIdx.x % TW) == 0) atomicAdd(&g_k1dbg[slot], clock64() - t_start);
    };
    extern __shared__ __align__(16) uint8_t sm[];
    const int tid = threadIdx.x, lane = tid & 31;
    const int team = tid / TW, tt = tid % TW;
    const float* const scj = reinterpret_cast<const float*>(sm + p.s_cj);
    const uint16_t* const spj = reinterpret_cast<const uint16_t*>(sm + p.s_pj);
    const int4* const swsrc = reinterpret_cast<const int4*>(sm + p.s_wsrc);
    const int4* const shot = reinterpret_cast<const int4*>(sm + p.s_hotm);  // {j, cap, off, rs32}
    const int32_t* const shotg = reinterpret_cast<const int32_t*>(sm + p.s_hotg);
    uint8_t* const base = sm + p.per_team0 + team * p.per_team;
    int8_t* const fl = reinterpret_cast<int8_t*>(base + p.fl);
    uint8_t* const pk = base + p.pk;
    uint2* const queue = reinterpret_cast<uint2*>(base + p.queue);
    uint4* const runs = reinterpret_cast<uint4*>(base + p.runs);
    uint16_t* const hotx = reinterpret_cast<uint16_t*>(base + p.hotx);
    __shared__ int qlen_s[TEAMS], nrun_s[TEAMS], rsum_s[TEAMS];
    int& qlen = qlen_s[team];
    int& nrun = nrun_s[team];
    int& rsum_t = rsum_s[team];

    const int k = p.k, kp = p.kp, c1 = p.c1, ng_all = k >> 3;
    const SplitConsts& sc = p.sc;
    const int full = sc.qT;
    const int worker = blockIdx.x * TEAMS + team, nworkers = gridDim.x * TEAMS;
    const int nch = (ng_all + TW * kCh - 1) / (TW * kCh);  // chunks per row
    const int nrows_w = worker < p.m ? (p.m - 1 - worker) / nworkers + 1 : 0;
    const int nchunks = nrows_w * nch;
    const uint4* x4 = static_cast<const uint4*>(p.x);
    const int64_t ldx4 = p.ldx >> 3;

    auto load_chunk = [&](uint4 (&buf)[kCh], int t) {
        if (t >= nchunks) return;
        const int row = worker + (t / nch) * nworkers, c = t % nch;
        const uint4* src = x4 + static_cast<int64_t>(row) * ldx4;
#pragma unroll
        for (int i = 0; i < kCh; ++i) {
            const int g = (c * kCh + i) * TW + tt;
            if (g < ng_all) buf[i] = __ldg(src + g);
        }
    };

    // the first x chunk is in flight while the tables are staged
    uint4 xa[kCh], xb[kCh];
    load_chunk(xa, 0);

    // stage the per-layer tables (shared by the CTA's teams) with 1-D bulk copies
    uint64_t* tbar = reinterpret_cast<uint64_t*>(sm + p.s_tbar);
    if (tid == 0) {
        ptx::mbar_init(tbar, 1);
        ptx::fence_barrier_init();
        const uint32_t b_cj = static_cast<uint32_t>(k) * 4, b_pj = static_cast<uint32_t>(k) * 2;
        const uint32_t b_ws = static_cast<uint32_t>(kp - c1) * 4;
        const uint32_t b_hm = static_cast<uint32_t>(p.nhot) * 16;
        ptx::mbar_arrive_expect_tx(tbar, b_cj + b_pj + b_ws + b_hm + p.hotg_bytes);
        ptx::bulk_load(sm + p.s_cj, p.cj, b_cj, tbar);
        ptx::bulk_load(sm + p.s_pj, p.pj, b_pj, tbar);
        if (b_ws) ptx::bulk_load(sm + p.s_wsrc, p.wsrc, b_ws, tbar);
        if (b_hm) ptx::bulk_load(sm + p.s_hotm, p.hotm, b_hm, tbar);
        ptx::bulk_load(sm + p.s_hotg, p.hotg, p.hotg_bytes, tbar);
    }
    if (tt == 0) {
        qlen = 0;
        nrun = 0;
        rsum_t = 0;
        fl[kp] = 0;
    }
    __syncthreads();
    ptx::mbar_wait(tbar, 0);
    mark(0);

    unsigned long long sat = 0;
    // Row sum of the final operand, kept incrementally (tier-1 words, tier-2
    // corrections and extension pieces, plan_w copies) instead of a re-read pass.
    const bool want_rs = p.rowsum != nullptr;
    int rs_run = 0;
    // Row start: the team's previous bulk store has read fl / pk; zero the
    // plan_x extension slots [K, C1); fetch the hot channels' x values.
    auto row_begin = [&](int row) {
        rs_run = 0;
        if (tt == 0) ptx::bulk_wait_read_all();
        team_sync<TW>(team);
        const int z0 = (k + 15) & ~15;
        if (z0 != k && tt == 0) *reinterpret_cast<uint2*>(fl + k) = make_uint2(0u, 0u);
        for (int i = tt; i < (c1 - z0) >> 4; i += TW)
            *reinterpret_cast<uint4*>(fl + z0 + 16 * i) = make_uint4(0u, 0u, 0u, 0u);
    };
    // ---- tier 1 on one chunk: one FFMA per element; tier-2 elements are queued ----
    auto tier1 = [&](const uint4 (&buf)[kCh], int c) {
#pragma unroll
        for (int i = 0; i < kCh; ++i) {
            const int g = (c * kCh + i) * TW + tt;
            if (g >= ng_all) break;
            const float4 ca = reinterpret_cast<const float4*>(scj)[2 * g];
            const float4 cb = reinterpret_cast<const float4*>(scj)[2 * g + 1];
            const uint4 pw = reinterpret_cast<const uint4*>(spj)[g];
            const float cc[8] = {ca.x, ca.y, ca.z, ca.w, cb.x, cb.y, cb.z, cb.w};
            const uint32_t pv[4] = {pw.x, pw.y, pw.z, pw.w};
            const uint4 xw = buf[i];
            const uint32_t w[4] = {xw.x, xw.y, xw.z, xw.w};
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
            *reinterpret_cast<uint2*>(fl + 8 * g) = make_uint2(wlo, whi);
            if (want_rs) {
                rs_run = __dp4a(static_cast<int>(wlo), 0x01010101, rs_run);
                rs_run = __dp4a(static_cast<int>(whi), 0x01010101, rs_run);
            }
            if (const uint32_t hg = static_cast<uint32_t>(shotg[g]); (hg & 0xFFu) != 0u) {
                uint32_t hm = hg & 0xFFu;  // hot channels of the group: keep their x for tier 2
                int hi = static_cast<int>(hg >> 8);
                while (hm != 0u) {
                    const int e = __ffs(static_cast<int>(hm)) - 1;
                    hm &= hm - 1u;
                    const uint32_t wd = (e & 4) ? ((e & 2) ? xw.w : xw.z) : ((e & 2) ? xw.y : xw.x);
                    hotx[hi++] = static_cast<uint16_t>(wd >> ((e & 1) << 4));
                }
            }
            const uint32_t all = tw[0] & tw[1] & tw[2] & tw[3] & 0x80008000u;
            if (all != 0x80008000u) {
                uint32_t msk = ((~tw[0] >> 15) & 1u) | ((~tw[0] >> 30) & 2u) |
                               ((~tw[1] >> 13) & 4u) | ((~tw[1] >> 28) & 8u) |
                               ((~tw[2] >> 11) & 16u) | ((~tw[2] >> 26) & 32u) |
                               ((~tw[3] >> 9) & 64u) | ((~tw[3] >> 24) & 128u);
                int slot = atomicAdd(&qlen, __popc(msk));
                while (msk != 0u) {
                    const int e = __ffs(static_cast<int>(msk)) - 1;
                    msk &= msk - 1u;
                    const uint32_t wd = (e & 4) ? ((e & 2) ? xw.w : xw.z) : ((e & 2) ? xw.y : xw.x);
                    if (slot < kQCap)
                        queue[slot] = make_uint2(static_cast<uint32_t>(8 * g + e),
                                                 (wd >> ((e & 1) << 4)) & 0xFFFFu);
                    ++slot;
                }
            }
        }
    };
    auto exact = [&](int j, uint32_t xb, int cap_e, float rs32_j, int& ce, int& qe, int& fv) {
        const float xf = mag_to_f32<F16>(xb & 0x7FFFu) * ((xb & 0x8000u) ? -1.0f : 1.0f);
        const uint64_t res = split_quant_elem(xf, static_cast<double>(xf), p.s + j, p.rs + j,
                                              rs32_j, cap_e, sc);
        ce = static_cast<int>(res & 0xFFFF);
        qe = static_cast<int>(static_cast<int16_t>(res >> 16));
        fv = (res >> 32) & 1 ? -full : full;
        sat += (res >> 33) & 1;
    };
    // Row end: tier 2, extension runs, plan_w copies, pack / sums, bulk store.
    auto row_end = [&](int row) {
        mark(1);
        team_sync<TW>(team);
        const int nq = qlen;
        const bool overflow = nq > kQCap;
        if (overflow) {  // pathological inputs: every non-hot tier-2 element inline
            const uint16_t* xr = static_cast<const uint16_t*>(p.x) + static_cast<int64_t>(row) * p.ldx;
            for (int j = tt; j < k; j += TW) {
                const uint32_t xb = __ldg(xr + j);
                if (spj[j] - (xb & 0x7FFFu) >= 0x8000u) continue;  // tier 1 or hot
                int ce, qe, fv;
                const int cap_e = __ldg(p.cap + j);
                exact(j, xb, cap_e, __ldg(p.rs32 + j), ce, qe, fv);
                const int v0 = ce >= 1 ? fv : qe;
                if (want_rs) rs_run += v0 - fl[j];
                fl[j] = static_cast<int8_t>(v0);
                const int last = ce >= 1 ? min(ce, cap_e - 1) : 0;
                fill_pieces(fl + k + __ldg(p.off + j), last, ce, fv, qe);
                if (want_rs && ce >= 1) rs_run += min(ce - 1, last) * fv + (ce <= last ? qe : 0);
            }
        }
        const int nitems = p.nhot + (overflow ? 0 : nq);
        for (int i = tt; i < nitems; i += TW) {
            int j, cap_e, off_j;
            float rs32_j;
            uint32_t xb;
            if (i < p.nhot) {
                const int4 hm = shot[i];
                j = hm.x, cap_e = hm.y, off_j = hm.z, rs32_j = __int_as_float(hm.w);
                xb = hotx[i];
            } else {
                const uint2 e = queue[i - p.nhot];
                j = static_cast<int>(e.x);
                xb = e.y;
                cap_e = __ldg(p.cap + j), off_j = __ldg(p.off + j), rs32_j = __ldg(p.rs32 + j);
            }
            int ce, qe, fv;
            exact(j, xb, cap_e, rs32_j, ce, qe, fv);
            const int v0 = ce >= 1 ? fv : qe;
            if (want_rs) rs_run += v0 - fl[j];  // tier 1 left its (replaced) byte in slot j
            fl[j] = static_cast<int8_t>(v0);  // slot j = piece 0
            if (ce >= 1) {  // pieces 1 .. E -> the (zeroed) extension slots
                const int last = min(ce, cap_e - 1);
                fill_pieces(fl + k + off_j, last, ce, fv, qe);
                if (want_rs) rs_run += min(ce - 1, last) * fv + (ce <= last ? qe : 0);
            }
        }
        team_sync<TW>(team);
        mark(2);
        if (tt == 0) qlen = 0, nrun = 0;
        mark(3);
        // plan_w copies [C1, K'): byte gathers from the flattened row
#pragma unroll 4
        for (int u = tt; u < ((kp - c1) >> 2); u += TW) {
            const int4 sv = swsrc[u];
            const uint32_t b0 = static_cast<uint8_t>(fl[sv.x]), b1 = static_cast<uint8_t>(fl[sv.y]);
            const uint32_t b2 = static_cast<uint8_t>(fl[sv.z]), b3 = static_cast<uint8_t>(fl[sv.w]);
            const uint32_t wv =
                __byte_perm(__byte_perm(b0, b1, 0x0040), __byte_perm(b2, b3, 0x0040), 0x5410);
            *reinterpret_cast<uint32_t*>(fl + c1 + 4 * u) = wv;
            if (want_rs) rs_run = __dp4a(static_cast<int>(wv), 0x01010101, rs_run);
        }
        if constexpr (PACK4) {  // byte i = q[i] & 15 | q[16 + i] << 4
            team_sync<TW>(team);
            for (int u = tt; u < (kp >> 5); u += TW) {
                const uint4 lo = *reinterpret_cast<const uint4*>(fl + 32 * u);
                const uint4 hi = *reinterpret_cast<const uint4*>(fl + 32 * u + 16);
                *reinterpret_cast<uint4*>(pk + 16 * u) =
                    make_uint4(pack_i4_word(lo.x, hi.x), pack_i4_word(lo.y, hi.y),
                               pack_i4_word(lo.z, hi.z), pack_i4_word(lo.w, hi.w));
            }
        }
        if (want_rs) {
            int rsum = rs_run;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) rsum += __shfl_xor_sync(0xffffffffu, rsum, o);
            if (lane == 0) atomicAdd(&rsum_t, rsum);
        }
        ptx::fence_proxy_async_smem();
        team_sync<TW>(team);
        mark(4);
        if (tt == 0) {
            ptx::bulk_store(p.q + static_cast<int64_t>(row) * p.ldq,
                            PACK4 ? static_cast<const void*>(pk) : static_cast<const void*>(fl),
                            PACK4 ? static_cast<uint32_t>(kp >> 1) : static_cast<uint32_t>(kp));
            ptx::bulk_commit();
            if (p.rowsum != nullptr) {
                p.rowsum[row] = rsum_t;
                rsum_t = 0;  // next use is after this team's next row_begin barrier
            }
        }
    };
    auto step = [&](const uint4 (&buf)[kCh], int t) {
        const int row = worker + (t / nch) * nworkers, c = t % nch;
        if (c == 0) row_begin(row);
        if (c == 0) mark(7);
        tier1(buf, c);
        if (c == nch - 1) row_end(row);
    };

    // software pipeline over this team's chunk stream: chunk t + 1 loads while t computes
    for (int t = 0; t < nchunks; t += 2) {
        load_chunk(xb, t + 1);
        step(xa, t);
        if (t + 1 >= nchunks) break;
        load_chunk(xa, t + 2);
        step(xb, t + 1);
    }
    mark(5);
    if (tt == 0) ptx::bulk_wait_all();
    mark(6);
    if (p.sat != nullptr) {
        sat = warp_sum(sat);
        if (lane == 0 && sat) atomicAdd(p.sat, sat);
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
    if (a.cj == nullptr || a.pj == nullptr || a.wsrc16 == nullptr || a.hotg == nullptr ||
        a.amax != nullptr)
        return false;
    if (a.x_dtype != FQG_BF16 && a.x_dtype != FQG_F16) return false;
    if (a.k % 8 != 0 || a.k >= (1 << 24) || a.ldx % 8 != 0 || a.nhot > kMaxHot ||
        reinterpret_cast<uintptr_t>(a.x) % 16 != 0)
        return false;
    if (reinterpret_cast<uintptr_t>(a.q) % 16 != 0 || a.ldq % 16 != 0) return false;
    constexpr int TW = 32;  // threads per row team
    const K1Smem w = k1_smem(static_cast<int>(a.k), static_cast<int>(a.kp), static_cast<int>(a.c1),
                             a.pack4, kWarps * 32 / TW);
    if (w.total > 220 * 1024) return false;
    K16Params p{};
    p.x = a.x;
    p.ldx = a.ldx;
    p.m = static_cast<int>(a.m);
    p.k = static_cast<int>(a.k);
    p.kp = static_cast<int>(a.kp);
    p.c1 = static_cast<int>(a.c1);
    p.ldf = w.ldf;
    p.nhot = static_cast<int>(a.nhot);
    p.s_cj = w.cj, p.s_pj = w.pj, p.s_wsrc = w.wsrc, p.s_hotm = w.hotm, p.per_team0 = w.per_team0;
    p.s_hotg = w.hotg, p.s_tbar = w.tbar, p.hotg_bytes = w.hotg_bytes;
    p.hotm = a.hotm;
    p.hotg = a.hotg;
    p.fl = w.fl, p.pk = w.pk, p.queue = w.queue, p.runs = w.runs, p.hotx = w.hotx;
    p.per_team = w.per_team;
    p.cj = a.cj;
    p.pj = a.pj;
    p.hot = a.hot;
    p.off = a.off;
    p.wsrc = a.wsrc16;
    p.s = a.s;
    p.rs = a.rs;
    p.rs32 = a.rs32;
    p.cap = a.cap;
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
    static const int dbg = [] {
        const char* e = std::getenv("FQG_K1_DEBUG");
        return e ? std::atoi(e) : 0;
    }();
    p.dbg = dbg;
    if (dbg) {
        static unsigned long long zeros[16] = {};
        FQG_CUDA(cudaMemcpyToSymbol(g_k1dbg, zeros, sizeof(zeros)));
    }
    auto run = [&](auto kern) {
        FQG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(w.total)));
        int occ = 0;
        FQG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kWarps * 32, w.total));
        constexpr int teams = kWarps * 32 / TW;
        const int64_t ctas_needed = (a.m + teams - 1) / teams;
        const int grid = static_cast<int>(
            std::max<int64_t>(1, std::min<int64_t>(ctas_needed, std::max(1, occ) * a.num_sms)));
        kern<<<grid, kWarps * 32, w.total, st>>>(p);
        FQG_CUDA(cudaGetLastError());
        if (dbg) {
            unsigned long long h[16];
            FQG_CUDA(cudaDeviceSynchronize());
            FQG_CUDA(cudaMemcpyFromSymbol(h, g_k1dbg, sizeof(h)));
            const double nt = static_cast<double>(grid) * (kWarps * 32 / TW);  // team leaders
            std::fprintf(stderr,
                         "[fqg k1] avg cycles since start per team: staged %.0f, row_begin done "
                         "%.0f, tier1 done %.0f, tier2 done %.0f, runs done %.0f, copies done %.0f, "
                         "loop end %.0f, stores done %.0f (grid %d)\n",
                         h[0] / nt, h[7] / nt, h[1] / nt, h[2] / nt, h[3] / nt, h[4] / nt,
                         h[5] / nt, h[6] / nt, grid);
        }
    };
    const bool f16 = a.x_dtype == FQG_F16;
    if (f16 && a.pack4)
        run(k_flatten16<true, true, TW>);
    else if (f16)
        run(k_flatten16<true, false, TW>);
    else if (a.pack4)
        run(k_flatten16<false, true, TW>);
    else
        run(k_flatten16<false, false, TW>);
    return true;
}

}  // namespace fqg
