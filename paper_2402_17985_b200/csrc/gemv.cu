// gemv.cu — K4 for decode-size M (1 or 2 token rows, int8 weights): the same
// exact INT32 product and epilogue as the tensor-core kernels
// (quantize.cpp:166-198), computed on the CUDA cores with dp4a while the
// weights stream from HBM.
//
// At M <= 2 the layer is bound by the weight stream (M = 1 at 8192 x 14848:
// 122 MB of int8 weights); the 256-row tensor-core tiles spend their time on
// empty rows and on split-K fix-ups instead (49.5 us there, 32.8 us here). Every
// warp owns groups of 4 output columns: lane l reads 16 weight bytes of each
// column per step (512 contiguous bytes per column and warp), the matching
// activation bytes come from L1, and the 4 x 2 INT32 sums are reduced across
// the warp at the end; the epilogue is the exact FP64 one. With dp4a at 4 bytes
// per instruction the stream is issue-bound near 3.7 TB/s, so from 3 rows on (and
// for packed int4 weights, which need unpacking) the tensor-core path is faster.
#include "gemm_kernels.cuh"

namespace fqg {
namespace {

constexpr int kGvRows = 2;   // rows per launch (M <= 2)
constexpr int kGvCols = 4;   // output columns per warp pass
constexpr int kGvThreads = 256;

template <int OUT>
__global__ void __launch_bounds__(kGvThreads) k_gemv_i8(const uint8_t* __restrict__ a, int64_t lda,
                                                       const uint8_t* __restrict__ b, int64_t ldb,
                                                       int m, int n, int kp, void* __restrict__ y,
                                                       int64_t ldy, const double* __restrict__ scale,
                                                       const void* __restrict__ bias, int bias_dt) {
    constexpr int KL = 16;  // k per lane and step (16 weight bytes)
    const int lane = threadIdx.x & 31;
    const double s = OUT == FQG_I32 ? 1.0 : __dmul_rn(scale[0], scale[1]);
    const int steps = (kp + 32 * KL - 1) / (32 * KL);
    // column group g (4 columns) -> CTA g % grid, warp (g / grid) % 8: consecutive
    // groups land on different SMs, so every SM streams the same share
    const int groups = (n + kGvCols - 1) / kGvCols;
    const int wic = threadIdx.x >> 5, wpc = blockDim.x >> 5;
    for (int g = blockIdx.x + static_cast<int>(gridDim.x) * wic; g < groups;
         g += static_cast<int>(gridDim.x) * wpc) {
        const int n0 = g * kGvCols;
        int acc[kGvCols][kGvRows];
#pragma unroll
        for (int c = 0; c < kGvCols; ++c)
#pragma unroll
            for (int r = 0; r < kGvRows; ++r) acc[c][r] = 0;
#pragma unroll 4
        for (int st = 0; st < steps; ++st) {
            // lanes past K' (last step) read k = 0 and contribute zero weights
            const bool kin = (st * 32 + lane) * KL < kp;
            const int k0 = kin ? (st * 32 + lane) * KL : 0;
            uint4 w[kGvCols];
#pragma unroll
            for (int c = 0; c < kGvCols; ++c) {
                const int col = min(n0 + c, n - 1);  // (a repeated column is never stored)
                w[c] = __ldcs(reinterpret_cast<const uint4*>(b + col * ldb + k0));
                if (!kin) w[c] = make_uint4(0u, 0u, 0u, 0u);  // zero bytes add nothing
            }
#pragma unroll
            for (int r = 0; r < kGvRows; ++r) {
                if (r >= m) break;
                const uint4* xr = reinterpret_cast<const uint4*>(a + r * lda + k0);
                const uint4 x0 = __ldg(xr);
                const uint32_t xa[4] = {x0.x, x0.y, x0.z, x0.w};
#pragma unroll
                for (int c = 0; c < kGvCols; ++c) {
                    const uint32_t wv[4] = {w[c].x, w[c].y, w[c].z, w[c].w};
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        acc[c][r] = __dp4a(static_cast<int>(wv[q]), static_cast<int>(xa[q]), acc[c][r]);
                }
            }
        }
        // one 32-lane reduction per (column, row); lane c * kGvRows + r keeps its sum
        int mine = 0;
#pragma unroll
        for (int c = 0; c < kGvCols; ++c)
#pragma unroll
            for (int r = 0; r < kGvRows; ++r) {
                const int v = __reduce_add_sync(0xffffffffu, acc[c][r]);
                if (lane == c * kGvRows + r) mine = v;
            }
        if (lane < kGvCols * kGvRows) {
            const int c = lane / kGvRows, r = lane % kGvRows, col = n0 + c;
            if (r < m && col < n) {
                const double bv = (OUT != FQG_I32 && bias != nullptr) ? load_bias(bias, bias_dt, col) : 0.0;
                store_one<OUT>(y, static_cast<int64_t>(r) * ldy + col, mine, s, bv);
            }
        }
    }
}

void launch_gemv(const GemmArgs& g, const GemmPlan& p, cudaStream_t st) {
    auto go = [&](auto kern) {
        kern<<<static_cast<unsigned>(p.ctas), kGvThreads, 0, st>>>(
            static_cast<const uint8_t*>(g.a), g.lda, static_cast<const uint8_t*>(g.b), g.ldb,
            static_cast<int>(g.m), static_cast<int>(g.n), static_cast<int>(g.kp), g.y, g.ldy, g.scale,
            g.bias, g.bias_dtype);
        FQG_CUDA(cudaGetLastError());
    };
    switch (g.y_dtype) {
        case FQG_I32: return go(k_gemv_i8<FQG_I32>);
        case FQG_F64: return go(k_gemv_i8<FQG_F64>);
        case FQG_F32: return go(k_gemv_i8<FQG_F32>);
        case FQG_F16: return go(k_gemv_i8<FQG_F16>);
        case FQG_BF16: return go(k_gemv_i8<FQG_BF16>);
        default: throw Error(FQG_ERR_INVALID, "gemm: unsupported output dtype");
    }
}

}  // namespace

void gemv_i8(const GemmArgs& g, const GemmPlan& p, cudaStream_t st) {
    require(g.m <= kGvRows && g.a_fmt == FQG_I8 && g.b_fmt == FQG_I8,
            "gemv: M <= 2 rows, int8 activations and weights");
    require(reinterpret_cast<uintptr_t>(g.a) % 16 == 0 && g.lda % 16 == 0 &&
                reinterpret_cast<uintptr_t>(g.b) % 16 == 0 && g.ldb % 16 == 0,
            "gemv: 16-byte aligned operands");
    launch_gemv(g, p, st);
}

}  // namespace fqg
