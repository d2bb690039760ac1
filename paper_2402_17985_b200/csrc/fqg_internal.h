// fqg_internal.h — declarations shared by the host launcher code and the
// kernels of libfqg (not part of the public C ABI in include/fqg.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/fqg.h"

namespace fqg {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define FQG_CUDA(expr)                                                                     \
    do {                                                                                   \
        cudaError_t e_ = (expr);                                                           \
        if (e_ != cudaSuccess)                                                             \
            throw ::fqg::Error(FQG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

inline void require(bool ok, const std::string& what) {
    if (!ok) throw Error(FQG_ERR_INVALID, what);
}

inline int dtype_size(int dt) {
    switch (dt) {
        case FQG_F64: return 8;
        case FQG_F32: return 4;
        case FQG_F16: return 2;
        case FQG_BF16: return 2;
        case FQG_I32: return 4;
        case FQG_I8: return 1;
        default: return 0;
    }
}

int num_sms(int device);

// The dynamic shared-memory limit is a per-device function attribute: set it
// once per (kernel, device), not once per process.
template <auto Kern>
void ensure_smem_attr(int bytes) {
    static std::atomic<uint64_t> done{0};
    int dev = 0;
    FQG_CUDA(cudaGetDevice(&dev));
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    FQG_CUDA(cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.fetch_or(bit, std::memory_order_acq_rel);
}

extern thread_local std::string g_last_error;

// Runs f, converting exceptions into fqg_status codes + fqg_last_error().
template <class F>
int guard(F&& f) {
    try {
        f();
        return FQG_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return FQG_ERR_INVALID;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return FQG_ERR_RUNTIME;
    }
}

// Internal operand format: packed int4 with biased nibbles (q + 8), the layer's
// weight storage (gemm.cu); not part of the public ABI.
constexpr int FQG_I4_BIASED = 106;

// ---- K4: tcgen05 kind::i8 GEMM -------------------------------------------
// Y[M, N] = epilogue( A[M, K'] . B[N, K']^T ), A/B K-major int8 or packed int4.
struct GemmArgs {
    const void* a;        // [M][lda] bytes, K-major
    int a_fmt;            // FQG_I8 | FQG_I4 (two nibbles per byte, low = even k)
    int64_t lda;          // row stride in bytes
    const void* b;        // [N][ldb] bytes, K-major
    int b_fmt;
    int64_t ldb;
    int64_t m, n, kp;     // kp = logical K' (elements)
    void* y;
    int y_dtype;          // FQG_F64/F32/F16/BF16 or FQG_I32 (raw accumulators)
    int64_t ldy;          // elements
    const double* scale;  // device: scale[0] = s_x, scale[1] = s_w
    const void* bias;     // device [N] or nullptr
    int bias_dtype;
    int variant = 0;      // 0 auto, 1 single-CTA kernel, 2 CTA-pair kernel
    const int32_t* rowsum = nullptr;  // [M] sum of each A row (FQG_I4_BIASED weights)
    int qmax_a = 0, qmax_b = 0;       // operand value bounds (0: from the format)
};
void gemm_i8(const GemmArgs& g, cudaStream_t stream);

// The launch gemm_i8 makes for a shape (fqg_gemm_plan exposes it).
struct GemmPlan {
    int kernel = 0;           // 1: 1-CTA 128 x tile_n tiles; 2: CTA pair 256 x tile_n;
                              // 3: decode-size M on CUDA cores (gemv.cu)
    int tile_m = 0, tile_n = 0;
    int splits = 0;           // >= 2: split-K with the in-kernel fix-up
    int ctas = 0;             // grid size
};
GemmPlan plan_gemm(int64_t m, int64_t n, int64_t kp, int a_fmt, int b_fmt, int variant, int sms);

// TMA descriptor construction through the driver entry point (no -lcuda).
void make_tmap_2d_u8(CUtensorMap* map, const void* base, uint64_t inner_bytes, uint64_t rows,
                     uint64_t row_stride_bytes, uint32_t box_inner, uint32_t box_rows,
                     CUtensorMapSwizzle swz);

}  // namespace fqg
