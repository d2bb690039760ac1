// api.cu — the C ABI (include/fqg.h): error plumbing, device queries and the
// standalone GEMM entry point. Layer handles live in layer.cu.
#include <cstring>
#include <string>

#include "fqg_internal.h"
#include "host_pool.h"

namespace fqg {

thread_local std::string g_last_error;

int num_sms(int device) {
    static int cache[64] = {0};
    if (device < 0 || device >= 64) device = 0;
    if (cache[device] == 0) {
        int v = 0;
        FQG_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
        // Per-call scratch (K1 operand, GEMM stream-K workspace) comes from the
        // device's default stream-ordered pool: keep freed blocks cached instead
        // of returning them to the OS at every synchronisation (which makes the
        // next cudaMallocAsync a real allocation, tens of microseconds).
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cache[device] = v;
    }
    return cache[device];
}

}  // namespace fqg

using namespace fqg;

extern "C" {

const char* fqg_last_error(void) { return g_last_error.c_str(); }

int fqg_version(void) { return 1; }

int fqg_gemm(const void* a_dev, int a_fmt, int64_t lda, const void* b_dev, int b_fmt, int64_t ldb,
             int64_t m, int64_t n, int64_t kp, void* y_dev, int y_dtype, int64_t ldy,
             const double* scale_dev, const void* bias_dev, int bias_dtype, void* stream) {
    return guard([&] {
        GemmArgs g{a_dev, a_fmt, lda, b_dev, b_fmt, ldb, m, n, kp, y_dev, y_dtype, ldy,
                   scale_dev, bias_dev, bias_dev ? bias_dtype : FQG_NONE};
        require(y_dtype == FQG_I32 || scale_dev != nullptr, "fqg_gemm: scale_dev is required");
        gemm_i8(g, static_cast<cudaStream_t>(stream));
    });
}

uint64_t fqg_hash64(const void* data, size_t bytes, uint64_t seed) {
    // Fixed 1 MiB blocks hashed in parallel, block hashes folded in order: the
    // value does not depend on the thread count.
    constexpr size_t kBlock = size_t{1} << 20;
    const auto* p = static_cast<const uint8_t*>(data);
    auto mix = [](uint64_t h, uint64_t w) {
        h ^= w * 0x9E3779B97F4A7C15ull;
        h = (h << 31) | (h >> 33);
        return h * 0xBF58476D1CE4E5B9ull;
    };
    auto block = [&](size_t b0, size_t b1, uint64_t h) {
        size_t i = b0;
        for (; i + 8 <= b1; i += 8) {
            uint64_t w;
            std::memcpy(&w, p + i, 8);
            h = mix(h, w);
        }
        uint64_t t = 0;
        if (i < b1) std::memcpy(&t, p + i, b1 - i);
        return mix(h, t ^ (static_cast<uint64_t>(b1 - b0) << 56));
    };
    const int nb = static_cast<int>((bytes + kBlock - 1) / kBlock);
    std::vector<uint64_t> hs(static_cast<size_t>(std::max(nb, 1)));
    if (nb <= 1) {
        hs[0] = block(0, bytes, seed);
    } else {
        HostPool::get().parallel_for(nb, [&](int b) {
            const size_t b0 = static_cast<size_t>(b) * kBlock;
            hs[b] = block(b0, std::min(bytes, b0 + kBlock), seed + static_cast<uint64_t>(b));
        });
    }
    uint64_t h = seed ^ static_cast<uint64_t>(bytes);
    for (uint64_t v : hs) h = mix(h, v);
    return h;
}

int fqg_gemm_plan(int64_t m, int64_t n, int64_t kp, int a_fmt, int b_fmt, int y_dtype,
                  fqg_gemm_plan_info* out) {
    return guard([&] {
        require(out != nullptr && m >= 1 && n >= 1 && kp >= 1, "fqg_gemm_plan: bad argument");
        require(dtype_size(y_dtype) > 0 && y_dtype != FQG_I8, "fqg_gemm_plan: bad output dtype");
        int dev = 0;
        FQG_CUDA(cudaGetDevice(&dev));
        const GemmPlan p = plan_gemm(m, n, kp, a_fmt, b_fmt, 0, num_sms(dev));
        *out = {p.kernel, p.tile_m, p.tile_n, p.splits, p.ctas};
    });
}

}  // extern "C"
