// tma_stream.cu — how fast can TMA stream the decode-size weight operand?
// One CTA per SM; one thread issues 2-D TMA loads of 128-row x 128-byte boxes
// into a STAGES-deep ring, another releases each stage as soon as it lands (no
// math). Layout 0: the weights row-major [N][K'] (what K4 reads: every box is
// 128 separate 128-byte row segments, K' apart). Layout 1: the same bytes
// k-block-major, every box one contiguous 16 KB block.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_stream tma_stream.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2402_17985_b200/csrc/ptx.cuh"

using namespace fqg;

constexpr int kStages = 12;
constexpr int kBox = 128 * 128;

// Work item i (0 .. nblk * kblk): n-block i / kblk, k-block i % kblk; CTA c takes
// items [c * per, (c + 1) * per) (one n-block's k range in order, as a split-K CTA).
__global__ void __launch_bounds__(64, 1) k_stream(const __grid_constant__ CUtensorMap tm, int layout,
                                                  int nblk, int kblk, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[kStages], empty[kStages];
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        ptx::fence_barrier_init();
    }
    __syncthreads();
    const long long items = static_cast<long long>(nblk) * kblk;
    const long long per = (items + gridDim.x - 1) / gridDim.x;
    const long long i0 = blockIdx.x * per, i1 = min(items, i0 + per);
    if (threadIdx.x == 0) {
        int stage = 0;
        uint32_t phase = 0;
        for (long long i = i0; i < i1; ++i) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            ptx::mbar_arrive_expect_tx(&full[stage], kBox);
            const int nb = static_cast<int>(i / kblk), kb = static_cast<int>(i % kblk);
            // layout 0: coords (k byte, row); layout 1: (byte in block row, row of the
            // [nblk * kblk * 128] x 128 view)
            const int c0 = layout == 0 ? kb * 128 : 0;
            const int c1 = layout == 0 ? nb * 128 : static_cast<int>(i * 128);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
                "[%0], [%1, {%2, %3}], [%4];" ::"r"(ptx::smem_u32(sm + stage * kBox)),
                "l"(reinterpret_cast<uint64_t>(&tm)), "r"(c0), "r"(c1), "r"(ptx::smem_u32(&full[stage]))
                : "memory");
            if (++stage == kStages) stage = 0, phase ^= 1;
        }
    } else if (threadIdx.x == 32) {
        int stage = 0;
        uint32_t phase = 0;
        unsigned long long acc = 0;
        for (long long i = i0; i < i1; ++i) {
            ptx::mbar_wait(&full[stage], phase);
            acc += sm[stage * kBox + (i & 127)];
            ptx::mbar_arrive(&empty[stage]);
            if (++stage == kStages) stage = 0, phase ^= 1;
        }
        if (acc == 0x123456789ull) *sink = acc;
    }
}

// Plain vectorized loads by every thread (grid-stride), for comparison.
__global__ void __launch_bounds__(256) k_ldg(const uint4* __restrict__ w, size_t n16,
                                             unsigned long long* sink) {
    uint32_t acc = 0;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
    for (; i + 3 * stride < n16; i += 4 * stride) {
        const uint4 a = __ldcs(w + i), b = __ldcs(w + i + stride), c = __ldcs(w + i + 2 * stride),
                    d = __ldcs(w + i + 3 * stride);
        acc ^= a.x ^ b.y ^ c.z ^ d.w;
    }
    for (; i < n16; i += stride) acc ^= __ldcs(w + i).x;
    if (acc == 0x12345678u) *sink = acc;
}

int main() {
    const int n = 8192, kp = 14848;
    const int nblk = n / 128, kblk = kp / 128;
    const size_t bytes = static_cast<size_t>(n) * kp;
    uint8_t* w;
    unsigned long long* sink;
    cudaMalloc(&w, bytes);
    cudaMalloc(&sink, 8);
    cudaMemset(w, 1, bytes);
    uint8_t* flush;
    cudaMalloc(&flush, 256 << 20);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = kStages * kBox + 1024;
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    for (int layout = 0; layout < 2; ++layout) {
        CUtensorMap tm;
        const cuuint64_t dims[2] = {layout == 0 ? static_cast<cuuint64_t>(kp) : 128,
                                    layout == 0 ? static_cast<cuuint64_t>(n)
                                                : static_cast<cuuint64_t>(bytes / 128)};
        const cuuint64_t strides[1] = {layout == 0 ? static_cast<cuuint64_t>(kp) : 128};
        const cuuint32_t box[2] = {128, 128}, estr[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, w, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int grid : {sms / 2 * 2 - 20, sms}) {
            float best = 1e9f;
            for (int rep = 0; rep < 6; ++rep) {
                cudaMemset(flush, rep, 256 << 20);
                cudaEvent_t e0, e1;
                cudaEventCreate(&e0);
                cudaEventCreate(&e1);
                cudaEventRecord(e0);
                k_stream<<<grid, 64, smem>>>(tm, layout, nblk, kblk, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep > 0 && ms < best) best = ms;
            }
            std::printf("layout %s, %d CTAs, %d stages: %.1f us, %.0f GB/s\n",
                        layout == 0 ? "row-major [N][K'] (128-byte row segments)"
                                    : "k-block-major (16 KB contiguous boxes)",
                        grid, kStages, best * 1e3, bytes / (best * 1e-3) / 1e9);
        }
    }
    for (int bpsm : {4, 8}) {
        float best = 1e9f;
        for (int rep = 0; rep < 6; ++rep) {
            cudaMemset(flush, rep, 256 << 20);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            k_ldg<<<sms * bpsm, 256>>>(reinterpret_cast<const uint4*>(w), bytes / 16, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep > 0 && ms < best) best = ms;
        }
        std::printf("plain LDG.128 stream, %d CTAs of 256: %.1f us, %.0f GB/s\n", sms * bpsm, best * 1e3,
                    bytes / (best * 1e-3) / 1e9);
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) std::printf("error: %s\n", cudaGetErrorString(e));
    return 0;
}
