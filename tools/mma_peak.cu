// mma_peak.cu — raw tcgen05.mma throughput on this B200 (no global memory):
// one CTA per SM issues back-to-back MMAs on smem-resident operands into TMEM.
// Reports TOPS for kind::i8 (128x256x32, and the CTA-pair 256x256x32),
// kind::f8f6f4 e4m3 (128x256x32) and kind::f16 bf16 (128x256x16).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_peak mma_peak.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cudaTypedefs.h>

#include "../paper_2402_17985_b200/csrc/ptx.cuh"

using namespace fqg;

__device__ __forceinline__ void mma_kind(int kind, uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
    if (kind == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(a), "l"(b), "r"(id));
    else if (kind == 1)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(a), "l"(b), "r"(id));
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(a), "l"(b), "r"(id));
}

__global__ void __launch_bounds__(128, 1) k_peak(int iters, int kind, uint32_t idesc) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const bool rnd = kind >= 10;
    kind = kind % 10;
    for (int i = threadIdx.x; i < 48 * 1024 / 16; i += blockDim.x) {
        uint32_t h = (i * 2654435761u) ^ (blockIdx.x * 40503u);
        auto nx = [&]() { h ^= h << 13; h ^= h >> 17; h ^= h << 5; return h; };
        reinterpret_cast<uint4*>(sm)[i] = rnd ? make_uint4(nx(), nx(), nx(), nx()) : make_uint4(0, 0, 0, 0);
    }
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
    }
    if (threadIdx.x < 32) {
        ptx::tmem_alloc(&tbase, 512);
        ptx::tmem_relinquish();
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t a = ptx::smem_u32(sm), b = a + 16 * 1024;
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                mma_kind(kind, tbase + (i & 1) * 256, ptx::smem_desc_sw128_kmajor(a + 32 * k),
                         ptx::smem_desc_sw128_kmajor(b + 32 * k), idesc);
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tbase, 512);
    }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_peak_pair(int iters, uint32_t idesc) {
    __shared__ __align__(1024) uint8_t sm[32 * 1024];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 32 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
    }
    if (threadIdx.x < 32) {
        ptx::tmem_alloc_pair(&tbase, 512);
        ptx::tmem_relinquish_pair();
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    if (threadIdx.x == 0 && ptx::cluster_ctarank() == 0) {
        const uint32_t a = ptx::smem_u32(sm), b = a + 16 * 1024;
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                ptx::mma_i8_pair(tbase + (i & 1) * 256, ptx::smem_desc_sw128_kmajor(a + 32 * k),
                                 ptx::smem_desc_sw128_kmajor(b + 32 * k), idesc, 1);
        ptx::mma_commit_pair(&bar, 0x3);
    }
    if (threadIdx.x == 0) ptx::mbar_wait(&bar, 0);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (threadIdx.x < 32) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_pair(tbase, 512);
    }
}


// MMA peak with concurrent TMA traffic: warp 2 streams `tma_bytes` per
// `mma_per_tma` MMAs into a separate smem buffer (L2-resident source).
__global__ void __launch_bounds__(128, 1)
    k_peak_tma(const __grid_constant__ CUtensorMap tm, int iters, uint32_t idesc, int tma_every) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    uint8_t* tbuf = sm + 48 * 1024;  // 2 x 32 KB TMA landing buffers
    __shared__ uint64_t bar, tbar[2];
    __shared__ uint32_t tbase;
    __shared__ volatile int done;
    for (int i = threadIdx.x; i < 48 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::mbar_init(&tbar[0], 1);
        ptx::mbar_init(&tbar[1], 1);
        done = 0;
        ptx::fence_barrier_init();
    }
    if (threadIdx.x < 32) {
        ptx::tmem_alloc(&tbase, 512);
        ptx::tmem_relinquish();
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t a = ptx::smem_u32(sm), b = a + 16 * 1024;
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                mma_kind(0, tbase + (i & 1) * 256, ptx::smem_desc_sw128_kmajor(a + 32 * k),
                         ptx::smem_desc_sw128_kmajor(b + 32 * k), idesc);
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
        done = 1;
    } else if (threadIdx.x == 64 && tma_every > 0) {
        uint32_t ph[2] = {0, 0};
        int it = 0;
        while (!done) {
            const int buf = it & 1;
            if (it >= 2) { ptx::mbar_wait(&tbar[buf], ph[buf]); ph[buf] ^= 1; }
            ptx::mbar_arrive_expect_tx(&tbar[buf], 32 * 1024);
            ptx::tma_load_2d(tbuf + buf * 32 * 1024, &tm, &tbar[buf], 0, ((blockIdx.x * 7 + it) % 256) * 256);
            ++it;
        }
        for (int b2 = 0; b2 < 2 && b2 < it; ++b2) ptx::mbar_wait(&tbar[(it - 1 - b2) & 1], ph[(it - 1 - b2) & 1]);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tbase, 512);
    }
}


// MMA issue loop shaped like the GEMM main loop: per 128-deep k-block,
// 4 MMAs then tcgen05.commit to the stage's mbarrier; before reusing a stage
// the issuer waits for the commit of STAGES k-blocks ago (the producer's
// empty-barrier wait), and optionally waits on an already-completed "full"
// barrier (try_wait fast path) first.
__global__ void __launch_bounds__(128, 1) k_peak_loop(int iters, uint32_t idesc, int mode) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t empty[4], fullb, bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 48 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) ptx::mbar_init(&empty[i], 1);
        ptx::mbar_init(&fullb, 1);
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
    }
    if (threadIdx.x < 32) {
        ptx::tmem_alloc(&tbase, 512);
        ptx::tmem_relinquish();
    }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (threadIdx.x == 0) {
        ptx::mbar_arrive(&fullb);  // phase 0 complete: waits on parity 0 succeed at once
        const uint32_t a = ptx::smem_u32(sm), b = a + 16 * 1024;
        int stage = 0;
        uint32_t phase = 0;
        for (int i = 0; i < iters; ++i) {
            if (mode >= 1 && i >= 4) ptx::mbar_wait(&empty[stage], phase ^ 1);
            if (mode >= 2) ptx::mbar_wait(&fullb, 0);
            ptx::tc_fence_after();
#pragma unroll
            for (int k = 0; k < 4; ++k)
                mma_kind(0, tbase + (i & 1) * 256, ptx::smem_desc_sw128_kmajor(a + 32 * k),
                         ptx::smem_desc_sw128_kmajor(b + 32 * k), idesc);
            if (mode >= 1) ptx::mma_commit(&empty[stage]);
            if (++stage == 4) { stage = 0; phase ^= 1; }
        }
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tbase, 512);
    }
}


// TMA-only streaming with the GEMM's pattern: per k-block one 128x128 B box
// of A (rows of this CTA's m tile) and 128x128 of B (n half), STAGES-deep
// ring, consumer releases a stage as soon as it lands (no MMA).
template <int STAGES>
__global__ void __launch_bounds__(64, 1)
    k_tma_stream(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                 int num_kb, int tiles) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[STAGES], empty[STAGES];
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 1); }
        ptx::fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int stage = 0; uint32_t phase = 0;
        for (int t = 0; t < tiles; ++t) {
            const int tile = blockIdx.x + t * gridDim.x;
            const int mb = tile % 8, nb = tile / 8;
            for (int kb = 0; kb < num_kb; ++kb) {
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                ptx::mbar_arrive_expect_tx(&full[stage], 32 * 1024);
                ptx::tma_load_2d(sm + stage * 32768, &ta, &full[stage], kb * 128, mb * 256 + (blockIdx.x & 1) * 128);
                ptx::tma_load_2d(sm + stage * 32768 + 16384, &tb, &full[stage], kb * 128, (nb % 16) * 256 + (blockIdx.x & 1) * 128);
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (threadIdx.x == 32) {
        int stage = 0; uint32_t phase = 0;
        for (int t = 0; t < tiles; ++t)
            for (int kb = 0; kb < num_kb; ++kb) {
                ptx::mbar_wait(&full[stage], phase);
                ptx::mbar_arrive(&empty[stage]);
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
    }
}


// Full-rate MMA stream (warp 0) concurrent with a full-rate TMA stream (warp 1
// producer, warp 2 consumer) into a separate 5 x 32 KB ring.
__global__ void __launch_bounds__(96, 1)
    k_mma_plus_tma(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                   int iters, int num_kb, int do_mma, int do_tma, unsigned long long* cyc) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    uint8_t* ring = sm + 48 * 1024;
    constexpr int ST = 5;
    __shared__ uint64_t full[ST], empty[ST], bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 48 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (int i = 0; i < ST; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 1); }
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
    }
    if (threadIdx.x < 32) { ptx::tmem_alloc(&tbase, 512); ptx::tmem_relinquish(); }
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const long long t0 = clock64();
    if (threadIdx.x == 0 && do_mma) {
        const uint32_t a = ptx::smem_u32(sm), b = a + 16 * 1024;
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k)
                mma_kind(0, tbase + (i & 1) * 256, ptx::smem_desc_sw128_kmajor(a + 32 * k),
                         ptx::smem_desc_sw128_kmajor(b + 32 * k), ptx::idesc_i8(128, 256));
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
        cyc[blockIdx.x * 2] = clock64() - t0;
    } else if (threadIdx.x == 32 && do_tma) {
        int stage = 0; uint32_t phase = 0;
        const int mb = blockIdx.x % 8;
        for (int kb = 0; kb < num_kb; ++kb) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            ptx::mbar_arrive_expect_tx(&full[stage], 32 * 1024);
            ptx::tma_load_2d(ring + stage * 32768, &ta, &full[stage], (kb % 57) * 128, mb * 256);
            ptx::tma_load_2d(ring + stage * 32768 + 16384, &tb, &full[stage], (kb % 57) * 128, ((blockIdx.x / 8) % 16) * 256);
            if (++stage == ST) { stage = 0; phase ^= 1; }
        }
    } else if (threadIdx.x == 64 && do_tma) {
        int stage = 0; uint32_t phase = 0;
        for (int kb = 0; kb < num_kb; ++kb) {
            ptx::mbar_wait(&full[stage], phase);
            ptx::mbar_arrive(&empty[stage]);
            if (++stage == ST) { stage = 0; phase ^= 1; }
        }
        cyc[blockIdx.x * 2 + 1] = clock64() - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { ptx::tc_fence_after(); ptx::tmem_dealloc(tbase, 512); }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(k_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
    const int iters = 4000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Case {
        const char* name;
        int kind;
        uint32_t idesc;
        double macs;  // per MMA
    } cases[] = {
        {"i8     128x256x32 cta_group::1", 0, ptx::idesc_i8(128, 256), 128.0 * 256 * 32},
        // f8f6f4: c_format F32 (1 << 4), a/b e4m3 (0)
        {"e4m3   128x256x32 cta_group::1", 1, (1u << 4) | ((256u >> 3) << 17) | ((128u >> 4) << 24),
         128.0 * 256 * 32},
        // f16 kind: c F32, a/b BF16 (1)
        {"bf16   128x256x16 cta_group::1", 2,
         (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24),
         128.0 * 256 * 16},
    };
    for (int kk : {0, 10}) {
        for (int its : {4000, 40000}) {
            k_peak<<<sms, 128, 50 * 1024>>>(200, kk, ptx::idesc_i8(128, 256));
            cudaEventRecord(e0);
            k_peak<<<sms, 128, 50 * 1024>>>(its, kk, ptx::idesc_i8(128, 256));
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = 2.0 * 128.0 * 256 * 32 * 4.0 * its * sms;
            printf("i8 128x256x32 %s data, %d iters: %8.1f TOPS (%.3f ms)\n", kk ? "random" : "zero  ",
                   its, ops / (ms * 1e-3) / 1e12, ms);
        }
    }
    return 0;
    for (int rep = 0; rep < 2; ++rep) {
        for (auto& c : cases) {
            k_peak<<<sms, 128, 50 * 1024>>>(200, c.kind, c.idesc);
            cudaEventRecord(e0);
            k_peak<<<sms, 128, 50 * 1024>>>(iters, c.kind, c.idesc);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = 2.0 * c.macs * 4.0 * iters * sms;
            printf("%s: %8.1f TOPS  (%.3f ms, %s)\n", c.name, ops / (ms * 1e-3) / 1e12, ms,
                   cudaGetErrorString(cudaGetLastError()));
        }
        k_peak_pair<<<sms, 128>>>(200, ptx::idesc_i8(256, 256));
        cudaEventRecord(e0);
        k_peak_pair<<<sms, 128>>>(iters, ptx::idesc_i8(256, 256));
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 2.0 * 256.0 * 256 * 32 * 4.0 * iters * (sms / 2);
        printf("i8     256x256x32 cta_group::2: %8.1f TOPS  (%.3f ms, %s)\n",
               ops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
    }

    {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        void* g = nullptr;
        cudaMalloc(&g, 256ull * 256 * 128);  // 8 MB: 65536 rows x 128 B
        cudaMemset(g, 0, 256ull * 256 * 128);
        CUtensorMap tm;
        const cuuint64_t dims[2] = {128, 65536};
        const cuuint64_t strides[1] = {128};
        const cuuint32_t box[2] = {128, 256};
        const cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, g, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        cudaFuncSetAttribute(k_peak_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
        for (int te : {0, 1}) {
            k_peak_tma<<<sms, 128, 120 * 1024>>>(tm, 200, ptx::idesc_i8(128, 256), te);
            cudaEventRecord(e0);
            k_peak_tma<<<sms, 128, 120 * 1024>>>(tm, iters, ptx::idesc_i8(128, 256), te);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = 2.0 * 128.0 * 256 * 32 * 4.0 * iters * sms;
            printf("i8 128x256x32 with%s TMA stream: %8.1f TOPS (%.3f ms, %s)\n", te ? "" : "out",
                   ops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
        }
    }

    cudaFuncSetAttribute(k_peak_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
    for (int mode : {0, 1, 2}) {
        k_peak_loop<<<sms, 128, 50 * 1024>>>(200, ptx::idesc_i8(128, 256), mode);
        cudaEventRecord(e0);
        k_peak_loop<<<sms, 128, 50 * 1024>>>(iters, ptx::idesc_i8(128, 256), mode);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double ops = 2.0 * 128.0 * 256 * 32 * 4.0 * iters * sms;
        printf("i8 128x256x32 loop mode %d (%s): %8.1f TOPS (%.3f ms, %s)\n", mode,
               mode == 0 ? "no barriers" : mode == 1 ? "commit+wait(stage-4)" : "+wait(full)",
               ops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
    }

    {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        const uint64_t K = 7296;
        void *ga = nullptr, *gb = nullptr;
        cudaMalloc(&ga, 2048 * K);
        cudaMalloc(&gb, 4096 * K);
        cudaMemset(ga, 1, 2048 * K);
        cudaMemset(gb, 1, 4096 * K);
        CUtensorMap ta, tb;
        const cuuint64_t da[2] = {K, 2048}, db[2] = {K, 4096};
        const cuuint64_t st[1] = {K};
        const cuuint32_t box[2] = {128, 128};
        const cuuint32_t es[2] = {1, 1};
        enc(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, ga, da, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        enc(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, gb, db, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int nkb = 57, tiles = 2;
        cudaFuncSetAttribute(k_tma_stream<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768 + 1024);
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            k_tma_stream<6><<<sms, 64, 6 * 32768 + 1024>>>(ta, tb, nkb, tiles);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double bytes = 32768.0 * nkb * tiles * sms;
            printf("TMA stream 6x32KB ring, %d SMs: %.1f us, %.2f TB/s total, %.1f B/clk/SM @1.9GHz (%s)\n",
                   sms, ms * 1e3, bytes / (ms * 1e-3) / 1e12, bytes / sms / (ms * 1e-3) / 1.9e9,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }

    {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
        auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        const uint64_t K = 7296;
        void *ga = nullptr, *gb = nullptr;
        cudaMalloc(&ga, 2048 * K);
        cudaMalloc(&gb, 4096 * K);
        CUtensorMap ta, tb;
        const cuuint64_t da[2] = {K, 2048}, db[2] = {K, 4096};
        const cuuint64_t st[1] = {K};
        const cuuint32_t box[2] = {128, 128};
        const cuuint32_t es[2] = {1, 1};
        enc(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, ga, da, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        enc(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, gb, db, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        unsigned long long* cyc = nullptr;
        cudaMalloc(&cyc, sms * 16);
        const int smem = 48 * 1024 + 5 * 32768 + 1024;
        cudaFuncSetAttribute(k_mma_plus_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        // MMA-only iters ~= 2 tiles x 57 k-blocks; TMA k-blocks: same count
        const int it = 114, nkb = 114;
        for (int mode = 0; mode < 3; ++mode) {
            const int dm = mode != 1, dt = mode != 0;
            k_mma_plus_tma<<<sms, 96, smem>>>(ta, tb, it, nkb, dm, dt, cyc);
            cudaMemset(cyc, 0, sms * 16);
            cudaEventRecord(e0);
            k_mma_plus_tma<<<sms, 96, smem>>>(ta, tb, it, nkb, dm, dt, cyc);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            unsigned long long h[2 * 148] = {0};
            cudaMemcpy(h, cyc, sms * 16, cudaMemcpyDeviceToHost);
            double mm = 0, tt = 0;
            for (int i = 0; i < sms; ++i) { mm += h[2 * i]; tt += h[2 * i + 1]; }
            printf("%s: %.1f us; avg cycles mma %.0f tma %.0f (%s)\n",
                   mode == 0 ? "MMA only  " : mode == 1 ? "TMA only  " : "MMA + TMA ", ms * 1e3,
                   mm / sms, tt / sms, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}