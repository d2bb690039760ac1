// mma_ts.cu — tcgen05.mma kind::i8 issue rate with A in TMEM ("ts") vs A in
// SMEM ("ss"), one CTA per SM, operands resident (no memory traffic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_ts mma_ts.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2402_17985_b200/csrc/ptx.cuh"

using namespace fqg;

__global__ void __launch_bounds__(128, 1) k_ts(int iters, uint32_t idesc, int n, int ts) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
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
        const uint32_t a_tmem = tbase + 384;
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (ts)
                    ptx::mma_i8_ts(tbase, a_tmem + 8 * k, ptx::smem_desc_sw128_kmajor(b + 32 * k),
                                   idesc, 1u);
                else
                    ptx::mma_i8(tbase, ptx::smem_desc_sw128_kmajor(a + 32 * k),
                                ptx::smem_desc_sw128_kmajor(b + 32 * k), idesc, 1u);
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

// CTA pair: M = 256 (A from each CTA's TMEM), B N/2 rows per CTA from SMEM,
// cycling over `nst` B stages (16 KB apart) like a TMA ring.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_ts_pair(int iters, uint32_t idesc, int ts, int nst) {
    extern __shared__ __align__(1024) uint8_t dsm[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x)
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
        const uint32_t a = ptx::smem_u32(sm), b0 = a + 16 * 1024;
        const uint32_t a_tmem = tbase + 384;
        for (int i = 0; i < iters; ++i) {
            const uint32_t b = b0 + (i % nst) * 16 * 1024;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (ts)
                    ptx::mma_i8_ts_pair(tbase, a_tmem + 8 * k, ptx::smem_desc_sw128_kmajor(b + 32 * k),
                                        idesc, 1u);
                else
                    ptx::mma_i8_pair(tbase, ptx::smem_desc_sw128_kmajor(a + 32 * k),
                                     ptx::smem_desc_sw128_kmajor(b + 32 * k), idesc, 1u);
            }
        }
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

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(k_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int ts : {0, 1})
        for (int n : {128, 192, 256})
            for (int au : {0, 1}) {
                const uint32_t id = ptx::idesc_i8(128, n, false, au != 0);
                k_ts<<<sms, 128, 70 * 1024>>>(200, id, n, ts);
                cudaEventRecord(e0);
                k_ts<<<sms, 128, 70 * 1024>>>(iters, id, n, ts);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                const double ops = 2.0 * 128.0 * n * 32 * 4.0 * iters * sms;
                printf("i8 %s 128x%dx32 a_%s: %8.1f TOPS (%.3f ms, %s)\n", ts ? "ts" : "ss", n,
                       au ? "u8" : "s8", ops / (ms * 1e-3) / 1e12, ms,
                       cudaGetErrorString(cudaGetLastError()));
            }
    cudaFuncSetAttribute(k_ts_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024);
    for (int ts : {0, 1})
        for (int n : {160, 192, 256})
            for (int nst : {1, 8}) {
                const uint32_t id = ptx::idesc_i8(256, n, false, ts != 0);
                k_ts_pair<<<sms, 128, 180 * 1024>>>(200, id, ts, nst);
                cudaEventRecord(e0);
                k_ts_pair<<<sms, 128, 180 * 1024>>>(iters, id, ts, nst);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                const double ops = 2.0 * 256.0 * n * 32 * 4.0 * iters * (sms / 2);
                printf("i8 pair %s 256x%dx32 B-stages %d: %8.1f TOPS (%.3f ms, %s)\n", ts ? "ts" : "ss",
                       n, nst, ops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}
