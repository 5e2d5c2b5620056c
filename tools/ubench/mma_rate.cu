// Microbenchmark: tcgen05.mma kind::f16 issue/execution rate for one CTA per SM,
// SS vs TS (A in TMEM) and N = 64/128/256, M = 128, cta_group::1.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"
using namespace elm;

template <int N, bool TS>
__global__ void k_rate(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~uintptr_t(1023));
    __shared__ uint32_t tslot;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x / 32;
    if (warp == 0) { ptx::tmem_alloc(&tslot, 512); ptx::tmem_relinquish(); }
    if (threadIdx.x == 0) { ptx::mbar_init(&bar, 1); ptx::fence_mbar_init(); }
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0x3c003c00u;
    ptx::fence_proxy_async_smem();
    ptx::tc_fence_before(); __syncthreads(); ptx::tc_fence_after();
    const uint32_t tmem = tslot;
    if (threadIdx.x == 32) {
        constexpr uint32_t idesc = ptx::idesc_f16(128, N);
        uint64_t da = ptx::desc_sw128_kmajor(ptx::smem_u32(base));
        uint64_t db = ptx::desc_sw128_kmajor(ptx::smem_u32(base + 16384));
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                if (TS) ptx::mma_f16_ts(tmem, tmem + 256 + kk * 8, db + 2 * kk, idesc, 1);
                else ptx::mma_f16_ss(tmem, da + 2 * kk, db + 2 * kk, idesc, 1);
            }
        }
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
    }
    ptx::tc_fence_before(); __syncthreads();
    if (warp == 0) { ptx::tc_fence_after(); ptx::tmem_dealloc(tmem, 512); }
}

template <int N, bool TS>
void run(const char* name) {
    unsigned long long* d; cudaMalloc(&d, 8);
    int iters = 2000;
    cudaFuncSetAttribute(k_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    k_rate<N, TS><<<148, 128, 100 * 1024>>>(iters, d);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k_rate<N, TS><<<148, 128, 100 * 1024>>>(iters, d);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    double mmas = iters * 4.0;
    double flops = 2.0 * 128 * N * 16 * mmas * 148;
    printf("%-10s N=%3d: %.1f cycles/MMA (ideal %d)  %.0f TFLOP/s  err=%s\n", name, N, cyc / mmas, 128 * N / 256,
           flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run<64, false>("SS"); run<128, false>("SS"); run<256, false>("SS");
    run<64, true>("TS"); run<128, true>("TS"); run<256, true>("TS");
    return 0;
}
