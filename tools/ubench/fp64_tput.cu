// Aggregate FP64 throughput on one SM: vector DFMA (W warps x independent chains) and DMMA m8n8k4.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double* out, long long* cyc, int iters) {
    double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double m = 1.0000001, c = 1e-9;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
            a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void k_dmma(double* out, long long* cyc, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double d0[2] = {0, 0}, d1[2] = {0, 0}, d2[2] = {0, 0}, d3[2] = {0, 0};
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#define DM(d) asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
            DM(d0) DM(d1) DM(d2) DM(d3)
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = d0[0] + d1[1] + d2[0] + d3[1];
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8);
    const int iters = 2048;
    for (int w : {1, 2, 4, 8, 16, 32}) {
        for (int rep = 0; rep < 2; ++rep) {
            k_dfma<<<1, 32 * w>>>(o, c, iters);
            long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            if (rep) printf("DFMA  warps=%2d: %6.2f DFMA/clk/SM\n", w, 32.0 * w * 32 * iters / h);
        }
    }
    for (int w : {1, 2, 4, 8, 16}) {
        for (int rep = 0; rep < 2; ++rep) {
            k_dmma<<<1, 32 * w>>>(o, c, iters);
            long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            // m8n8k4 = 256 FMA per warp-instruction
            if (rep) printf("DMMA  warps=%2d: %6.2f FMA/clk/SM (m8n8k4)\n", w, 256.0 * w * 16 * iters / h);
        }
    }
    return 0;
}
