// DFMA latency / throughput and a few per-column-critical-path ops on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_lat(double* out, long long* cyc, int n) {
    double a = out[threadIdx.x], b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); a = fma(a, b, c); }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}
__global__ void k_thr(double* out, long long* cyc, int n) {
    double a0 = out[threadIdx.x], a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
    const double b = 1.0000001, c = 1e-9;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
        a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
    __syncthreads();
    long long t1 = clock64();
    out[threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
    if (threadIdx.x == 0) cyc[blockIdx.x] = (t1 - t0);
}
__global__ void k_rcp(double* out, long long* cyc, int n) {
    double a = out[threadIdx.x] + 2.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) { double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a)); a = r + 2.0; }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}
__global__ void k_bar(long long* cyc, int n) {
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}
int main() {
    double* d; long long* c; cudaMalloc(&d, 1 << 20); cudaMalloc(&c, 1 << 16);
    cudaMemset(d, 0, 1 << 20);
    long long h[1024];
    int n = 10000;
    k_lat<<<1, 32>>>(d, c, n); k_lat<<<1, 32>>>(d, c, n); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", h[0] / (4.0 * n));
    for (int w : {4, 8, 16, 32}) {
        k_thr<<<148, 32 * w>>>(d, c, n); k_thr<<<148, 32 * w>>>(d, c, n);
        cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
        printf("DFMA throughput, %2d warps/SM: %.1f DFMA/cycle/SM\n", w, 32.0 * w * 8 * n / h[0]);
    }
    k_rcp<<<1, 32>>>(d, c, n); k_rcp<<<1, 32>>>(d, c, n); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
    printf("rcp.approx.f64 + DADD latency: %.1f cycles\n", h[0] / (double)n);
    for (int w : {9, 17, 32}) {
        k_bar<<<1, 32 * w>>>(c, n); k_bar<<<1, 32 * w>>>(c, n); cudaMemcpy(h, c, 8, cudaMemcpyDeviceToHost);
        printf("__syncthreads, %2d warps: %.1f cycles\n", w, h[0] / (double)n);
    }
    return 0;
}
