// Panel-factorisation latency experiments (one warp, ROWS=32, 16 columns).
// Flags: HOIST (prefetch x0 / Rd row before the reductions), DEFER (write v to
// smem after the update), RSQ (rsqrt+rcp Newton instead of IEEE sqrt/div).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#ifndef HOIST
#define HOIST 0
#endif
#ifndef DEFER
#define DEFER 0
#endif
#ifndef RSQ
#define RSQ 0
#endif
constexpr int kNBW = 16;
__device__ __forceinline__ double rsq_nr(double t) {
    double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t));
    y = y * fma(-0.5 * t * y, y, 1.5);
    return y * fma(-0.5 * t * y, y, 1.5);
}
__device__ __forceinline__ double rcp_nr(double d) {
    double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0); r = fma(r, e, r); e = fma(-d, r, 1.0); return fma(r, e, r);
}
template <int ROWS>
__device__ __noinline__ void panel(double* __restrict__ C, int LDC, int p, double* Rd, double* cgv, double* cuv) {
    constexpr int RPL = ROWS / 4;
    const int lane = threadIdx.x & 31, rg = lane >> 3, cp = lane & 7, c0 = 2 * cp, c1 = c0 + 1;
    constexpr int nbp = 16;
    double a0[RPL], a1[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) { const double* row = C + (size_t)(rg + 4 * r) * LDC + p; a0[r] = row[c0]; a1[r] = row[c1]; }
    double x0n = Rd[0], rd0n = Rd[c0], rd1n = Rd[c1];
#pragma unroll
    for (int i = 0; i < kNBW; ++i) {
        constexpr unsigned F = 0xffffffffu;
        const int src = (lane & 24) | (i >> 1);
#if HOIST
        const double x0 = x0n, rd0 = rd0n, rd1 = rd1n;
        if (i + 1 < kNBW) { x0n = Rd[(i + 1) * kNBW + i + 1]; rd0n = Rd[(i + 1) * kNBW + c0]; rd1n = Rd[(i + 1) * kNBW + c1]; }
#endif
        double s2a = 0.0, s2b = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; r += 2) {
            const double x = (i & 1) ? a1[r] : a0[r], y = (i & 1) ? a1[r + 1] : a0[r + 1];
            s2a = fma(x, x, s2a); s2b = fma(y, y, s2b);
        }
        double s2 = s2a + s2b;
        s2 += __shfl_xor_sync(F, s2, 8);
        s2 += __shfl_xor_sync(F, s2, 16);
        double g = 0.0, u0 = 0.0;
        if (cp == (i >> 1)) {
#if !HOIST
            const double x0 = Rd[i * kNBW + i];
#endif
            if (s2 != 0.0) {
#if RSQ
                const double t = fma(x0, x0, s2);
                const double rs = rsq_nr(t);
                const double beta = -(x0 >= 0.0 ? 1.0 : -1.0) * (t * rs);
                u0 = x0 - beta;
                g = -rs * rs * rcp_nr(1.0 + fabs(x0) * rs);
#else
                const double beta = -(x0 >= 0.0 ? 1.0 : -1.0) * sqrt(fma(x0, x0, s2));
                u0 = x0 - beta;
                g = 1.0 / (beta * u0);
#endif
                if (rg == 0) Rd[i * kNBW + i] = beta;
            }
#if !DEFER
#pragma unroll
            for (int r = 0; r < RPL; ++r) C[(size_t)(rg + 4 * r) * LDC + p + i] = (i & 1) ? a1[r] : a0[r];
#endif
            if (rg == 0) { cgv[i] = g; cuv[i] = u0; }
        }
        g = __shfl_sync(F, g, i >> 1);
        u0 = __shfl_sync(F, u0, i >> 1);
        double v[RPL];
#pragma unroll
        for (int r = 0; r < RPL; ++r) v[r] = __shfl_sync(F, (i & 1) ? a1[r] : a0[r], src);
#if DEFER
        if (cp == (i >> 1)) {
#pragma unroll
            for (int r = 0; r < RPL; ++r) C[(size_t)(rg + 4 * r) * LDC + p + i] = v[r];
        }
#endif
        if (g != 0.0 && i + 1 < nbp) {
#if HOIST
            double w0 = (rg == 0 && c0 > i) ? u0 * rd0 : 0.0;
            double w1 = (rg == 0 && c1 > i) ? u0 * rd1 : 0.0;
#else
            double w0 = (rg == 0 && c0 > i) ? u0 * Rd[i * kNBW + c0] : 0.0;
            double w1 = (rg == 0 && c1 > i) ? u0 * Rd[i * kNBW + c1] : 0.0;
#endif
            double w0b = 0.0, w1b = 0.0;
#pragma unroll
            for (int r = 0; r < RPL; r += 2) {
                w0 = fma(v[r], a0[r], w0); w1 = fma(v[r], a1[r], w1);
                w0b = fma(v[r + 1], a0[r + 1], w0b); w1b = fma(v[r + 1], a1[r + 1], w1b);
            }
            w0 += w0b; w1 += w1b;
            w0 += __shfl_xor_sync(F, w0, 8); w1 += __shfl_xor_sync(F, w1, 8);
            w0 += __shfl_xor_sync(F, w0, 16); w1 += __shfl_xor_sync(F, w1, 16);
            const double f0 = (c0 > i) ? g * w0 : 0.0, f1 = (c1 > i) ? g * w1 : 0.0;
#pragma unroll
            for (int r = 0; r < RPL; ++r) { a0[r] = fma(f0, v[r], a0[r]); a1[r] = fma(f1, v[r], a1[r]); }
            if (rg == 0) {
#if HOIST
                if (c0 > i) Rd[i * kNBW + c0] = fma(f0, u0, rd0);
                if (c1 > i) Rd[i * kNBW + c1] = fma(f1, u0, rd1);
#else
                if (c0 > i) Rd[i * kNBW + c0] = fma(f0, u0, Rd[i * kNBW + c0]);
                if (c1 > i) Rd[i * kNBW + c1] = fma(f1, u0, Rd[i * kNBW + c1]);
#endif
            }
        }
    }
    __syncwarp();
}
template <int ROWS>
__global__ void kp(double* Cg, int LDC, long long* cyc, int reps) {
    extern __shared__ double sm[];
    double* C = sm; double* Rd = C + ROWS * LDC; double* cg = Rd + 256; double* cu = cg + 16;
    for (int e = threadIdx.x; e < ROWS * LDC; e += 32) C[e] = Cg[e];
    for (int e = threadIdx.x; e < 256; e += 32) Rd[e] = (e / 16 <= e % 16) ? 1.0 + 0.01 * e : 0.0;
    __syncwarp();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) panel<ROWS>(C, LDC, 0, Rd, cg, cu);
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
    Cg[0] = C[5] + cg[3];
}
int main() {
    const int ROWS = 32, LDC = 264;
    std::vector<double> h(ROWS * LDC);
    for (auto& x : h) x = rand() / (double)RAND_MAX - 0.5;
    double* d; long long* c; cudaMalloc(&d, h.size() * 8); cudaMalloc(&c, 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    size_t smem = (ROWS * LDC + 256 + 32) * 8;
    cudaFuncSetAttribute(kp<ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kp<ROWS><<<1, 32, smem>>>(d, LDC, c, 64);
    long long hc; cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("HOIST=%d DEFER=%d RSQ=%d: %lld cycles/panel, %lld per column\n", HOIST, DEFER, RSQ, hc, hc / 16);
}
