// wy_panel<32> copy with clock probes per phase (one warp, uncontended).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
constexpr int kNBW = 16;
#ifndef SQRTDIV
#define SQRTDIV 0
#endif
__device__ __forceinline__ double rsq_nr(double t) {   // rsqrt + 2 Newton steps
    double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t));
    y = y * fma(-0.5 * t * y, y, 1.5);
    return y * fma(-0.5 * t * y, y, 1.5);
}
__device__ __forceinline__ double rcp_nr(double d) {
    double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0); r = fma(r, e, r); e = fma(-d, r, 1.0); return fma(r, e, r);
}
template <int ROWS>
__global__ void kp(double* Cg, int LDC, long long* out, int reps) {
    extern __shared__ double sm[];
    double* C = sm; double* Rd = C + ROWS * LDC; double* cgv = Rd + 256; double* cuv = cgv + 16;
    for (int e = threadIdx.x; e < ROWS * LDC; e += 32) C[e] = Cg[e];
    for (int e = threadIdx.x; e < 256; e += 32) Rd[e] = (e / 16 <= e % 16) ? 1.0 + 0.01 * e : 0.0;
    __syncwarp();
    long long acc[6] = {0, 0, 0, 0, 0, 0};
    constexpr int RPL = ROWS / 4;
    const int lane = threadIdx.x & 31, rg = lane >> 3, cp = lane & 7, c0 = 2 * cp, c1 = c0 + 1;
    const int p = 0, nbp = 16;
    for (int rep = 0; rep < reps; ++rep) {
    double a0[RPL], a1[RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) { const double* row = C + (size_t)(rg + 4 * r) * LDC + p; a0[r] = row[c0]; a1[r] = row[c1]; }
#pragma unroll
    for (int i = 0; i < kNBW; ++i) {
        constexpr unsigned F = 0xffffffffu;
        const int src = (lane & 24) | (i >> 1);
        long long t0 = clock64();
        double s2a = 0.0, s2b = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; r += 2) {
            const double x = (i & 1) ? a1[r] : a0[r], y = (i & 1) ? a1[r + 1] : a0[r + 1];
            s2a = fma(x, x, s2a); s2b = fma(y, y, s2b);
        }
        double s2 = s2a + s2b;
        s2 += __shfl_xor_sync(F, s2, 8);
        s2 += __shfl_xor_sync(F, s2, 16);
        long long t1 = clock64();
        double g = 0.0, u0 = 0.0;
        if (cp == (i >> 1)) {
            const double x0 = Rd[i * kNBW + i];
            if (s2 != 0.0) {
#if SQRTDIV == 0
                const double beta = -(x0 >= 0.0 ? 1.0 : -1.0) * sqrt(fma(x0, x0, s2));
                const double uu = x0 - beta;
                u0 = uu; g = 1.0 / (beta * uu);
#else
                const double t = fma(x0, x0, s2);
                const double rs = rsq_nr(t);
                const double beta = -(x0 >= 0.0 ? 1.0 : -1.0) * (t * rs);
                u0 = x0 - beta;
                g = -rs * rs * rcp_nr(1.0 + fabs(x0) * rs);
#endif
                if (rg == 0) Rd[i * kNBW + i] = beta;
            }
#pragma unroll
            for (int r = 0; r < RPL; ++r) C[(size_t)(rg + 4 * r) * LDC + p + i] = (i & 1) ? a1[r] : a0[r];
            if (rg == 0) { cgv[i] = g; cuv[i] = u0; }
        }
        long long t2 = clock64();
        g = __shfl_sync(F, g, i >> 1);
        u0 = __shfl_sync(F, u0, i >> 1);
        double v[RPL];
#pragma unroll
        for (int r = 0; r < RPL; ++r) v[r] = __shfl_sync(F, (i & 1) ? a1[r] : a0[r], src);
        long long t3 = clock64();
        if (g != 0.0 && i + 1 < nbp) {
            double w0 = (rg == 0 && c0 > i) ? u0 * Rd[i * kNBW + c0] : 0.0;
            double w1 = (rg == 0 && c1 > i) ? u0 * Rd[i * kNBW + c1] : 0.0;
            double w0b = 0.0, w1b = 0.0;
#pragma unroll
            for (int r = 0; r < RPL; r += 2) {
                w0 = fma(v[r], a0[r], w0); w1 = fma(v[r], a1[r], w1);
                w0b = fma(v[r + 1], a0[r + 1], w0b); w1b = fma(v[r + 1], a1[r + 1], w1b);
            }
            w0 += w0b; w1 += w1b;
            w0 += __shfl_xor_sync(F, w0, 8); w1 += __shfl_xor_sync(F, w1, 8);
            w0 += __shfl_xor_sync(F, w0, 16); w1 += __shfl_xor_sync(F, w1, 16);
            long long t4 = clock64();
            acc[3] += t4 - t3;
            const double f0 = (c0 > i) ? g * w0 : 0.0, f1 = (c1 > i) ? g * w1 : 0.0;
#pragma unroll
            for (int r = 0; r < RPL; ++r) { a0[r] = fma(f0, v[r], a0[r]); a1[r] = fma(f1, v[r], a1[r]); }
            if (rg == 0) {
                if (c0 > i) Rd[i * kNBW + c0] = fma(f0, u0, Rd[i * kNBW + c0]);
                if (c1 > i) Rd[i * kNBW + c1] = fma(f1, u0, Rd[i * kNBW + c1]);
            }
            long long t5 = clock64();
            acc[4] += t5 - t4;
        }
        acc[0] += t1 - t0; acc[1] += t2 - t1; acc[2] += t3 - t2;
    }
    __syncwarp();
    }
    if (threadIdx.x == 0) for (int k = 0; k < 5; ++k) out[k] = acc[k] / reps / 16;
    Cg[0] = C[5] + cgv[3];
}
int main() {
    const int ROWS = 32, LDC = 264;
    std::vector<double> h(ROWS * LDC);
    for (auto& x : h) x = rand() / (double)RAND_MAX - 0.5;
    double* d; long long* c; cudaMalloc(&d, h.size() * 8); cudaMalloc(&c, 64);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    size_t smem = (ROWS * LDC + 256 + 32) * 8;
    cudaFuncSetAttribute(kp<ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kp<ROWS><<<1, 32, smem>>>(d, LDC, c, 8);
    long long o[5]; cudaMemcpy(o, c, 40, cudaMemcpyDeviceToHost);
    printf("SQRTDIV=%d per column: norm+reduce %lld | reflector(owner) %lld | bcast g,u0,v %lld | dot+reduce %lld | axpy+Rd %lld  err=%s\n",
           SQRTDIV, o[0], o[1], o[2], o[3], o[4], cudaGetErrorString(cudaGetLastError()));
}
