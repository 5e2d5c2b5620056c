// Per-warp fold prototype (small n): lane l owns columns l, l+32, l+64 (CPL <= 3) of a
// TR-row tile in registers; per column k the owner lane forms the reflector over its
// TR rows (+ R_kk), publishes (v, g, u0) through shared memory, __syncwarp, and every
// lane applies it to its columns > k.  No block barrier.  Cycles per column step.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsqrt_nr(double t) {
    double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t));
    y = y * fma(-0.5 * t * y, y, 1.5); return y * fma(-0.5 * t * y, y, 1.5);
}
__device__ __forceinline__ double rcp_nr(double d) {
    double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0); r = fma(r, e, r); e = fma(-d, r, 1.0); return fma(r, e, r);
}
template <int TR, int CPL>
__global__ void kw(double* out, int n, long long* cyc) {
    __shared__ __align__(16) double vs[2][TR + 2];   // v tail, g, u0 (double-buffered)
    __shared__ double Rs[32 * 96];
    const int lane = threadIdx.x & 31;
    double a[CPL][TR], rrow[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) {
        rrow[c] = 1.0 + lane + 32 * c;
#pragma unroll
        for (int i = 0; i < TR; ++i) a[c][i] = 0.001 * ((lane + 32 * c) * 7 % 13 + i + 1);
    }
    __syncwarp();
    long long t0 = clock64();
    for (int k = 0; k < n; ++k) {
        const int oc = k >> 5, ol = k & 31;   // owner column slot, owner lane
        const int b = k & 1;
        // owner: reflector of column k (its rows + R_kk)
        if (lane == ol) {
            double x0 = 0.0, s2a = 0.0, s2b = 0.0, s2c = 0.0, s2d = 0.0;
#pragma unroll
            for (int c = 0; c < CPL; ++c)
                if (c == oc) {
                    x0 = rrow[c];
#pragma unroll
                    for (int i = 0; i < TR; i += 4) {
                        s2a = fma(a[c][i], a[c][i], s2a); s2b = fma(a[c][i + 1], a[c][i + 1], s2b);
                        s2c = fma(a[c][i + 2], a[c][i + 2], s2c); s2d = fma(a[c][i + 3], a[c][i + 3], s2d);
                    }
#pragma unroll
                    for (int i = 0; i < TR; ++i) vs[b][i] = a[c][i];
                }
            const double s2 = (s2a + s2b) + (s2c + s2d);
            const double t = fma(x0, x0, s2);
            const double rs = rsqrt_nr(t);
            const double bt = -(x0 >= 0.0 ? 1.0 : -1.0) * (t * rs);
            vs[b][TR] = -rs * rs * rcp_nr(1.0 + fabs(x0) * rs);
            vs[b][TR + 1] = x0 - bt;
#pragma unroll
            for (int c = 0; c < CPL; ++c) if (c == oc) rrow[c] = bt;
        }
        __syncwarp();
        const double g = vs[b][TR], u0 = vs[b][TR + 1];
        double v[TR];
#pragma unroll
        for (int i = 0; i < TR; ++i) v[i] = vs[b][i];
#pragma unroll
        for (int c = 0; c < CPL; ++c) {
            if (lane + 32 * c > k && lane + 32 * c < n) {
                double w0 = u0 * rrow[c], w1 = 0, w2 = 0, w3 = 0;
#pragma unroll
                for (int i = 0; i < TR; i += 4) {
                    w0 = fma(v[i], a[c][i], w0); w1 = fma(v[i + 1], a[c][i + 1], w1);
                    w2 = fma(v[i + 2], a[c][i + 2], w2); w3 = fma(v[i + 3], a[c][i + 3], w3);
                }
                const double f = g * ((w0 + w1) + (w2 + w3));
                Rs[(k & 31) * 96 + lane + 32 * c] = fma(f, u0, rrow[c]);   // R row k (then the next R row would be loaded)
                rrow[c] = Rs[((k + 1) & 31) * 96 + lane + 32 * c];
#pragma unroll
                for (int i = 0; i < TR; ++i) a[c][i] = fma(f, v[i], a[c][i]);
            }
        }
    }
    long long t1 = clock64();
    if (lane == 0) cyc[0] = (t1 - t0) / n;
    double s = 0; for (int c = 0; c < CPL; ++c) for (int i = 0; i < TR; ++i) s += a[c][i];
    out[lane] = s;
}
int main() {
    double* d; cudaMalloc(&d, 4096); long long* c; cudaMalloc(&c, 8); long long h;
#define RUN(TR, CPL, N) for (int r = 0; r < 3; ++r) kw<TR, CPL><<<1, 32>>>(d, N, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); \
    printf("TR=%2d cols/lane=%d n=%d: %lld cycles per column (%s)\n", TR, CPL, N, h, cudaGetErrorString(cudaGetLastError()));
    RUN(32, 1, 21) RUN(16, 1, 21) RUN(32, 3, 65) RUN(16, 3, 65) RUN(24, 3, 65) RUN(32, 2, 64)
    return 0;
}
