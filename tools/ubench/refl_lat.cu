// Latency of the Householder reflector chain pieces on one warp (cycles per iteration).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp_fast(double d) {
    const double ad = fabs(d);
    if (!(ad > 1e-250 && ad < 1e250)) return 1.0 / d;
    double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0); r = fma(r, e, r); e = fma(-d, r, 1.0); return fma(r, e, r);
}
__device__ __forceinline__ double sqrt_fast(double t) {
    if (!(t > 1e-250 && t < 1e250)) return sqrt(t);
    double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t));
    y = y * fma(-0.5 * t * y, y, 1.5); double s = t * y; return fma(0.5 * y, fma(-s, s, t), s);
}
template <int MODE>
__global__ void k(double* out, long long* cyc, int iters) {
    __shared__ double sm[64];
    double a[16];
    for (int i = 0; i < 16; ++i) a[i] = 1.0 + 0.001 * (threadIdx.x + i);
    double x = 0.5;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        double r;
        if (MODE == 0) {            // DFMA dependent chain x16
            r = x;
#pragma unroll
            for (int i = 0; i < 16; ++i) r = fma(r, 1.0000001, 1e-9);
        } else if (MODE == 1) {     // norm: 16 FMA in 4 chains + adds
            double p0 = 0, p1 = 0, p2 = 0, p3 = 0;
#pragma unroll
            for (int i = 0; i < 16; i += 4) { p0 = fma(a[i] * x, a[i], p0); p1 = fma(a[i+1], a[i+1] * x, p1); p2 = fma(a[i+2], a[i+2] * x, p2); p3 = fma(a[i+3], a[i+3] * x, p3); }
            r = (p0 + p1) + (p2 + p3);
        } else if (MODE == 2) {     // two double butterfly shuffles
            r = x;
            r += __shfl_xor_sync(0xffffffffu, r, 1);
            r += __shfl_xor_sync(0xffffffffu, r, 2);
        } else if (MODE == 3) {     // sqrt_fast
            r = sqrt_fast(x + 1.0);
        } else if (MODE == 4) {     // rcp_fast
            r = rcp_fast(x + 1.0);
        } else if (MODE == 5) {     // smem round trip (store, syncwarp, load)
            sm[threadIdx.x] = x; __syncwarp(); r = sm[(threadIdx.x + 1) & 31];
        } else if (MODE == 6) {     // IEEE sqrt
            r = sqrt(x + 1.0);
        } else if (MODE == 7) {     // IEEE div
            r = 1.0 / (x + 1.0);
        } else if (MODE == 8) {     // __syncthreads (block of blockDim)
            r = x + 1e-9; __syncthreads();
        } else {                    // MUFU rsqrt only
            asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x + 1.0));
        }
        x = r * 0.5 + 0.25;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 8);
    const char* names[] = {"16 dep DFMA", "norm 16 (4 chains)", "2 dbl shfl", "sqrt_fast", "rcp_fast", "smem rt",
                           "IEEE sqrt", "IEEE div", "syncthreads(352)", "MUFU rsqrt64"};
    const int iters = 4096;
    for (int m = 0; m < 10; ++m) {
        for (int rep = 0; rep < 2; ++rep) {
            int threads = m == 8 ? 352 : 32;
            switch (m) {
            case 0: k<0><<<1, threads>>>(o, c, iters); break; case 1: k<1><<<1, threads>>>(o, c, iters); break;
            case 2: k<2><<<1, threads>>>(o, c, iters); break; case 3: k<3><<<1, threads>>>(o, c, iters); break;
            case 4: k<4><<<1, threads>>>(o, c, iters); break; case 5: k<5><<<1, threads>>>(o, c, iters); break;
            case 6: k<6><<<1, threads>>>(o, c, iters); break; case 7: k<7><<<1, threads>>>(o, c, iters); break;
            case 8: k<8><<<1, threads>>>(o, c, iters); break; default: k<9><<<1, threads>>>(o, c, iters); break;
            }
            long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            if (rep) printf("%-22s %7.1f cycles/iter (incl. x = r*0.5+0.25: 1 DFMA)\n", names[m], (double)h / iters);
        }
    }
    return 0;
}
