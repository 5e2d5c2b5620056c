// Per-column fold (k_tsqr_merge<24,2> shape) with parts switched off, to see where a
// column step's ~1.4k cycles go.  VAR: 0 full, 1 no reflector math (fixed coefs),
// 2 no apply (dot/axpy), 3 no barrier (__syncwarp only; numerically wrong), 4 R in smem.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
constexpr int TR = 24, P = 2, ROWS = 48;
__device__ __forceinline__ double rcp_fast(double d) {
    double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0); r = fma(r, e, r); e = fma(-d, r, 1.0); return fma(r, e, r);
}
__device__ __forceinline__ double sqrt_fast(double t) {
    double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t));
    y = y * fma(-0.5 * t * y, y, 1.5); double s = t * y; return fma(0.5 * y, fma(-s, s, t), s);
}
template <int VAR>
__device__ __forceinline__ void make_refl(const double (&a)[TR], double x0, double* v, double* coef, double* Rkk, int half, unsigned mask) {
    double p0 = 0, p1 = 0, p2 = 0, p3 = 0;
#pragma unroll
    for (int i = 0; i < TR; i += 4) { p0 = fma(a[i], a[i], p0); p1 = fma(a[i+1], a[i+1], p1); p2 = fma(a[i+2], a[i+2], p2); p3 = fma(a[i+3], a[i+3], p3); }
    double s2 = (p0 + p1) + (p2 + p3);
    s2 += __shfl_xor_sync(mask, s2, 1);
    double beta, u0, g;
    if (VAR == 1) { beta = x0 + s2; u0 = x0 - beta; g = 1e-3; }
    else {
        beta = -(x0 >= 0.0 ? 1.0 : -1.0) * sqrt_fast(fma(x0, x0, s2));
        u0 = x0 - beta;
        g = rcp_fast(beta * u0);
    }
#pragma unroll
    for (int i = 0; i < TR; ++i) v[half * TR + i] = a[i];
    if (half == 0) { coef[0] = g; coef[1] = u0; *Rkk = beta; }
}
template <int VAR>
__global__ void __launch_bounds__(192) kf(double* Rg, int n, long long* cyc) {
    __shared__ __align__(16) double vbuf[2 * ROWS];
    __shared__ double coefs[4];
    extern __shared__ double rsm[];
    double* R = (VAR == 4) ? rsm : Rg;
    if (VAR == 4) { for (int e = threadIdx.x; e < n * n; e += blockDim.x) rsm[e] = Rg[e]; __syncthreads(); }
    const int j = threadIdx.x / P, half = threadIdx.x % P;
    const bool own = j < n;
    double a[TR];
#pragma unroll
    for (int i = 0; i < TR; ++i) a[i] = (own ? 0.01 * (j + 1) * (i + half + 1) : 0.0);
    const double* Rj = R + j;
    auto ld = [&](int row) -> double { return (own && row < n && j >= row) ? Rj[(size_t)row * n] : 0.0; };
    double rq0 = ld(0), rq1 = ld(1), rq2 = ld(2);
    if (j == 0) make_refl<VAR>(a, rq0, vbuf, coefs, R, half, 0x3u);
    __syncthreads();
    long long t0 = clock64();
    for (int k = 0; k < n; ++k) {
        const double rkj = rq0; rq0 = rq1; rq1 = rq2; rq2 = ld(k + 3);
        const double g = coefs[2 * (k & 1)], u0 = coefs[2 * (k & 1) + 1];
        const bool upd = own && j > k && g != 0.0;
        const unsigned mu = __ballot_sync(0xffffffffu, upd);
        if (upd && VAR != 2) {
            const double2* v = reinterpret_cast<const double2*>(vbuf + (k & 1) * ROWS + half * TR);
            double w0 = (half == 0) ? u0 * rkj : 0.0, w1 = 0, w2 = 0, w3 = 0;
#pragma unroll
            for (int i = 0; i < TR; i += 4) {
                const double2 va = v[i / 2], vb = v[i / 2 + 1];
                w0 = fma(va.x, a[i], w0); w1 = fma(va.y, a[i + 1], w1); w2 = fma(vb.x, a[i + 2], w2); w3 = fma(vb.y, a[i + 3], w3);
            }
            double w = (w0 + w1) + (w2 + w3);
            w += __shfl_xor_sync(mu, w, 1);
            const double f = g * w;
            if (half == 0) R[(size_t)k * n + j] = fma(f, u0, rkj);
#pragma unroll
            for (int i = 0; i < TR; i += 2) { const double2 vv = v[i / 2]; a[i] = fma(f, vv.x, a[i]); a[i + 1] = fma(f, vv.y, a[i + 1]); }
        }
        const bool nxt = j == k + 1 && k + 1 < n;
        const unsigned mr = __ballot_sync(0xffffffffu, nxt);
        if (nxt) make_refl<VAR>(a, rq0, vbuf + ((k + 1) & 1) * ROWS, coefs + 2 * ((k + 1) & 1), R + (size_t)(k + 1) * n + (k + 1), half, mr);
        if (VAR == 3) __syncwarp(); else __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / n;
    if (VAR == 4) for (int e = threadIdx.x; e < n * n; e += blockDim.x) Rg[e] = rsm[e];
    if (a[3] == 12345.0) Rg[0] = a[5];
}
int main() {
    const int n = 65;
    double* d; cudaMalloc(&d, n * n * 8); cudaMemset(d, 0, n * n * 8);
    long long* c; cudaMalloc(&c, 8);
    const int threads = (2 * n + 31) / 32 * 32;
    const char* nm[] = {"full", "no reflector math", "no apply", "no barrier (warp sync)", "R in smem"};
    for (int v = 0; v < 5; ++v) {
        long long h = 0;
        for (int rep = 0; rep < 3; ++rep) {
            switch (v) {
            case 0: kf<0><<<1, threads>>>(d, n, c); break;
            case 1: kf<1><<<1, threads>>>(d, n, c); break;
            case 2: kf<2><<<1, threads>>>(d, n, c); break;
            case 3: kf<3><<<1, threads>>>(d, n, c); break;
            default: cudaFuncSetAttribute(kf<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, n * n * 8);
                     kf<4><<<1, threads, n * n * 8>>>(d, n, c); break;
            }
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
        }
        printf("n=%d %-24s %lld cycles per column  (%s)\n", n, nm[v], h, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
