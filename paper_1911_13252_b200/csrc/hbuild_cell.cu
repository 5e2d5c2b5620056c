// hbuild_cell.cu -- per-cell H builders (Elman; Jordan/NARMAX teacher forced).
//
// These architectures are cell independent: h_ij depends only on
// sample i's window and neuron j's weights, so the paper's (Row, Col) thread
// decomposition (Alg. 2) is exactly right.  B200 version: one
// thread per flattened cell c = i*M + j so consecutive threads store
// consecutive H elements (coalesced, each H(Q) element written once, R14);
// Elman's lag history lives in registers (fully unrolled over a compile-time
// bound QMAX >= Q) instead of the paper's global H[Row,Col,t] round trips.
// Both kernels are bound by HBM (H stores) or by MUFU, never by FMA.
#include "common.cuh"

namespace elm {

// Eq. 5, reading R4: a_j(t) = W[:,j].x(t) + b_j + sum_{k=1}^{t-1} alpha[j,k] h_j(t-k)
// Computed in fp64 and rounded once to fp32: the kernel is launch / HBM bound,
// and Elman's H on smooth series is ill-conditioned (cond ~ 6e6 at C1), so
// fp32 recurrence error would dominate the beta error (R26).
template <int QMAX>
__global__ void __launch_bounds__(256) k_elman(const float* __restrict__ X, int64_t ldx, int64_t N, int S, int M,
                                               int Q, int act, const float* __restrict__ W,
                                               const float* __restrict__ b, const float* __restrict__ alT,
                                               float* __restrict__ H, int64_t ldh) {
    int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (cell >= N * (int64_t)M) return;
    int64_t i = cell / M;
    int j = (int)(cell - i * M);
    const float* xi = X + i * ldx;
    double al[QMAX];
#pragma unroll
    for (int k = 0; k < QMAX; ++k) al[k] = (k < Q - 1) ? (double)__ldg(alT + (int64_t)k * M + j) : 0.0;
    const double bj = __ldg(b + j);
    double h[QMAX];
    double last = 0.0;
#pragma unroll
    for (int t = 0; t < QMAX; ++t) {
        if (t < Q) {
            double a = bj;
            for (int s = 0; s < S; ++s)
                a = fma((double)__ldg(W + (int64_t)s * M + j), (double)__ldg(xi + (int64_t)t * S + s), a);
#pragma unroll
            for (int k = 1; k <= t; ++k) a = fma(al[k - 1], h[t - k], a);
            h[t] = act_g64(a, act);
            last = h[t];
        }
    }
    H[i * ldh + j] = (float)last;
}

bool elman_supported(int Q) { return Q >= 1 && Q <= 128; }

cudaError_t launch_elman(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    int64_t cells = N * (int64_t)h->M;
    int threads = 256;
    int64_t blocks = (cells + threads - 1) / threads;
    if (blocks > INT32_MAX) return cudaErrorInvalidConfiguration;
    auto go = [&](auto kern) {
        kern<<<(unsigned)blocks, threads, 0, h->stream>>>(X, ldx, N, h->S, h->M, h->Q, h->act, h->W, h->b, h->rec, H,
                                                         ldh);
    };
    const int Q = h->Q;
    if (Q <= 8) go(k_elman<8>);
    else if (Q <= 16) go(k_elman<16>);
    else if (Q <= 32) go(k_elman<32>);
    else if (Q <= 64) go(k_elman<64>);
    else go(k_elman<128>);
    h->launches++;
    return cudaGetLastError();
}

// Eqs. 6-7 under teacher forcing (R7, R8): the feedback reads the
// teacher signal, never h, so H(Q) needs step Q only (one-step collapse):
//   a_j = W[:,j].x(Q) + b_j + sum_{k=1}^{nlag} rec[k-1][j] * y(Q-k)
// Jordan: rec = alpha^T, nlag = Q-1 (y(0) = 0).  NARMAX: rec = W'^T,
// nlag = min(F, Q-1); the W'' terms multiply e == 0.
// y(tau) = Yfb[i][tau-1], or X[i][tau][0] when Yfb == NULL.
__global__ void __launch_bounds__(256) k_teacher_forced(const float* __restrict__ X, int64_t ldx,
                                                        const float* __restrict__ Yfb, int64_t ldy, int64_t N, int S,
                                                        int M, int Q, int nlag, int act,
                                                        const float* __restrict__ W, const float* __restrict__ b,
                                                        const float* __restrict__ recT, float* __restrict__ H,
                                                        int64_t ldh) {
    int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (cell >= N * (int64_t)M) return;
    int64_t i = cell / M;
    int j = (int)(cell - i * M);
    const float* xi = X + i * ldx;
    float a = __ldg(b + j);
    for (int s = 0; s < S; ++s) a = fmaf(__ldg(W + (int64_t)s * M + j), __ldg(xi + (int64_t)(Q - 1) * S + s), a);
    if (Yfb) {
        const float* yi = Yfb + i * ldy;
        for (int k = 1; k <= nlag; ++k) a = fmaf(__ldg(recT + (int64_t)(k - 1) * M + j), __ldg(yi + (Q - k - 1)), a);
    } else {
        for (int k = 1; k <= nlag; ++k)
            a = fmaf(__ldg(recT + (int64_t)(k - 1) * M + j), __ldg(xi + (int64_t)(Q - k) * S), a);
    }
    H[i * ldh + j] = act_g(a, act);
}

cudaError_t launch_teacher_forced(elmrnn* h, const float* X, int64_t ldx, const float* Yfb, int64_t ldy, int64_t N,
                                  float* H, int64_t ldh) {
    int64_t cells = N * (int64_t)h->M;
    int threads = 256;
    int64_t blocks = (cells + threads - 1) / threads;
    if (blocks > INT32_MAX) return cudaErrorInvalidConfiguration;
    int nlag = h->Q - 1;
    if (h->arch == kArchNarmax) nlag = h->F < h->Q - 1 ? h->F : h->Q - 1;
    k_teacher_forced<<<(unsigned)blocks, threads, 0, h->stream>>>(X, ldx, Yfb, ldy, N, h->S, h->M, h->Q, nlag,
                                                                  h->act, h->W, h->b, h->rec, H, ldh);
    h->launches++;
    return cudaGetLastError();
}

}  // namespace elm
