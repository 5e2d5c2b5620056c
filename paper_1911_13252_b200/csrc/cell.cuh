// cell.cuh -- per-cell H(Q) evaluation for the cell-independent architectures
// (h_ij depends only on sample i's window and neuron j's weights), as
// device functions a fused consumer can call per (row, neuron): the fused
// build -> TSQR leaf of elmrnn_train computes each H
// element where the leaf would have loaded it, so H never exists in memory.
// Same arithmetic as the standalone builders of hbuild_cell.cu (Eq. 5 in fp64,
// reading R26; the teacher-forced one-step collapse of Eqs. 6-7, R7/R8).
#pragma once
#include "common.cuh"

namespace elm {

// Source of the leaf's H elements.
struct CellSrc {
    const float* X;   // [N][ldx], window [Q][S]
    int64_t ldx;
    const float* Yfb; // [N][ldy] teacher signal or null (y(tau) = X[i][tau][0])
    int64_t ldy;
    int S, M, Q, act, nlag;
    const float* W;   // [S][M]
    const float* b;   // [M]
    const float* rec; // Elman alpha^T [Q][M]; Jordan/NARMAX feedback weights^T [nlag][M]
};

// Eq. 5, reading R4: a_j(t) = W[:,j].x(t) + b_j + sum_{k=1}^{t-1} alpha[j,k] h_j(t-k),
// fp64 arithmetic, rounded once (R26).  QMAX >= Q.
template <int QMAX>
__device__ __forceinline__ float cell_elman(const CellSrc& c, int64_t i, int j) {
    const float* xi = c.X + i * c.ldx;
    double h[QMAX];
    double last = 0.0;
    const double bj = __ldg(c.b + j);
#pragma unroll
    for (int t = 0; t < QMAX; ++t) {
        if (t < c.Q) {
            double a = bj;
            for (int s = 0; s < c.S; ++s)
                a = fma((double)__ldg(c.W + (int64_t)s * c.M + j), (double)__ldg(xi + (int64_t)t * c.S + s), a);
            // the lag sum in 4 partial sums, in k_elman's order (bitwise-identical H)
            double p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll
            for (int k = 1; k <= t; ++k) {
                const double al = __ldg(c.rec + (int64_t)(k - 1) * c.M + j), v = h[t - k];
                if ((k & 3) == 1) a = fma(al, v, a);
                else if ((k & 3) == 2) p1 = fma(al, v, p1);
                else if ((k & 3) == 3) p2 = fma(al, v, p2);
                else p3 = fma(al, v, p3);
            }
            a = (a + p1) + (p2 + p3);
            h[t] = act_g64(a, c.act);
            last = h[t];
        }
    }
    return (float)last;
}

// Eqs. 6-7 under teacher forcing (R7, R8): one-step collapse,
// a_j = W[:,j].x(Q) + b_j + sum_{k=1}^{nlag} rec[k-1][j] y(Q-k).
__device__ __forceinline__ float cell_tf(const CellSrc& c, int64_t i, int j) {
    const float* xi = c.X + i * c.ldx;
    float a = __ldg(c.b + j);
    for (int s = 0; s < c.S; ++s) a = fmaf(__ldg(c.W + (int64_t)s * c.M + j), __ldg(xi + (int64_t)(c.Q - 1) * c.S + s), a);
    if (c.Yfb) {
        const float* yi = c.Yfb + i * c.ldy;
        for (int k = 1; k <= c.nlag; ++k) a = fmaf(__ldg(c.rec + (int64_t)(k - 1) * c.M + j), __ldg(yi + (c.Q - k - 1)), a);
    } else {
        for (int k = 1; k <= c.nlag; ++k)
            a = fmaf(__ldg(c.rec + (int64_t)(k - 1) * c.M + j), __ldg(xi + (int64_t)(c.Q - k) * c.S), a);
    }
    return act_g(a, c.act);
}

}  // namespace elm
