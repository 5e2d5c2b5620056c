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
#include <algorithm>

#include "common.cuh"

namespace elm {

// Eq. 5, reading R4: a_j(t) = W[:,j].x(t) + b_j + sum_{k=1}^{t-1} alpha[j,k] h_j(t-k)
// Computed in fp64 and rounded once to fp32: the kernel is launch / HBM bound,
// and Elman's H on smooth series is ill-conditioned (cond ~ 6e6 at C1), so
// fp32 recurrence error would dominate the beta error (R26).
// T = double for Elman (R26); T = float for FC by Eq. 8 (R29), whose lag sums
// are well conditioned at the C3 shape and whose Q^2 fp64 work would dominate.
__device__ __forceinline__ double act_T(double a, int act) { return act_g64(a, act); }
__device__ __forceinline__ float act_T(float a, int act) { return act_g(a, act); }

template <int QMAX, typename T = double>
__global__ void __launch_bounds__(256) k_elman(const float* __restrict__ X, int64_t ldx, int64_t N, int S, int M,
                                               int Q, int act, const float* __restrict__ W,
                                               const float* __restrict__ b, const float* __restrict__ alT,
                                               float* __restrict__ H, int64_t ldh, const double* __restrict__ rbeta,
                                               double* __restrict__ ryp) {
    const int64_t cell0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool live = cell0 < N * (int64_t)M;
    if (!live && !rbeta) return;   // the fused readout needs every lane of the warp
    const int64_t cell = live ? cell0 : 0;
    int64_t i = cell / M;
    int j = (int)(cell - i * M);
    const float* xi = X + i * ldx;
    T al[QMAX];
#pragma unroll
    for (int k = 0; k < QMAX; ++k) al[k] = (k < Q - 1) ? (T)__ldg(alT + (int64_t)k * M + j) : (T)0;
    const T bj = __ldg(b + j);
    T h[QMAX];
    T last = 0;
    T w4[4];   // W[:,j] for S <= 4 (larger S re-reads from L1)
#pragma unroll
    for (int s = 0; s < 4; ++s) w4[s] = s < S ? (T)__ldg(W + (int64_t)s * M + j) : (T)0;
#pragma unroll
    for (int t = 0; t < QMAX; ++t) {
        if (t < Q) {
            T a = bj;
            if (S <= 4) {
#pragma unroll
                for (int s = 0; s < 4; ++s)
                    if (s < S) a = fma(w4[s], (T)__ldg(xi + (int64_t)t * S + s), a);
            } else {
                for (int s = 0; s < S; ++s)
                    a = fma((T)__ldg(W + (int64_t)s * M + j), (T)__ldg(xi + (int64_t)t * S + s), a);
            }
            if constexpr (QMAX <= 32) {
                // lag sum in 4 independent partial sums (shortens the dependent chain 4x)
                T p1 = 0, p2 = 0, p3 = 0;
#pragma unroll
                for (int k = 1; k <= t; ++k) {
                    const T v = h[t - k];
                    if ((k & 3) == 1) a = fma(al[k - 1], v, a);
                    else if ((k & 3) == 2) p1 = fma(al[k - 1], v, p1);
                    else if ((k & 3) == 3) p2 = fma(al[k - 1], v, p2);
                    else p3 = fma(al[k - 1], v, p3);
                }
                a = (a + p1) + (p2 + p3);
            } else {
#pragma unroll
                for (int k = 1; k <= t; ++k) a = fma(al[k - 1], h[t - k], a);
            }
            h[t] = act_T(a, act);
            last = h[t];
        }
    }
    if (rbeta) ro_cell_store(live ? (double)(float)last * __ldg(rbeta + j) : 0.0, cell0, N, M, ryp);   // Eq. 4
    else H[i * ldh + j] = (float)last;
}

bool elman_supported(int Q) { return Q >= 1 && Q <= 128; }

// Diagonal-U LSTM / GRU: cell independent, so
// one thread per flattened cell c = i*M + j (coalesced H store) with h (and c)
// in registers for all Q steps; W_g[:,j], u_g[j], b_g[j] in registers (S <= 4
// compile-time padded, larger S re-read from L1).  Gate order as the dense
// kernels: LSTM (o, c, lambda, in), GRU (z, r, f).  fp32 arithmetic with the
// MUFU activations of the tensor-core epilogues (ex2 + rcp); bound by MUFU /
// issue, not by HBM.
template <bool IS_LSTM, int SS>
__global__ void __launch_bounds__(256) k_diag_gated(const float* __restrict__ X, int64_t ldx, int64_t N, int S, int M,
                                                    int Q, const float* __restrict__ W, const float* __restrict__ b,
                                                    const float* __restrict__ u, float* __restrict__ H, int64_t ldh,
                                                    const double* __restrict__ rbeta, double* __restrict__ ryp) {
    constexpr int G = IS_LSTM ? 4 : 3;
    const int64_t cell0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const bool live = cell0 < N * (int64_t)M;
    if (!live && !rbeta) return;   // the fused readout needs every lane of the warp
    const int64_t cell = live ? cell0 : 0;
    const int64_t i = cell / M;
    const int j = (int)(cell - i * M), GM = G * M;
    const float* xi = X + i * ldx;
    float ug[G], bg[G], wg[G][SS > 0 ? SS : 1];
#pragma unroll
    for (int g = 0; g < G; ++g) {
        ug[g] = __ldg(u + g * M + j);
        bg[g] = __ldg(b + g * M + j);
#pragma unroll
        for (int s = 0; s < SS; ++s) wg[g][s] = s < S ? __ldg(W + (int64_t)s * GM + g * M + j) : 0.0f;
    }
    float h = 0.0f, c = 0.0f;
    for (int t = 0; t < Q; ++t) {
        float a[G];
#pragma unroll
        for (int g = 0; g < G; ++g) a[g] = bg[g];
        if constexpr (SS > 0) {
#pragma unroll
            for (int s = 0; s < SS; ++s) {
                const float x = s < S ? __ldg(xi + (int64_t)t * S + s) : 0.0f;
#pragma unroll
                for (int g = 0; g < G; ++g) a[g] = fmaf(wg[g][s], x, a[g]);
            }
        } else {
            for (int s = 0; s < S; ++s) {
                const float x = __ldg(xi + (int64_t)t * S + s);
#pragma unroll
                for (int g = 0; g < G; ++g) a[g] = fmaf(__ldg(W + (int64_t)s * GM + g * M + j), x, a[g]);
            }
        }
        if constexpr (IS_LSTM) {
            const float o = sigmoid_fast(fmaf(ug[0], h, a[0]));
            const float cc = tanh_fast(fmaf(ug[1], h, a[1]));
            const float lam = sigmoid_fast(fmaf(ug[2], h, a[2]));
            const float in = sigmoid_fast(fmaf(ug[3], h, a[3]));
            c = fmaf(lam, c, in * cc);
            h = o * tanh_fast(c);
        } else {
            const float z = sigmoid_fast(fmaf(ug[0], h, a[0]));
            const float r = sigmoid_fast(fmaf(ug[1], h, a[1]));
            const float nn = tanh_fast(fmaf(ug[2], r * h, a[2]));
            h = fmaf(z, nn - h, h);   // (1 - z) h + z n
        }
    }
    if (rbeta) ro_cell_store(live ? (double)h * __ldg(rbeta + j) : 0.0, cell0, N, M, ryp);   // Eq. 4
    else H[i * ldh + j] = h;
}

cudaError_t launch_diag_gated(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    const int64_t cells = N * (int64_t)h->M;
    const int threads = 256;
    const int64_t blocks = (cells + threads - 1) / threads;
    if (blocks > INT32_MAX) return cudaErrorInvalidConfiguration;
    auto go = [&](auto kern) {
        kern<<<(unsigned)blocks, threads, 0, h->stream>>>(X, ldx, N, h->S, h->M, h->Q, h->W, h->b, h->rec, H, ldh,
                                                         h->ro_beta, h->ro_yp);
    };
    h->ro_slots = kRoCellSlots;
    const bool lstm = h->arch == kArchLSTMDiag;
    const int S = h->S;
    if (lstm) {
        if (S == 1) go(k_diag_gated<true, 1>); else if (S <= 2) go(k_diag_gated<true, 2>);
        else if (S <= 4) go(k_diag_gated<true, 4>); else go(k_diag_gated<true, 0>);
    } else {
        if (S == 1) go(k_diag_gated<false, 1>); else if (S <= 2) go(k_diag_gated<false, 2>);
        else if (S <= 4) go(k_diag_gated<false, 4>); else go(k_diag_gated<false, 0>);
    }
    h->launches++;
    return cudaGetLastError();
}

cudaError_t launch_elman(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    int64_t cells = N * (int64_t)h->M;
    int threads = 256;
    int64_t blocks = (cells + threads - 1) / threads;
    if (blocks > INT32_MAX) return cudaErrorInvalidConfiguration;
    auto go = [&](auto kern) {
        kern<<<(unsigned)blocks, threads, 0, h->stream>>>(X, ldx, N, h->S, h->M, h->Q, h->act, h->W, h->b, h->rec, H,
                                                         ldh, h->ro_beta, h->ro_yp);
    };
    h->ro_slots = kRoCellSlots;
    const int Q = h->Q;
    if (h->arch == kArchFCEq8) {
        if (Q <= 8) go(k_elman<8, float>);
        else if (Q <= 16) go(k_elman<16, float>);
        else if (Q <= 32) go(k_elman<32, float>);
        else if (Q <= 64) go(k_elman<64, float>);
        else go(k_elman<128, float>);
    } else if (Q <= 8) go(k_elman<8>);
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
// nlag = min(F, Q-1); the W'' terms multiply e == 0 (R8) unless an error
// window is given (R30): + sum_{l=1}^{nerr} W''^T[l-1][j] e(Q-l), nerr = min(R, Q-1).
// y(tau) = Yfb[i][tau-1], or X[i][tau][0] when Yfb == NULL; e(tau) = Ef[i][tau-1].
//
// Row tile of kTfRows samples per CTA: the tile's feedback windows (y and e,
// lag-major [k][row] so one 16-B shared load serves 4 rows) and x(Q) are
// staged in shared memory once; thread = neuron j (strided by the block size),
// each weight rec[k-1][j] is loaded once per tile (coalesced over j) and used
// for all rows of the tile from registers.  Stores are coalesced over j.  (The
// one-thread-per-cell form spent its issue slots on a 64-bit cell / M division
// and on per-cell weight re-loads: 97 us for C2 against a ~5 us HBM floor.)
constexpr int kTfRows = 32;
__global__ void __launch_bounds__(256) k_teacher_forced(const float* __restrict__ X, int64_t ldx,
                                                        const float* __restrict__ Yfb, int64_t ldy, int64_t N, int S,
                                                        int M, int Q, int nlag, int act,
                                                        const float* __restrict__ W, const float* __restrict__ b,
                                                        const float* __restrict__ recT, float* __restrict__ H,
                                                        int64_t ldh, const float* __restrict__ Ef, int64_t lde,
                                                        int nerr, const float* __restrict__ recE,
                                                        const double* __restrict__ rbeta, double* __restrict__ ryp) {
    extern __shared__ __align__(16) float tf_sm[];
    float* ys = tf_sm;                          // [nlag][kTfRows]: ys[k-1][r] = y_r(Q-k)
    float* es = ys + nlag * kTfRows;            // [nerr][kTfRows]: es[l-1][r] = e_r(Q-l)
    float* xs = es + nerr * kTfRows;            // [S][kTfRows]:    xs[s][r] = x_r(Q)[s]
    const int64_t r0 = (int64_t)blockIdx.x * kTfRows;
    const int rows = (int)min((int64_t)kTfRows, N - r0);
    for (int e = threadIdx.x; e < nlag * kTfRows; e += blockDim.x) {
        const int k = e / kTfRows + 1, r = e % kTfRows;
        float v = 0.0f;
        if (r < rows) v = Yfb ? __ldg(Yfb + (r0 + r) * ldy + (Q - k - 1)) : __ldg(X + (r0 + r) * ldx + (int64_t)(Q - k) * S);
        ys[e] = v;
    }
    for (int e = threadIdx.x; e < nerr * kTfRows; e += blockDim.x) {
        const int l = e / kTfRows + 1, r = e % kTfRows;
        es[e] = r < rows ? __ldg(Ef + (r0 + r) * lde + (Q - l - 1)) : 0.0f;
    }
    for (int e = threadIdx.x; e < S * kTfRows; e += blockDim.x) {
        const int s = e / kTfRows, r = e % kTfRows;
        xs[e] = r < rows ? __ldg(X + (r0 + r) * ldx + (int64_t)(Q - 1) * S + s) : 0.0f;
    }
    __syncthreads();
    double yacc[kTfRows];   // fused readout (Eq. 4): this thread's neurons' share of each row's H . beta
#pragma unroll
    for (int r = 0; r < kTfRows; ++r) yacc[r] = 0.0;
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
        float a[kTfRows];
        const float bj = __ldg(b + j);
#pragma unroll
        for (int r = 0; r < kTfRows; ++r) a[r] = bj;
        for (int s = 0; s < S; ++s) {
            const float w = __ldg(W + (int64_t)s * M + j);
            const float4* x4 = reinterpret_cast<const float4*>(xs + s * kTfRows);
#pragma unroll
            for (int q = 0; q < kTfRows / 4; ++q) {
                const float4 v = x4[q];
                a[4 * q] = fmaf(w, v.x, a[4 * q]);
                a[4 * q + 1] = fmaf(w, v.y, a[4 * q + 1]);
                a[4 * q + 2] = fmaf(w, v.z, a[4 * q + 2]);
                a[4 * q + 3] = fmaf(w, v.w, a[4 * q + 3]);
            }
        }
        for (int k = 1; k <= nlag; ++k) {
            const float w = __ldg(recT + (int64_t)(k - 1) * M + j);
            const float4* y4 = reinterpret_cast<const float4*>(ys + (k - 1) * kTfRows);
#pragma unroll
            for (int q = 0; q < kTfRows / 4; ++q) {
                const float4 v = y4[q];
                a[4 * q] = fmaf(w, v.x, a[4 * q]);
                a[4 * q + 1] = fmaf(w, v.y, a[4 * q + 1]);
                a[4 * q + 2] = fmaf(w, v.z, a[4 * q + 2]);
                a[4 * q + 3] = fmaf(w, v.w, a[4 * q + 3]);
            }
        }
        for (int l = 1; l <= nerr; ++l) {
            const float w = __ldg(recE + (int64_t)(l - 1) * M + j);
            const float4* e4 = reinterpret_cast<const float4*>(es + (l - 1) * kTfRows);
#pragma unroll
            for (int q = 0; q < kTfRows / 4; ++q) {
                const float4 v = e4[q];
                a[4 * q] = fmaf(w, v.x, a[4 * q]);
                a[4 * q + 1] = fmaf(w, v.y, a[4 * q + 1]);
                a[4 * q + 2] = fmaf(w, v.z, a[4 * q + 2]);
                a[4 * q + 3] = fmaf(w, v.w, a[4 * q + 3]);
            }
        }
        if (rbeta) {
            const double bj = __ldg(rbeta + j);
#pragma unroll
            for (int r = 0; r < kTfRows; ++r) yacc[r] = fma((double)act_g(a[r], act), bj, yacc[r]);
        } else {
#pragma unroll
            for (int r = 0; r < kTfRows; ++r)
                if (r < rows) H[(r0 + r) * ldh + j] = act_g(a[r], act);
        }
    }
    if (rbeta) {   // reduce over the CTA's neurons in a fixed order: lanes (shuffle tree), then warps
        __syncthreads();   // the staged windows are no longer read: reuse that shared memory
        double* red = reinterpret_cast<double*>(tf_sm);   // [warp][row]
        const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = (int)(blockDim.x >> 5);
#pragma unroll
        for (int r = 0; r < kTfRows; ++r) {
            double v = yacc[r];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            if (lane == r) red[warp * kTfRows + r] = v;
        }
        __syncthreads();
        if (threadIdx.x < rows) {
            double v = 0.0;
            for (int w = 0; w < nwarp; ++w) v += red[w * kTfRows + threadIdx.x];
            ryp[r0 + threadIdx.x] = v;
        }
    }
}

cudaError_t launch_teacher_forced(elmrnn* h, const float* X, int64_t ldx, const float* Yfb, int64_t ldy, int64_t N,
                                  float* H, int64_t ldh, const float* Ef, int64_t lde) {
    const int64_t blocks = (N + kTfRows - 1) / kTfRows;
    if (blocks > INT32_MAX) return cudaErrorInvalidConfiguration;
    int nlag = h->Q - 1;
    if (h->arch == kArchNarmax) nlag = h->F < h->Q - 1 ? h->F : h->Q - 1;
    const bool ef = Ef && h->arch == kArchNarmax;
    const int nerr = ef ? (h->R < h->Q - 1 ? h->R : h->Q - 1) : 0;
    size_t smem = sizeof(float) * kTfRows * (size_t)(nlag + nerr + h->S);
    if (h->ro_beta) smem = std::max(smem, sizeof(double) * kTfRows * 8);   // readout reduction: [8 warps][rows]
    if (smem > 227 * 1024) return cudaErrorInvalidConfiguration;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_teacher_forced, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e) return e;
    }
    const int threads = h->M >= 256 ? 256 : ((h->M + 31) / 32) * 32;
    k_teacher_forced<<<(unsigned)blocks, threads, smem, h->stream>>>(X, ldx, Yfb, ldy, N, h->S, h->M, h->Q, nlag,
                                                                     h->act, h->W, h->b, h->rec, H, ldh,
                                                                     ef ? Ef : nullptr, lde, nerr,
                                                                     h->rec + (size_t)h->F * h->M, h->ro_beta, h->ro_yp);
    h->ro_slots = 1;
    h->launches++;
    return cudaGetLastError();
}

}  // namespace elm
