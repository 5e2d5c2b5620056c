// readout.cu -- work on top of H(Q) and beta besides the solve:
//   * NARMAX error-feedback windows (reading R30),
//   * the free-running recursive forecast and the held-out RMSE (SURVEY 8(f)
//     row 3, reading R31).
// Citations "P:n" = PAPER.md line n.
#include <algorithm>

#include "common.cuh"

namespace elm {
// ---- NARMAX error feedback (Eq. 7, e(t) = y(t) - yhat(t) P:122; reading R30) ----
// r_k = Y_k - H_k . beta (Eq. 4, fp64 accumulation, rounded once), then
// Ef[i][tau-1] = r_{i+tau-Q} (0 when i+tau-Q < 0): rows are consecutive
// stride-1 windows of one series (R22).
__global__ void k_residual(const float* __restrict__ H, int64_t ldh, const float* __restrict__ Y, int64_t N, int M,
                           const double* __restrict__ beta, float* __restrict__ r) {
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= N) return;
    double s = 0.0;
    for (int j = lane; j < M; j += 32) s += (double)H[row * ldh + j] * beta[j];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) r[row] = (float)((double)Y[row] - s);
}

__global__ void k_error_windows(const float* __restrict__ r, int64_t N, int Q, float* __restrict__ Ef, int64_t lde) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N * Q; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / Q;
        const int tau = (int)(e - i * Q) + 1;
        const int64_t k = i + tau - Q;
        Ef[i * lde + tau - 1] = k >= 0 ? r[k] : 0.0f;
    }
}

cudaError_t launch_error_windows(elmrnn* h, const float* H, int64_t ldh, const float* Y, int64_t N,
                                 const double* beta, float* Ef, int64_t lde) {
    const int64_t blocks = (N * 32 + 255) / 256;
    if (blocks > INT32_MAX) return cudaErrorInvalidConfiguration;
    k_residual<<<(unsigned)blocks, 256, 0, h->stream>>>(H, ldh, Y, N, h->M, beta, h->rws);
    h->launches++;
    const int64_t b2 = std::min<int64_t>((N * h->Q + 255) / 256, (int64_t)h->sm_count * 16);
    k_error_windows<<<(unsigned)b2, 256, 0, h->stream>>>(h->rws, N, h->Q, Ef, lde);
    h->launches++;
    return cudaGetLastError();
}

// ---- free-running forecast (reading R31) ------------------------------------------------
// Window buffer w [N][ldw] (fp32, d = 1).  One step: yhat_i = H_i . beta (Eq. 4,
// the fused readout of the builders), Yhat[i][k] = fp32(yhat_i), then
// w_i <- (w_i[1:], fp32(yhat_i)) in k_readout_finish.
__global__ void k_window_init(const float* __restrict__ X, int64_t ldx, int64_t N, int Q, float* __restrict__ w,
                              int64_t ldw) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N * Q; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / Q;
        const int t = (int)(e - i * Q);
        w[i * ldw + t] = X[i * ldx + t];
    }
}

cudaError_t launch_window_init(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* w, int64_t ldw) {
    const int64_t b0 = std::min<int64_t>((N * h->Q + 255) / 256, (int64_t)h->sm_count * 16);
    k_window_init<<<(unsigned)b0, 256, 0, h->stream>>>(X, ldx, N, h->Q, w, ldw);
    h->launches++;
    return cudaGetLastError();
}

// ---- fused readout finish (Eq. 4) ---------------------------------
// The builders ran with a readout sink (elmrnn::ro_beta): row i's partial dot
// products H_i[segment] . beta sit in its slots; sum them in slot order (fixed:
// deterministic), round once to fp32.  Forecast (w != null, reading R31): the
// row's warp then shifts its window and appends yhat.
__global__ void k_readout_finish(const double* __restrict__ yp, int64_t N, int M, int slots, float* __restrict__ yout,
                                 int64_t ldyo, float* __restrict__ w, int64_t ldw, int Q) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    if (row >= N) return;
    const int ns = slots > 0 ? slots : (int)(((row + 1) * M - 1) / 32 - (row * M) / 32 + 1);
    double s = 0.0;
    for (int k = 0; k < ns; ++k) s += yp[k * N + row];
    const float y = (float)s;
    if (w) {
        float* wr = w + row * ldw;
        float v[4];   // Q <= 128 (checked by the caller)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int t = lane + 32 * q;
            v[q] = (t >= 1 && t < Q) ? wr[t] : 0.0f;
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int t = lane + 32 * q;
            if (t >= 1 && t < Q) wr[t - 1] = v[q];
        }
        if (lane == 0) wr[Q - 1] = y;
    }
    if (lane == 0) yout[row * ldyo] = y;
}

cudaError_t launch_readout_finish(elmrnn* h, const double* yp, int64_t N, int slots, float* yout, int64_t ldyo,
                                  float* w, int64_t ldw) {
    const int64_t blocks = (N * 32 + 255) / 256;
    if (blocks > INT32_MAX) return cudaErrorInvalidConfiguration;
    k_readout_finish<<<(unsigned)blocks, 256, 0, h->stream>>>(yp, N, h->M, slots, yout, ldyo, w, ldw, h->Q);
    h->launches++;
    return cudaGetLastError();
}

// ---- held-out RMSE: sqrt(mean((yhat - y)^2)), one CTA, fixed summation order ----------
__global__ void __launch_bounds__(1024) k_rmse(const float* __restrict__ yhat, const float* __restrict__ y, int64_t N,
                                               double* __restrict__ out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) {
        const double d = (double)yhat[i] - (double)y[i];
        s = fma(d, d, s);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
        *out = sqrt(t / (double)N);
    }
}

cudaError_t launch_rmse(elmrnn* h, const float* yhat, const float* y, int64_t N, double* out) {
    k_rmse<<<1, 1024, 0, h->stream>>>(yhat, y, N, out);
    h->launches++;
    return cudaGetLastError();
}
}  // namespace elm
