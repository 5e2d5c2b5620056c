/*
 * elmrnn.h -- C ABI of the B200-native ELM-RNN trainer (libelmrnn.so).
 *
 * Implements the data-parallel hot path of El Zini, Rizk & Awad,
 * "An Optimized and Energy-Efficient Parallel Implementation of
 * Non-Iteratively Trained Recurrent Neural Networks" (arXiv 1911.13252),
 * Alg. 1 "S-RELM":
 *   1. randomly assign the fixed weights             -> elmrnn_init
 *   2. compute H(t), t = 1..Q, keep H(Q) in R^{N x M} -> elmrnn_build_H
 *   3. beta = H(Q)^+ Y by Householder QR, z = Q^T Y,
 *      back substitution (S4.2)           -> elmrnn_solve_beta
 * and the readout of Eq. 4               -> elmrnn_predict.
 * "P:n" cites /root/reference/PAPER.md line n; readings R1..R25 of the paper's
 * silent or garbled points are listed in DESIGN.md.
 *
 * Conventions (all calls):
 *  - Pointers marked "dev" are CUDA device pointers on the handle's device,
 *    owned by the caller; "host" pointers are ordinary host memory.  The
 *    library owns its weights and workspace (freed by elmrnn_destroy).
 *  - Work is enqueued on the handle's stream (elmrnn_set_stream; default the
 *    legacy stream 0) and the call returns without synchronising, except where
 *    a host-side output (info) is requested: then the call synchronises that
 *    stream before returning.
 *  - Arguments are validated on the host before anything is launched: an
 *    error status means nothing was enqueued.  Handles are not thread safe.
 *  - Row-major layouts with explicit leading dimensions (in elements).
 *  - No CPU fallback: every arithmetic step runs in this library's CUDA
 *    kernels (sm_100a).  A missing/failed device returns ELMRNN_ERR_CUDA.
 */
#ifndef ELMRNN_H
#define ELMRNN_H

#if defined(__GNUC__)
#define ELMRNN_API __attribute__((visibility("default")))
#else
#define ELMRNN_API
#endif

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct elmrnn* elmrnn_t;

/* The six architectures of S2.2, plus three paper-literal per-cell variants. */
typedef enum {
    ELMRNN_ELMAN = 0,   /* Eq. 5: self recurrence over Q lags            */
    ELMRNN_JORDAN = 1,  /* Eq. 6: output feedback, teacher forced (R7)   */
    ELMRNN_NARMAX = 2,  /* Eq. 7: output (+ error, e == 0) feedback (R8) */
    ELMRNN_FC = 3,      /* S2.2.4: all neurons, Q lags (prose, R9)       */
    ELMRNN_LSTM = 4,    /* S2.2.5: dense U, gates (o, c, lambda, in)     */
    ELMRNN_GRU = 5,     /* S2.2.6: dense U, Cho form, gates (z, r, f)    */
    /* Paper-literal per-cell variants: cell independent, as
     * Alg. 2's thread decomposition and Table 2 assume. */
    ELMRNN_LSTM_DIAG = 6, /* S2.2.5 with diagonal recurrent weights u_g[j] */
    ELMRNN_GRU_DIAG = 7,  /* S2.2.6 (Cho) with diagonal recurrent weights u_g[j]        */
    ELMRNN_FC_EQ8 = 8     /* Eq. 8 by the letter: own history scaled by
                           * sum_l alpha[j,l,k]                         */
} elmrnn_arch;

typedef enum {
    ELMRNN_OK = 0,
    ELMRNN_WARN_RIDGE = 1,            /* rank-deficient R: beta from the ridge fallback (R19) */
    ELMRNN_ERR_ARG = -1,              /* null pointer, arch out of range, d/M/Q < 1, N < 0    */
    ELMRNN_ERR_SHAPE = -2,            /* leading dimension smaller than the logical row       */
    ELMRNN_ERR_UNDERDETERMINED = -3,  /* N_total < M                                          */
    ELMRNN_ERR_NONFINITE = -4,        /* NaN/Inf met in H or Y during the solve               */
    ELMRNN_ERR_UNSUPPORTED = -5,      /* size beyond the implemented range   */
    ELMRNN_ERR_CUDA = -6,             /* CUDA error; text in elmrnn_last_error                */
    ELMRNN_ERR_OOM = -7               /* device allocation failed                             */
} elmrnn_status;

/* Options (elmrnn_opts_default fills the defaults shown). */
typedef struct {
    int F, R;         /* NARMAX output / error lags; -1 -> Q ("max number of time
                         dependencies", Table 1; reading R8)                 */
    int act;          /* g for Elman/Jordan/NARMAX/FC: 0 sigmoid (default), 1 tanh (R3) */
    int rec_scale;    /* 0: blocks multiplying the hidden state are scaled by
                         1/sqrt(fan_in) (default, R1); 1: unit U[-1,1) everywhere     */
    int weight_grid;  /* MMA blocks (FC A, LSTM/GRU U): 0 fp32 (default), 1 rounded
                         to the fp16 grid, 2 rounded to the tf32 grid (RNA)            */
    int fc_lags;      /* FC lags L; -1 -> Q (prose reading R9); 1 = first-order FC     */
    int force_path;   /* H-builder choice: 0 auto, 1 FP32-FMA kernels, 2 tensor cores */
    int fused_train;  /* elmrnn_train route: 0 (default) build_H + solve, measured faster
                         (C1 133 vs 238 us, C2 0.94 vs 1.08 ms: the per-column leaf
                         has too few threads to also compute H); 1 the fused
                         build -> TSQR leaf where supported (H never in memory) */
} elmrnn_opts;

/* Diagnostics of a solve (host struct). */
typedef struct {
    double rho;             /* || H beta - Y ||_2 = || R_aug [beta; -1] ||_2        */
    double rmse;            /* rho / sqrt(n_total): training RMSE                   */
    double rdiag_min_abs;   /* min_k |R_kk|, k < M                                  */
    double rdiag_max_abs;   /* max_k |R_kk|, k < M                                  */
    double ridge_lambda;    /* 0, or the ridge lambda used (R19)                    */
    int rank_flag;          /* 0 full rank, 1 ridge fallback used                   */
    int64_t n_total;        /* rows that entered the factorisation                  */
} elmrnn_solve_info;

ELMRNN_API void elmrnn_opts_default(elmrnn_opts* opts);

/* Alg. 1 line 1: create a handle on the current CUDA device and draw
 * the fixed random weights on the GPU with the counter-based generator of
 * DESIGN.md "Weights" (R1, R2).  arch: elmrnn_arch; d = S input dimension
 * (Table 1); M hidden neurons; Q window length / lags; seed: weight seed.
 * Errors: ARG, UNSUPPORTED (M > 1024; Elman/fc_eq8 with Q > 128; a forced
 * tensor-core path the shape does not admit), OOM, CUDA.  *out is NULL on error. */
ELMRNN_API elmrnn_status elmrnn_init(elmrnn_t* out, int arch, int d, int M, int Q, uint64_t seed);
ELMRNN_API elmrnn_status elmrnn_init_ex(elmrnn_t* out, int arch, int d, int M, int Q, uint64_t seed,
                             const elmrnn_opts* opts);

/* Enqueue subsequent work on this cudaStream_t (NULL = legacy stream). */
ELMRNN_API elmrnn_status elmrnn_set_stream(elmrnn_t h, void* cuda_stream);

/* Alg. 1 line 2, Eqs. 5-10: H(Q) for N windows.
 *   X   dev fp32 [N][ldx], window i at X + i*ldx laid out [Q][d] (time-major,
 *       Table 1: x_j in R^{S x Q}); ldx >= Q*d.
 *   Yfb dev fp32 [N][ldy] teacher signal, Yfb[i][tau-1] = y_i(tau) (R7), or NULL:
 *       then y_i(tau) = X[i][tau][0] (univariate autoregressive window).
 *       Used by Jordan/NARMAX only; ldy >= Q when given.
 *   H   dev fp32 [N][ldh] output, ldh >= M.  Only H(Q) is written (R14), each
 *       element exactly once.
 * N == 0 is a no-op.  Errors: ARG, SHAPE, CUDA. */
ELMRNN_API elmrnn_status elmrnn_build_H(elmrnn_t h, const float* X, int64_t ldx, const float* Yfb,
                             int64_t ldy, int64_t N, float* H, int64_t ldh);

/* Eq. 7 with real error feedback (reading R30):
 * elmrnn_build_H plus, for NARMAX, the error terms sum_{l=1}^{R} W''[j][l] e(t-l).
 *   Ef  dev fp32 [N][lde] error window, Ef[i][tau-1] = e_i(tau), or NULL (e == 0,
 *       R8: identical to elmrnn_build_H); lde >= Q.  Typically the output of
 *       elmrnn_error_windows for the previous pass's beta.
 * Other arguments as elmrnn_build_H.  Errors: ARG (Ef given for another
 * architecture), SHAPE, CUDA. */
ELMRNN_API elmrnn_status elmrnn_build_H_ef(elmrnn_t h, const float* X, int64_t ldx, const float* Yfb,
                                int64_t ldy, const float* Ef, int64_t lde, int64_t N, float* H,
                                int64_t ldh);

/* NARMAX error windows for the second pass ("e(t) = y(t) - yhat(t)",
 * Eq. 4 for yhat; reading R30): with the rows of H being consecutive stride-1
 * windows of one series (R22), window i's e(tau) is the residual of window
 * k = i + tau - Q:
 *     Ef[i][tau-1] = Y[k] - sum_j H[k][j] beta[j]   (k >= 0; else 0), tau = 1..Q,
 * accumulated in fp64 and rounded once to fp32.
 *   H dev fp32 [N][ldh] (pass-0 H), Y dev fp32 [N], beta dev fp64 [M],
 *   Ef dev fp32 [N][lde] output, lde >= Q.  Uses an N-float library workspace.
 * Asynchronous.  Errors: ARG, SHAPE, OOM, CUDA. */
ELMRNN_API elmrnn_status elmrnn_error_windows(elmrnn_t h, const float* H, int64_t ldh, const float* Y,
                                   int64_t N, const double* beta, float* Ef, int64_t lde);

/* S4.2: beta = argmin ||H beta - Y||_2 by fp64 Householder
 * tall-skinny QR of [H | Y] (the reflectors are applied to Y as the augmented
 * column, so z = Q^T Y comes out of the factorisation), sign normalisation,
 * rank check with ridge fallback (R19), and back substitution R beta = z.
 *   H dev fp32 [N][ldh], Y dev fp32 [N], beta dev fp64 [M] (output).
 *   info host (optional): when non-NULL the call synchronises the stream and
 *   fills it; non-finite input is then reported as ERR_NONFINITE and a ridge
 *   solve as WARN_RIDGE.  With info == NULL the call is fully asynchronous and
 *   returns OK once enqueued.
 * Errors: ARG, SHAPE, UNDERDETERMINED (N < M), NONFINITE, OOM, CUDA. */
ELMRNN_API elmrnn_status elmrnn_solve_beta(elmrnn_t h, const float* H, int64_t ldh, const float* Y,
                                int64_t N, double* beta, elmrnn_solve_info* info);

/* Alg. 1 lines 2-3 in one call: H(Q) of the N windows (as
 * elmrnn_build_H) and beta (as elmrnn_solve_beta) -- SURVEY 8(f) row 2, "the two
 * CPU intensive operations" of P:246 fused.  For the cell-independent archs
 * (Elman with Q <= 32, Jordan, NARMAX) whose solve takes the per-column
 * TSQR (M + 1 <= 128), with opts.fused_train = 1, the TSQR leaf computes every
 * H element where it would have loaded it, so H never exists in memory
 * (elmrnn_train_fused(h) == 1); otherwise (the default, measured faster) H goes
 * through a library workspace (N*M floats) between build_H and the solve.
 *   X, Yfb as elmrnn_build_H; Y dev fp32 [N]; beta dev fp64 [M]; info as
 *   elmrnn_solve_beta.
 * Errors: ARG, SHAPE, UNDERDETERMINED (N < M), NONFINITE, OOM, CUDA. */
ELMRNN_API elmrnn_status elmrnn_train(elmrnn_t h, const float* X, int64_t ldx, const float* Yfb, int64_t ldy,
                           const float* Y, int64_t N, double* beta, elmrnn_solve_info* info);

/* Row-sharded step 1 of elmrnn_train: this rank's packed R of [H | Y] (as
 * elmrnn_solve_local) directly from its windows.  N may be 0.  Asynchronous.
 * Errors: ARG, SHAPE, OOM, CUDA. */
ELMRNN_API elmrnn_status elmrnn_train_local(elmrnn_t h, const float* X, int64_t ldx, const float* Yfb,
                                 int64_t ldy, const float* Y, int64_t N, double* Rpk);

/* 1 when elmrnn_train / elmrnn_train_local run the fused build -> leaf on this handle. */
ELMRNN_API int elmrnn_train_fused(elmrnn_t h);

/* Multi-output least squares (the paper's future work,
 * P:655): B = argmin ||H B - Y||_F for P outputs at once, by one fp64
 * Householder TSQR of [H | Y_1 .. Y_P] (the reflectors are applied to all P
 * augmented columns, z = Q^T Y), then P back substitutions with the same R.
 * Each output's beta equals elmrnn_solve_beta on that column (up to rounding).
 *   H dev fp32 [N][ldh]; Y dev fp32 [N][ldy], ldy >= P; beta dev fp64 [P][M]
 *   (output p at beta + p*M); rmse host fp64 [P] or NULL (synchronises);
 *   info as elmrnn_solve_beta, describing output 0 (the rank check and ridge
 *   are properties of H and shared by all outputs).
 * Errors: ARG, SHAPE, UNDERDETERMINED (N < M), UNSUPPORTED (M + P > 1536),
 * NONFINITE, OOM, CUDA. */
ELMRNN_API elmrnn_status elmrnn_solve_beta_multi(elmrnn_t h, const float* H, int64_t ldh, const float* Y,
                                      int64_t ldy, int P, int64_t N, double* beta, double* rmse,
                                      elmrnn_solve_info* info);

/* Row-sharded solve, step 1 (one per rank / row block): factor the local
 * [H | Y] (N rows) into its (M+1)x(M+1) upper-triangular R, written packed
 * row-major (row k holds R[k][k..M]) to Rpk dev fp64 [elmrnn_packed_r_len(h)].
 * N may be 0 (R = 0).  Asynchronous.  Errors: ARG, SHAPE, OOM, CUDA. */
ELMRNN_API elmrnn_status elmrnn_solve_local(elmrnn_t h, const float* H, int64_t ldh, const float* Y,
                                 int64_t N, double* Rpk);

/* Row-sharded solve, step 2: merge P packed R factors (dev fp64
 * [P][elmrnn_packed_r_len(h)], e.g. the output of an NCCL all-gather) by
 * Householder QR of their stack, then solve as elmrnn_solve_beta.  N_total is
 * the total row count (for the RMSE).  beta dev fp64 [M]; info as above.
 * Errors: ARG, UNDERDETERMINED, NONFINITE, OOM, CUDA. */
ELMRNN_API elmrnn_status elmrnn_solve_merge(elmrnn_t h, const double* Rpk_all, int P, int64_t N_total,
                                 double* beta, elmrnn_solve_info* info);

/* Row-sharded multi-output solve, step 1: factor the
 * local [H | Y_1 .. Y_P] (N rows) into its (M+P)x(M+P) upper-triangular R, packed
 * row-major to Rpk dev fp64 [elmrnn_packed_r_len_multi(h, P)].  H dev fp32
 * [N][ldh]; Y dev fp32 [N][ldy], ldy >= P.  N may be 0.  Asynchronous.
 * Errors: ARG, SHAPE, UNSUPPORTED (M + P > 1536), OOM, CUDA. */
ELMRNN_API elmrnn_status elmrnn_solve_local_multi(elmrnn_t h, const float* H, int64_t ldh, const float* Y,
                                       int64_t ldy, int P, int64_t N, double* Rpk);

/* Step 2: merge `ranks` packed R factors of step 1 (dev fp64 [ranks][len]) by
 * Householder QR of their stack, then P back substitutions as
 * elmrnn_solve_beta_multi: beta dev fp64 [P][M]; rmse host fp64 [P] or NULL
 * (synchronises); info as elmrnn_solve_beta_multi.
 * Errors: ARG, UNSUPPORTED, UNDERDETERMINED (N_total < M), NONFINITE, OOM, CUDA. */
ELMRNN_API elmrnn_status elmrnn_solve_merge_multi(elmrnn_t h, const double* Rpk_all, int ranks, int P,
                                       int64_t N_total, double* beta, double* rmse,
                                       elmrnn_solve_info* info);

/* (M+P)(M+P+1)/2: length of one packed multi-output R in doubles (-1 if P < 1). */
ELMRNN_API int64_t elmrnn_packed_r_len_multi(elmrnn_t h, int P);

/* Synchronise the handle's stream and report what asynchronous solves (info ==
 * NULL) could not: ERR_NONFINITE when any solve since the last synchronising
 * check (this call, or a solve with info != NULL) met NaN/Inf in H or Y (the
 * leaf kernels OR a device flag that the solve kernel accumulates).  The
 * flag is cleared.  Errors: ARG, NONFINITE, CUDA. */
ELMRNN_API elmrnn_status elmrnn_sync(elmrnn_t h);

/* (M+1)(M+2)/2: length of one packed R in doubles. */
ELMRNN_API int64_t elmrnn_packed_r_len(elmrnn_t h);

/* Eq. 4: Yhat[i] = sum_j beta_j H(Q)[i][j] (no output bias, R16),
 * fused into the H builders: the same kernels as
 * elmrnn_build_H run with a readout epilogue that writes no H(Q), only the fp64
 * partial products of each thread's H(Q) row segment with beta (a library
 * workspace of ceil(M/32)+1 doubles per row for the flattened-cell archs, 4 for
 * the others); a finish kernel sums each row's partials in a fixed order
 * (bitwise repeatable) and rounds once to fp32.
 * X, Yfb as in elmrnn_build_H; beta dev fp64 [M]; Yhat dev fp32 [N].
 * Errors: ARG, SHAPE, OOM, CUDA. */
ELMRNN_API elmrnn_status elmrnn_predict(elmrnn_t h, const float* X, int64_t ldx, const float* Yfb,
                             int64_t ldy, int64_t N, const double* beta, float* Yhat);

/* Free-running (recursive) K-step forecast (reading R31):
 * for univariate autoregressive windows (d = 1), w_0 = X[i][0..Q-1]; step k
 * computes yhat_k = H(w_k) . beta (Eq. 4; Jordan/NARMAX feed back
 * y(tau) = w_k[tau], the Yfb == NULL convention of elmrnn_build_H) and shifts
 * the prediction in as the next observation: w_{k+1} = (w_k[1:], fp32(yhat_k)).
 *   X dev fp32 [N][ldx], ldx >= Q; beta dev fp64 [M];
 *   Yhat dev fp32 [N][ldyh] output, Yhat[i][k] = yhat_k of window i, ldyh >= K.
 * Runs K (fused build -> readout, shift) rounds on the handle's stream with
 * library workspaces of N*(Q+1) floats (windows) and the readout partials of
 * elmrnn_predict.  N == 0 or K == 0 is a no-op.
 * Errors: ARG, SHAPE, UNSUPPORTED (d != 1, Q > 128), OOM, CUDA. */
ELMRNN_API elmrnn_status elmrnn_forecast(elmrnn_t h, const float* X, int64_t ldx, int64_t N,
                              const double* beta, int K, float* Yhat, int64_t ldyh);

/* Held-out RMSE (SPEC "rmse_test"): sqrt(mean_i (yhat_i - Y_i)^2)
 * with yhat = elmrnn_predict(X, Yfb, beta) on evaluation windows; fp64
 * accumulation in one CTA (fixed order).  X, Yfb as elmrnn_build_H; Y dev fp32
 * [N]; rmse host fp64 (the call synchronises the stream).
 * Errors: ARG (N < 1), SHAPE, OOM, CUDA. */
ELMRNN_API elmrnn_status elmrnn_test_rmse(elmrnn_t h, const float* X, int64_t ldx, const float* Yfb,
                               int64_t ldy, const float* Y, int64_t N, const double* beta,
                               double* rmse);

/* Parity hook: copy logical weight block block_id (DESIGN.md "Weights" block
 * map, row-major logical layout) to host_dst (count floats, must equal the
 * block's length).  Synchronous.  Errors: ARG, CUDA. */
ELMRNN_API elmrnn_status elmrnn_get_weights(elmrnn_t h, int block_id, float* host_dst, int64_t count);

/* Length of weight block block_id, or -1 when out of range. */
ELMRNN_API int64_t elmrnn_weight_block_len(elmrnn_t h, int block_id);

/* Which H-builder the handle uses: 1 FP32-FMA kernels, 2 tcgen05 tensor cores. */
ELMRNN_API int elmrnn_path(elmrnn_t h);

/* Number of CUDA kernels this handle has launched so far (evidence counter). */
ELMRNN_API int64_t elmrnn_launch_count(elmrnn_t h);

/* Text of the last error on this handle (or of the last failed init when h is NULL). */
ELMRNN_API const char* elmrnn_last_error(elmrnn_t h);

/* Free weights and workspace.  NULL is a no-op. */
ELMRNN_API void elmrnn_destroy(elmrnn_t h);

#ifdef __cplusplus
}
#endif
#endif /* ELMRNN_H */
