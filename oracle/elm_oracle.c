/*
 * elm_oracle.c -- TEST INFRASTRUCTURE ONLY.  A plain, slow, fp64 CPU oracle for
 * ELM training of the six RNN architectures of El Zini, Rizk & Awad,
 * "An Optimized and Energy-Efficient Parallel Implementation of
 * Non-Iteratively Trained Recurrent Neural Networks" (arXiv 1911.13252).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library.  It shares no code with the CUDA path
 * under paper_1911_13252_b200/ (no headers, no helpers, no tables); the weight
 * generator below is an independent implementation of the counter-based RNG
 * specified in DESIGN.md "Weights".
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n (section / equation named).
 *
 *   Alg. 1 (S-RELM), P:214-223     : init -> H(t), t=1..Q -> beta = H(Q)^+ Y
 *   Eq. 5  Elman,  P:226-228       : self recurrence over Q lags
 *   Eq. 6  Jordan, P:229-231       : output feedback (teacher forced, reading R7)
 *   Eq. 7  NARMAX, P:232-234       : output + error feedback (e == 0, reading R8;
 *                                    or a given e: SURVEY 8(f) row 4, reading R30)
 *   S2.2.4 fully connected, P:125-127 (prose reading R9: all neurons, Q lags)
 *   S2.2.5 LSTM, P:128-142 ; S2.2.6 GRU, P:144-150 (dense U, reading R10/R11)
 *   S4.2   QR solve, P:327-328     : H = QR, z = Q^T Y, R beta = z
 * Paper-literal per-cell variants (readings R9/R10):
 *   LSTM / GRU with DIAGONAL recurrent weights u_g[j] (the only
 *   structure consistent with Alg. 2's cell independence), and FC by the
 *   letter of Eq. 8: own history scaled by
 *   sum_l alpha[j,l,k].
 *
 * Readings R1..R25 are listed in DESIGN.md.  Everything is computed in fp64
 * from fp32 inputs and fp32 (or grid-rounded) weights widened exactly.
 * Compile with -O2 -ffp-contract=off so no FMA contraction changes rounding.
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py
 * (closed forms, library reductions, brute force).  None is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { ARCH_ELMAN = 0, ARCH_JORDAN, ARCH_NARMAX, ARCH_FC, ARCH_LSTM, ARCH_GRU,
       ARCH_LSTM_DIAG, ARCH_GRU_DIAG, ARCH_FC_EQ8 };

/* ------------------------------------------------------------------------ */
/* Weights: counter-based generator (reading R1/R2).    */
/* "Randomly assign W, alpha, b" -- Alg. 1 line 1; distribution       */
/* unstated -> U[-1,1) scaled per block.                              */
/* ------------------------------------------------------------------------ */
static uint64_t orc_splitmix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* nearest-even fp16-representable value of an fp32 value (|f| < 65504). */
static float orc_round_fp16(float f) {
    double a = fabs((double)f);
    if (a == 0.0) return f;
    int e;
    frexp(a, &e);                 /* a = m * 2^e, m in [0.5,1) -> exponent of leading bit is e-1 */
    int lead = e - 1;
    if (lead < -14) lead = -14;   /* fp16 subnormal spacing 2^-24 */
    double ulp = ldexp(1.0, lead - 10);
    double q = (double)f / ulp;
    double r = nearbyint(q);      /* default rounding mode: nearest-even */
    return (float)(r * ulp);
}

/* tf32 (10 explicit mantissa bits), round-half-away (RNA), of an fp32 value. */
static float orc_round_tf32(float f) {
    double a = fabs((double)f);
    if (a == 0.0) return f;
    int e;
    frexp(a, &e);
    int lead = e - 1;
    if (lead < -126) lead = -126;
    double ulp = ldexp(1.0, lead - 10);
    double q = a / ulp;
    double r = floor(q + 0.5);
    double v = r * ulp;
    return (float)(f < 0 ? -v : v);
}

/* Number of weight blocks and each block's logical element count and scale.
 * Returns element count, or -1 when block_id is out of range.  The block map
 * is the one tabulated in DESIGN.md "Weights". */
static int64_t orc_block_info(int arch, int S, int M, int Q, int F, int R, int fc_lags,
                              int rec_scale, int block_id, double* scale, int* is_mma) {
    *scale = 1.0;
    *is_mma = 0;
    int unit = (rec_scale == 1);
    switch (arch) {
    case ARCH_ELMAN:
    case ARCH_JORDAN:
        if (block_id == 0) return (int64_t)S * M;
        if (block_id == 1) return M;
        if (block_id == 2) {
            if (arch == ARCH_ELMAN && !unit) *scale = 1.0 / sqrt((double)Q);
            return (int64_t)M * Q;
        }
        return -1;
    case ARCH_NARMAX:
        if (block_id == 0) return (int64_t)S * M;
        if (block_id == 1) return M;
        if (block_id == 2) return (int64_t)M * F;
        if (block_id == 3) return (int64_t)M * R;
        return -1;
    case ARCH_FC_EQ8:   /* same blocks as FC; alpha[j,l,k] = A[k-1][l][j]; no MMA */
        if (block_id == 0) return (int64_t)S * M;
        if (block_id == 1) return M;
        if (block_id == 2) {
            if (!unit) *scale = 1.0 / sqrt((double)M * (double)fc_lags);
            return (int64_t)fc_lags * M * M;
        }
        return -1;
    case ARCH_LSTM_DIAG:
    case ARCH_GRU_DIAG: {   /* per gate: W_g [S][M], u_g [M] (diagonal, fan-in 1), b_g [M] */
        int G = (arch == ARCH_LSTM_DIAG) ? 4 : 3;
        if (block_id < 0 || block_id >= 3 * G) return -1;
        return (block_id % 3 == 0) ? (int64_t)S * M : M;
    }
    case ARCH_FC:
        if (block_id == 0) return (int64_t)S * M;
        if (block_id == 1) return M;
        if (block_id == 2) {
            if (!unit) *scale = 1.0 / sqrt((double)M * (double)fc_lags);
            *is_mma = 1;
            return (int64_t)fc_lags * M * M;
        }
        return -1;
    case ARCH_LSTM:
    case ARCH_GRU: {
        int G = (arch == ARCH_LSTM) ? 4 : 3;
        if (block_id < 0 || block_id >= 3 * G) return -1;
        int kind = block_id % 3;
        if (kind == 0) return (int64_t)S * M;
        if (kind == 1) {
            if (!unit) *scale = 1.0 / sqrt((double)M);
            *is_mma = 1;
            return (int64_t)M * M;
        }
        return M;
    }
    }
    return -1;
}

/* exported for the generator's known-answer test */
uint64_t orc_rng_u64(uint64_t z) { return orc_splitmix64(z); }

int orc_num_blocks(int arch) {
    switch (arch) {
    case ARCH_ELMAN: case ARCH_JORDAN: case ARCH_FC: case ARCH_FC_EQ8: return 3;
    case ARCH_NARMAX: return 4;
    case ARCH_LSTM: case ARCH_LSTM_DIAG: return 12;
    case ARCH_GRU: case ARCH_GRU_DIAG: return 9;
    }
    return -1;
}

int64_t orc_block_len(int arch, int S, int M, int Q, int F, int R, int fc_lags, int block_id) {
    double sc; int mm;
    return orc_block_info(arch, S, M, Q, F, R, fc_lags, 0, block_id, &sc, &mm);
}

/* Generate one logical weight block as fp32 values (weight_grid 0 = fp32,
 * 1 = fp16-representable, 2 = tf32-representable; grid applies to MMA blocks). */
int orc_gen_block(int arch, int S, int M, int Q, int F, int R, int fc_lags, int rec_scale,
                  int weight_grid, uint64_t seed, int block_id, float* out) {
    double scale; int is_mma;
    int64_t n = orc_block_info(arch, S, M, Q, F, R, fc_lags, rec_scale, block_id, &scale, &is_mma);
    if (n < 0) return -1;
    uint64_t key = orc_splitmix64(seed ^ (0xD1B54A32D192ED03ULL * (uint64_t)(block_id + 1)));
    for (int64_t idx = 0; idx < n; ++idx) {
        uint64_t r = orc_splitmix64(key + (uint64_t)idx);
        double u = (double)(r >> 11) * 0x1p-53;
        double w = (2.0 * u - 1.0) * scale;
        float f = (float)w;
        if (is_mma && weight_grid == 1) f = orc_round_fp16(f);
        if (is_mma && weight_grid == 2) f = orc_round_tf32(f);
        out[idx] = f;
    }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Activations (reading R3): sigma for g and all gates, tanh for g_c, g_f.   */
/* ------------------------------------------------------------------------ */
static double orc_sigmoid(double a) {
    if (a >= 0) return 1.0 / (1.0 + exp(-a));
    double e = exp(a);
    return e / (1.0 + e);
}
static double orc_g(double a, int act) { return act == 1 ? tanh(a) : orc_sigmoid(a); }

/* ------------------------------------------------------------------------ */
/* H build.  Weights are passed as an array of block pointers (fp32, logical */
/* layouts of DESIGN.md "Weights").  X fp32 [N][Q][S] with row stride ldx.   */
/* Yfb fp32 [N][Q] (row stride ldy) or NULL -> y_i(tau) = X[i][tau][0].      */
/* H out fp64 [N][M].  Zero history: h, c, y = 0 for tau <= 0 (R13).         */
/* ------------------------------------------------------------------------ */
typedef struct {
    int arch, S, M, Q, F, R, act, fc_lags;
    const float* const* blk;
} orc_net;

/* teacher signal y_i(tau), 1-based tau (reading R7) */
static double orc_y(const float* Xi, const float* Yi, int S, int tau) {
    if (tau <= 0) return 0.0;
    if (Yi) return (double)Yi[tau - 1];
    return (double)Xi[(int64_t)tau * S + 0];
}

/* W.x(t) + b for neuron j; x(t) is X[i][t-1][:] (1-based t) */
static double orc_wx_b(const float* W, const float* b, const float* Xi, int S, int M, int t, int j) {
    double a = 0.0;
    for (int s = 0; s < S; ++s) a += (double)W[(int64_t)s * M + j] * (double)Xi[(int64_t)(t - 1) * S + s];
    return a + (double)b[j];
}

/* Eq. 5 (Elman): a_j(t) = W[:,j].x(t) + b_j + sum_{k=1}^{t-1} alpha[j,k] h_j(t-k) */
static void orc_row_elman(const orc_net* n, const float* Xi, double* hist /*[Q+1]*/, double* Hrow) {
    const float *W = n->blk[0], *b = n->blk[1], *al = n->blk[2];
    for (int j = 0; j < n->M; ++j) {
        hist[0] = 0.0;
        for (int t = 1; t <= n->Q; ++t) {
            double a = orc_wx_b(W, b, Xi, n->S, n->M, t, j);
            for (int k = 1; k <= t - 1; ++k) a += (double)al[(int64_t)j * n->Q + (k - 1)] * hist[t - k];
            hist[t] = orc_g(a, n->act);
        }
        Hrow[j] = hist[n->Q];
    }
}

/* Eq. 6 (Jordan) / Eq. 7 (NARMAX) under teacher forcing: full t-loop.
 * The feedback terms read the teacher signal, never h, so h_j(Q) depends
 * only on step Q (collapse identity; asserted by tests). */
/* e(tau) of reading R30: Ei[tau-1] when an error window is given, else 0 (R8);
 * e(tau <= 0) = 0 like y (R13). */
static double orc_e(const float* Ei, int tau) {
    if (tau <= 0 || !Ei) return 0.0;
    return (double)Ei[tau - 1];
}
static double orc_tf_step(const orc_net* n, const float* Xi, const float* Yi, const float* Ei, int t, int j) {
    double a = orc_wx_b(n->blk[0], n->blk[1], Xi, n->S, n->M, t, j);
    if (n->arch == ARCH_JORDAN) {
        const float* al = n->blk[2];
        for (int k = 1; k <= n->Q; ++k) a += (double)al[(int64_t)j * n->Q + (k - 1)] * orc_y(Xi, Yi, n->S, t - k);
    } else {
        const float *W1 = n->blk[2], *W2 = n->blk[3];
        for (int l = 1; l <= n->F; ++l) a += (double)W1[(int64_t)j * n->F + (l - 1)] * orc_y(Xi, Yi, n->S, t - l);
        for (int l = 1; l <= n->R; ++l) a += (double)W2[(int64_t)j * n->R + (l - 1)] * orc_e(Ei, t - l);
    }
    return orc_g(a, n->act);
}
static void orc_row_tf(const orc_net* n, const float* Xi, const float* Yi, const float* Ei, double* Hrow) {
    for (int j = 0; j < n->M; ++j) {
        double h = 0.0;
        for (int t = 1; t <= n->Q; ++t) h = orc_tf_step(n, Xi, Yi, Ei, t, j);
        Hrow[j] = h;
    }
}

/* S2.2.4 prose (R9): a_j(t) = W.x(t) + b_j + sum_{k=1}^{min(t-1,L)} sum_m A_k[m][j] h_m(t-k) */
static void orc_row_fc(const orc_net* n, const float* Xi, double* hist /*[(Q+1)*M]*/, double* Hrow) {
    const float *W = n->blk[0], *b = n->blk[1], *A = n->blk[2];
    int M = n->M, L = n->fc_lags;
    for (int j = 0; j < M; ++j) hist[j] = 0.0;
    for (int t = 1; t <= n->Q; ++t) {
        for (int j = 0; j < M; ++j) {
            double a = orc_wx_b(W, b, Xi, n->S, M, t, j);
            for (int k = 1; k <= t - 1 && k <= L; ++k)
                for (int m = 0; m < M; ++m)
                    a += (double)A[((int64_t)(k - 1) * M + m) * M + j] * hist[(int64_t)(t - k) * M + m];
            hist[(int64_t)t * M + j] = orc_g(a, n->act);
        }
    }
    for (int j = 0; j < M; ++j) Hrow[j] = hist[(int64_t)n->Q * M + j];
}

/* S2.2.5 (LSTM), dense U (R10): gates (o, c, lambda, in) = 0..3.
 *   a_g = x(t) W_g + h(t-1) U_g + b_g
 *   c(t) = sigma(a_lambda) c(t-1) + sigma(a_in) tanh(a_c);  h(t) = sigma(a_o) tanh(c(t)) */
static void orc_row_lstm(const orc_net* n, const float* Xi, double* work /*[6M]*/, double* Hrow) {
    int M = n->M;
    double *h = work, *c = work + M, *a = work + 2 * M; /* a: 4M */
    for (int j = 0; j < M; ++j) { h[j] = 0.0; c[j] = 0.0; }
    for (int t = 1; t <= n->Q; ++t) {
        for (int g = 0; g < 4; ++g) {
            const float *W = n->blk[3 * g], *U = n->blk[3 * g + 1], *b = n->blk[3 * g + 2];
            for (int j = 0; j < M; ++j) {
                double s = orc_wx_b(W, b, Xi, n->S, M, t, j);
                for (int m = 0; m < M; ++m) s += h[m] * (double)U[(int64_t)m * M + j];
                a[(int64_t)g * M + j] = s;
            }
        }
        for (int j = 0; j < M; ++j) {
            double o = orc_sigmoid(a[0 * M + j]);
            double cc = tanh(a[1 * M + j]);
            double lam = orc_sigmoid(a[2 * M + j]);
            double in = orc_sigmoid(a[3 * M + j]);
            c[j] = lam * c[j] + in * cc;
            h[j] = o * tanh(c[j]);
        }
    }
    for (int j = 0; j < M; ++j) Hrow[j] = h[j];
}

/* S2.2.6 (GRU), Cho form with dense U (R11, R12): gates (z, r, f).
 *   z = sigma(x W_z + h U_z + b_z);  r = sigma(x W_r + h U_r + b_r)
 *   n = tanh(x W_f + (r o h) U_f + b_f);  h(t) = (1 - z) o h(t-1) + z o n */
static void orc_row_gru(const orc_net* n, const float* Xi, double* work /*[5M]*/, double* Hrow) {
    int M = n->M;
    double *h = work, *z = work + M, *r = work + 2 * M, *rh = work + 3 * M, *nn = work + 4 * M;
    for (int j = 0; j < M; ++j) h[j] = 0.0;
    for (int t = 1; t <= n->Q; ++t) {
        for (int j = 0; j < M; ++j) {
            double sz = orc_wx_b(n->blk[0], n->blk[2], Xi, n->S, M, t, j);
            double sr = orc_wx_b(n->blk[3], n->blk[5], Xi, n->S, M, t, j);
            for (int m = 0; m < M; ++m) {
                sz += h[m] * (double)n->blk[1][(int64_t)m * M + j];
                sr += h[m] * (double)n->blk[4][(int64_t)m * M + j];
            }
            z[j] = orc_sigmoid(sz);
            r[j] = orc_sigmoid(sr);
        }
        for (int m = 0; m < M; ++m) rh[m] = r[m] * h[m];
        for (int j = 0; j < M; ++j) {
            double s = orc_wx_b(n->blk[6], n->blk[8], Xi, n->S, M, t, j);
            for (int m = 0; m < M; ++m) s += rh[m] * (double)n->blk[7][(int64_t)m * M + j];
            nn[j] = tanh(s);
        }
        for (int j = 0; j < M; ++j) h[j] = (1.0 - z[j]) * h[j] + z[j] * nn[j];
    }
    for (int j = 0; j < M; ++j) Hrow[j] = h[j];
}

/* Eq. 8 by the letter:
 *   a_j(t) = W[:,j].x(t) + b_j + sum_{k=1}^{min(t-1,L)} sum_{l=1}^{M} alpha[j,l,k] h_j(t-k)
 * with alpha[j,l,k] = A[k-1][l][j] (the FC block).  Cell independent. */
static void orc_row_fc_eq8(const orc_net* n, const float* Xi, double* hist /*[Q+1]*/, double* Hrow) {
    const float *W = n->blk[0], *b = n->blk[1], *A = n->blk[2];
    int M = n->M, L = n->fc_lags;
    for (int j = 0; j < M; ++j) {
        hist[0] = 0.0;
        for (int t = 1; t <= n->Q; ++t) {
            double a = orc_wx_b(W, b, Xi, n->S, M, t, j);
            for (int k = 1; k <= t - 1 && k <= L; ++k)
                for (int l = 0; l < M; ++l) a += (double)A[((int64_t)(k - 1) * M + l) * M + j] * hist[t - k];
            hist[t] = orc_g(a, n->act);
        }
        Hrow[j] = hist[n->Q];
    }
}

/* LSTM with diagonal recurrent weights: per neuron j, gates
 * (o, c, lambda, in) = 0..3, a_g = W_g[:,j].x(t) + u_g[j] h_j(t-1) + b_g[j];
 * c = sigma(a_lambda) c + sigma(a_in) tanh(a_c);  h = sigma(a_o) tanh(c). */
static void orc_row_lstm_diag(const orc_net* n, const float* Xi, double* Hrow) {
    for (int j = 0; j < n->M; ++j) {
        double h = 0.0, c = 0.0;
        for (int t = 1; t <= n->Q; ++t) {
            double a[4];
            for (int g = 0; g < 4; ++g)
                a[g] = orc_wx_b(n->blk[3 * g], n->blk[3 * g + 2], Xi, n->S, n->M, t, j) +
                       (double)n->blk[3 * g + 1][j] * h;
            c = orc_sigmoid(a[2]) * c + orc_sigmoid(a[3]) * tanh(a[1]);
            h = orc_sigmoid(a[0]) * tanh(c);
        }
        Hrow[j] = h;
    }
}

/* GRU (Cho form, R11/R12) with diagonal recurrent weights: gates (z, r, f),
 *   z = sigma(W_z x + u_z h + b_z), r = sigma(W_r x + u_r h + b_r),
 *   n = tanh(W_f x + u_f (r h) + b_f), h = (1 - z) h + z n. */
static void orc_row_gru_diag(const orc_net* n, const float* Xi, double* Hrow) {
    for (int j = 0; j < n->M; ++j) {
        double h = 0.0;
        for (int t = 1; t <= n->Q; ++t) {
            double z = orc_sigmoid(orc_wx_b(n->blk[0], n->blk[2], Xi, n->S, n->M, t, j) + (double)n->blk[1][j] * h);
            double r = orc_sigmoid(orc_wx_b(n->blk[3], n->blk[5], Xi, n->S, n->M, t, j) + (double)n->blk[4][j] * h);
            double nn = tanh(orc_wx_b(n->blk[6], n->blk[8], Xi, n->S, n->M, t, j) + (double)n->blk[7][j] * (r * h));
            h = (1.0 - z) * h + z * nn;
        }
        Hrow[j] = h;
    }
}

/* Alg. 1 line 2: H(Q) for every sample row; rows are independent
 * (the parallel decomposition of P:250), so an OpenMP row split gives
 * bitwise-identical results for any thread count. */
int orc_build_H_ef(int arch, int S, int M, int Q, int F, int R, int act, int fc_lags,
                   const float* const* blocks, const float* X, int64_t ldx,
                   const float* Yfb, int64_t ldy, const float* Efb, int64_t lde,
                   int64_t N, double* H, int64_t ldh, int threads) {
    if (arch < 0 || arch > ARCH_FC_EQ8 || S < 1 || M < 1 || Q < 1) return -1;
    orc_net net = { arch, S, M, Q, F, R, act, fc_lags, blocks };
    int64_t wlen = (int64_t)(Q + 1) * M + 8 * M + Q + 8;
#ifdef _OPENMP
    if (threads < 1) threads = 1;
#pragma omp parallel num_threads(threads)
#endif
    {
        double* work = (double*)malloc(sizeof(double) * wlen);
#ifdef _OPENMP
#pragma omp for schedule(static)
#endif
        for (int64_t i = 0; i < N; ++i) {
            const float* Xi = X + i * ldx;
            const float* Yi = Yfb ? Yfb + i * ldy : NULL;
            const float* Ei = (Efb && arch == ARCH_NARMAX) ? Efb + i * lde : NULL;
            double* Hrow = H + i * ldh;
            switch (arch) {
            case ARCH_ELMAN: orc_row_elman(&net, Xi, work, Hrow); break;
            case ARCH_JORDAN: case ARCH_NARMAX: orc_row_tf(&net, Xi, Yi, Ei, Hrow); break;
            case ARCH_FC: orc_row_fc(&net, Xi, work, Hrow); break;
            case ARCH_LSTM: orc_row_lstm(&net, Xi, work, Hrow); break;
            case ARCH_GRU: orc_row_gru(&net, Xi, work, Hrow); break;
            case ARCH_LSTM_DIAG: orc_row_lstm_diag(&net, Xi, Hrow); break;
            case ARCH_GRU_DIAG: orc_row_gru_diag(&net, Xi, Hrow); break;
            case ARCH_FC_EQ8: orc_row_fc_eq8(&net, Xi, work, Hrow); break;
            }
        }
        free(work);
    }
    return 0;
}

int orc_build_H(int arch, int S, int M, int Q, int F, int R, int act, int fc_lags,
                const float* const* blocks, const float* X, int64_t ldx,
                const float* Yfb, int64_t ldy, int64_t N, double* H, int64_t ldh, int threads) {
    return orc_build_H_ef(arch, S, M, Q, F, R, act, fc_lags, blocks, X, ldx, Yfb, ldy, NULL, 0, N, H, ldh, threads);
}

/* NARMAX error feedback (Eq. 7, "e(t) = y(t) - yhat(t)" P:122;
 * SURVEY 8(f) row 4; reading R30).  Rows are the consecutive stride-1 windows
 * of one series (R22): window i's output y(tau) is the target of window
 * k = i + tau - Q, so
 *     e_i(tau) = Y[k] - yhat[k],  yhat[k] = sum_j H[k][j] beta[j]  (Eq. 4),
 * and e_i(tau) = 0 when k < 0 (before the first window, like R13).
 * Ef[i][tau-1] holds e_i(tau) for tau = 1..Q, stored as fp32 (the GPU's
 * input type), rounded once from fp64. */
void orc_error_windows(const double* H, int64_t ldh, const double* Y, int64_t N, int M, int Q,
                       const double* beta, float* Ef, int64_t lde) {
    for (int64_t i = 0; i < N; ++i) {
        for (int tau = 1; tau <= Q; ++tau) {
            int64_t k = i + tau - Q;
            double e = 0.0;
            if (k >= 0) {
                double yhat = 0.0;
                for (int j = 0; j < M; ++j) yhat += H[k * ldh + j] * beta[j];
                e = Y[k] - yhat;
            }
            Ef[i * lde + (tau - 1)] = (float)e;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Least squares by unblocked Householder QR (S4.2; R18-R20).      */
/* A = [H | Y] (N x (M+1)) fp64, LAPACK dlarfg convention, sign(0) = +1.      */
/* ------------------------------------------------------------------------ */
typedef struct {
    double rho, rmse, rdiag_min_abs, rdiag_max_abs, ridge_lambda;
    int rank_flag;
    int64_t n_total;
} orc_info;

/* In-place Householder QR of A (m x n, row-major, lda).  On return the upper
 * triangle of A[0:min(m,n), :] holds R. */
/* Threads for the column updates of orc_householder (default 1).  Each column
 * j's update is computed by one thread in the same order for any thread count,
 * so the result is bitwise identical. */
static int g_qr_threads = 1;
void orc_set_qr_threads(int t) { g_qr_threads = t < 1 ? 1 : t; }

static void orc_householder(double* A, int64_t m, int n, int64_t lda) {
    /* A is stored COLUMN-major: element (i, j) at A[j * lda + i] (lda >= m),
     * so every loop over i below is a contiguous sweep. */
#define AE(i, j) A[(int64_t)(j) * lda + (i)]
    for (int k = 0; k < n && k < m; ++k) {
        double x0 = AE(k, k);
        double sigma2 = 0.0;
        for (int64_t i = k + 1; i < m; ++i) sigma2 += AE(i, k) * AE(i, k);
        double sigma = sqrt(sigma2);
        if (sigma == 0.0) continue;                      /* tau = 0, H = I */
        double beta = -(x0 >= 0 ? 1.0 : -1.0) * hypot(x0, sigma);
        double tau = (beta - x0) / beta;
        double inv = 1.0 / (x0 - beta);
        for (int64_t i = k + 1; i < m; ++i) AE(i, k) *= inv;  /* v (v0 = 1 implicit) */
        AE(k, k) = beta;
#ifdef _OPENMP
#pragma omp parallel for schedule(static) num_threads(g_qr_threads) if (g_qr_threads > 1 && (m - k) * (int64_t)(n - k) > 65536)
#endif
        for (int j = k + 1; j < n; ++j) {
            double w = AE(k, j);
            for (int64_t i = k + 1; i < m; ++i) w += AE(i, k) * AE(i, j);
            AE(k, j) -= tau * w;
            for (int64_t i = k + 1; i < m; ++i) AE(i, j) -= tau * AE(i, k) * w;
        }
        for (int64_t i = k + 1; i < m; ++i) AE(i, k) = 0.0;
    }
#undef AE
}

/* Solve from the (M+1)x(M+1) upper-triangular R of [H|Y] (row-major, full
 * storage).  Sign-normalises R in place, rank check, ridge fallback by an
 * appended sqrt(lambda)(I|0) block (R19), back substitution, rho, rmse.
 * Returns 0 ok, 1 ridge used. */
int orc_solve_from_R(double* Rf, int M, int64_t n_total, double* beta, orc_info* info) {
    int n = M + 1;
    for (int k = 0; k < n; ++k)
        if (Rf[(int64_t)k * n + k] < 0)
            for (int j = k; j < n; ++j) Rf[(int64_t)k * n + j] = -Rf[(int64_t)k * n + j];
    double dmin = INFINITY, dmax = 0.0, fro2 = 0.0;
    for (int k = 0; k < M; ++k) {
        double d = fabs(Rf[(int64_t)k * n + k]);
        if (d < dmin) dmin = d;
        if (d > dmax) dmax = d;
        for (int j = k; j < M; ++j) fro2 += Rf[(int64_t)k * n + j] * Rf[(int64_t)k * n + j];
    }
    int ridge = (dmin <= DBL_EPSILON * (double)M * dmax);
    double lambda = 0.0;
    double* Rs = Rf;
    double* big = NULL;
    if (ridge) {
        lambda = 1e-8 * fro2 / (double)M;
        double sl = sqrt(lambda);
        /* [R[:M, :]; sqrt(lambda) (I | 0)], 2M x n, column-major for orc_householder */
        double* cm = (double*)calloc((size_t)(2 * M) * n, sizeof(double));
        for (int k = 0; k < M; ++k)
            for (int j = 0; j < n; ++j) cm[(int64_t)j * (2 * M) + k] = Rf[(int64_t)k * n + j];
        for (int k = 0; k < M; ++k) cm[(int64_t)k * (2 * M) + M + k] = sl;
        orc_householder(cm, 2 * M, n, 2 * M);
        big = (double*)calloc((size_t)M * n, sizeof(double));   /* its R, row-major */
        for (int k = 0; k < M; ++k)
            for (int j = k; j < n; ++j) big[(int64_t)k * n + j] = cm[(int64_t)j * (2 * M) + k];
        free(cm);
        for (int k = 0; k < M; ++k)
            if (big[(int64_t)k * n + k] < 0)
                for (int j = k; j < n; ++j) big[(int64_t)k * n + j] = -big[(int64_t)k * n + j];
        Rs = big;
    }
    for (int k = M - 1; k >= 0; --k) {
        double s = Rs[(int64_t)k * n + M];
        for (int j = k + 1; j < M; ++j) s -= Rs[(int64_t)k * n + j] * beta[j];
        beta[k] = s / Rs[(int64_t)k * n + k];
    }
    /* rho = || R_aug [beta; -1] || = || H beta - Y ||  (exact identity) */
    double rho2 = 0.0;
    for (int k = 0; k < n; ++k) {
        double s = 0.0;
        for (int j = k; j < M; ++j) s += Rf[(int64_t)k * n + j] * beta[j];
        s -= Rf[(int64_t)k * n + M];
        rho2 += s * s;
    }
    if (info) {
        info->rho = sqrt(rho2);
        info->rmse = sqrt(rho2) / sqrt((double)n_total);
        info->rdiag_min_abs = dmin;
        info->rdiag_max_abs = dmax;
        info->ridge_lambda = lambda;
        info->rank_flag = ridge;
        info->n_total = n_total;
    }
    free(big);
    return ridge;
}

/* beta = argmin || H beta - Y ||_2 for H fp64 [N][M] (ldh), Y fp64.
 * Returns 0 ok, 1 ridge, -3 underdetermined (N < M), -4 nonfinite.  When
 * N == M the bottom row of R (rho) is zero.  Rout (optional)
 * receives the sign-normalised (M+1)x(M+1) R of [H|Y] (full storage). */
int orc_lstsq(const double* H, int64_t ldh, const double* Y, int64_t N, int M,
              double* beta, orc_info* info, double* Rout) {
    int n = M + 1;
    if (N < M || M < 1) return -3;
    double* A = (double*)malloc(sizeof(double) * (size_t)N * n);   /* [H | Y], column-major */
    for (int64_t i = 0; i < N; ++i) {
        for (int j = 0; j < M; ++j) {
            double v = H[i * ldh + j];
            if (!isfinite(v)) { free(A); return -4; }
            A[(int64_t)j * N + i] = v;
        }
        if (!isfinite(Y[i])) { free(A); return -4; }
        A[(int64_t)M * N + i] = Y[i];
    }
    orc_householder(A, N, n, N);
    double* Rf = (double*)calloc((size_t)n * n, sizeof(double));
    for (int k = 0; k < n && k < N; ++k)
        for (int j = k; j < n; ++j) Rf[(int64_t)k * n + j] = A[(int64_t)j * N + k];
    free(A);
    int rc = orc_solve_from_R(Rf, M, N, beta, info);
    if (Rout) memcpy(Rout, Rf, sizeof(double) * (size_t)n * n);
    free(Rf);
    return rc;
}

/* Eq. 4: yhat_i = sum_j beta_j H[i][j] (no output bias, R16). */
void orc_predict(const double* H, int64_t ldh, int64_t N, int M, const double* beta, double* yhat) {
    for (int64_t i = 0; i < N; ++i) {
        double s = 0.0;
        for (int j = 0; j < M; ++j) s += H[i * ldh + j] * beta[j];
        yhat[i] = s;
    }
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
