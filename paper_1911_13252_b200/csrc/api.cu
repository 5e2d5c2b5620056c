// api.cu -- the C ABI of include/elmrnn.h: validation, dispatch, workspace.
// Every arithmetic step is a kernel of this library; there is no host or
// library fallback.  Citations "P:n" = PAPER.md line n.
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>
#include <cmath>
#include <cstdlib>

#include "common.cuh"

using namespace elm;

static thread_local std::string g_init_error;

static elmrnn_status fail(elmrnn* h, elmrnn_status st, const std::string& msg) {
    if (h) h->err = msg; else g_init_error = msg;
    return st;
}

static elmrnn_status cuda_fail(elmrnn* h, cudaError_t e, const char* where) {
    std::string m = std::string(where) + ": " + cudaGetErrorString(e);
    return fail(h, e == cudaErrorMemoryAllocation ? ELMRNN_ERR_OOM : ELMRNN_ERR_CUDA, m);
}

extern "C" {

void elmrnn_opts_default(elmrnn_opts* o) {
    if (!o) return;
    o->F = -1; o->R = -1; o->act = 0; o->rec_scale = 0; o->weight_grid = 0; o->fc_lags = -1; o->force_path = 0; o->fused_train = 0;
}

elmrnn_status elmrnn_init(elmrnn_t* out, int arch, int d, int M, int Q, uint64_t seed) {
    return elmrnn_init_ex(out, arch, d, M, Q, seed, nullptr);
}

elmrnn_status elmrnn_init_ex(elmrnn_t* out, int arch, int d, int M, int Q, uint64_t seed, const elmrnn_opts* opts) {
    if (!out) return fail(nullptr, ELMRNN_ERR_ARG, "out is NULL");
    *out = nullptr;
    elmrnn_opts o;
    elmrnn_opts_default(&o);
    if (opts) o = *opts;
    if (arch < ELMRNN_ELMAN || arch > ELMRNN_FC_EQ8) return fail(nullptr, ELMRNN_ERR_ARG, "arch out of range");
    if (d < 1 || M < 1 || Q < 1) return fail(nullptr, ELMRNN_ERR_ARG, "d, M and Q must be >= 1");
    if (o.F < 0) o.F = Q;
    if (o.R < 0) o.R = Q;
    if (o.fc_lags < 0) o.fc_lags = Q;
    if (o.act < 0 || o.act > 1 || o.rec_scale < 0 || o.rec_scale > 1 || o.weight_grid < 0 || o.weight_grid > 2 ||
        o.force_path < 0 || o.force_path > 2 || o.fc_lags < 1 || o.fused_train < 0 || o.fused_train > 1)
        return fail(nullptr, ELMRNN_ERR_ARG, "invalid option value");
    if ((arch == ELMRNN_ELMAN || arch == ELMRNN_FC_EQ8) && !elman_supported(Q))
        return fail(nullptr, ELMRNN_ERR_UNSUPPORTED, "Elman supports Q <= 128");
    if (M > 1024) return fail(nullptr, ELMRNN_ERR_UNSUPPORTED, "M <= 1024 (the widest BASELINE config, C5)");

    elmrnn* h = new (std::nothrow) elmrnn();
    if (!h) return fail(nullptr, ELMRNN_ERR_OOM, "host allocation failed");
    h->arch = arch; h->S = d; h->M = M; h->Q = Q; h->F = o.F; h->R = o.R; h->act = o.act;
    h->fc_lags = o.fc_lags; h->rec_scale = o.rec_scale; h->weight_grid = o.weight_grid;
    h->force_path = o.force_path; h->fused_train = o.fused_train; h->seed = seed; h->G = gates_of(arch); h->stream = nullptr;
    h->path = 1;
    h->nrhs = 1;
    if (const char* t = std::getenv("ELMRNN_TESTING"); t && std::atoi(t) == 1) {   // test overrides, read once
        if (const char* e = std::getenv("ELMRNN_TSQR_WY")) h->tune.tsqr_wy = std::atoi(e);
        if (const char* e = std::getenv("ELMRNN_TSQR_WY_ROWS")) h->tune.wy_rows = std::atoi(e);
        if (const char* e = std::getenv("ELMRNN_PW_MODE")) h->tune.pw_mode = std::atoi(e);
        if (const char* e = std::getenv("ELMRNN_WY_NW")) h->tune.wy_nw = std::atoi(e);
        if (const char* e = std::getenv("ELMRNN_TSQR_MAXSLABS")) h->tune.max_slabs = std::atoi(e);
        if (const char* e = std::getenv("ELMRNN_WY_2PHASE")) h->tune.wy_2phase = std::atoi(e);
        if (const char* e = std::getenv("ELMRNN_MERGE_SMALL")) h->tune.merge_small = std::atoi(e);
        if (const char* e = std::getenv("ELMRNN_WIDE_PAIR")) h->tune.wide_pair = std::atoi(e);
    }
    cudaError_t e;
    if ((e = cudaGetDevice(&h->device))) { elmrnn_destroy(h); return cuda_fail(nullptr, e, "cudaGetDevice"); }
    if ((e = cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->device))) {
        elmrnn_destroy(h);
        return cuda_fail(nullptr, e, "cudaDeviceGetAttribute");
    }
    const int64_t GM = (int64_t)h->G * M;
    switch (arch) {
    case ELMRNN_ELMAN: case ELMRNN_JORDAN: h->rec_len = (int64_t)Q * M; break;
    case ELMRNN_NARMAX: h->rec_len = (int64_t)(o.F + o.R > 0 ? o.F + o.R : 1) * M; break;
    case ELMRNN_FC: h->rec_len = (int64_t)o.fc_lags * M * M; break;
    case ELMRNN_FC_EQ8: h->rec_len = (int64_t)Q * M; break;
    case ELMRNN_LSTM_DIAG: case ELMRNN_GRU_DIAG: h->rec_len = GM; break;
    default: h->rec_len = (int64_t)M * GM; break;
    }
    if ((e = cudaMalloc(&h->W, sizeof(float) * d * GM)) || (e = cudaMalloc(&h->b, sizeof(float) * GM)) ||
        (e = cudaMalloc(&h->rec, sizeof(float) * h->rec_len))) {
        elmrnn_destroy(h);
        return cuda_fail(nullptr, e, "weight allocation");
    }
    if ((e = gen_weights(h))) { elmrnn_destroy(h); return cuda_fail(nullptr, e, "gen_weights"); }
    // H-builder choice: tensor cores when the recurrence is a real dense
    // contraction, else FP32 FMA.
    if ((arch == ELMRNN_LSTM || arch == ELMRNN_GRU || arch == ELMRNN_FC) && o.force_path != 1 && tc_supported(h) &&
        (o.force_path == 2 || M >= 128)) {
        if ((e = tc_prepare(h))) { elmrnn_destroy(h); return cuda_fail(nullptr, e, "tc_prepare"); }
        h->path = 2;
    } else if (o.force_path == 2) {
        elmrnn_destroy(h);
        return fail(nullptr, ELMRNN_ERR_UNSUPPORTED, "tensor-core path not available for this shape");
    }
    if ((e = cudaStreamSynchronize(h->stream))) { elmrnn_destroy(h); return cuda_fail(nullptr, e, "init sync"); }
    *out = h;
    return ELMRNN_OK;
}

elmrnn_status elmrnn_set_stream(elmrnn_t h, void* s) {
    if (!h) return ELMRNN_ERR_ARG;
    h->stream = reinterpret_cast<cudaStream_t>(s);
    return ELMRNN_OK;
}

static elmrnn_status build_impl(elmrnn* h, const float* X, int64_t ldx, const float* Yfb, int64_t ldy, int64_t N,
                                float* H, int64_t ldh, const float* Ef = nullptr, int64_t lde = 0) {
    cudaError_t e;
    switch (h->arch) {
    case ELMRNN_ELMAN: case ELMRNN_FC_EQ8: e = launch_elman(h, X, ldx, N, H, ldh); break;
    case ELMRNN_LSTM_DIAG: case ELMRNN_GRU_DIAG: e = launch_diag_gated(h, X, ldx, N, H, ldh); break;
    case ELMRNN_JORDAN: case ELMRNN_NARMAX: e = launch_teacher_forced(h, X, ldx, Yfb, ldy, N, H, ldh, Ef, lde); break;
    default:
        e = h->path == 2 ? launch_dense_tc(h, X, ldx, N, H, ldh) : launch_dense_fma(h, X, ldx, N, H, ldh);
        if (e == cudaErrorInvalidConfiguration)
            return fail(h, ELMRNN_ERR_UNSUPPORTED, "recurrent state of one sample tile does not fit on chip");
        break;
    }
    if (e) return cuda_fail(h, e, "build_H");
    return ELMRNN_OK;
}

elmrnn_status elmrnn_build_H(elmrnn_t h, const float* X, int64_t ldx, const float* Yfb, int64_t ldy, int64_t N,
                             float* H, int64_t ldh) {
    if (!h) return ELMRNN_ERR_ARG;
    if (N < 0) return fail(h, ELMRNN_ERR_ARG, "N < 0");
    if (N == 0) return ELMRNN_OK;
    if (!X || !H) return fail(h, ELMRNN_ERR_ARG, "X or H is NULL");
    if (ldx < (int64_t)h->Q * h->S) return fail(h, ELMRNN_ERR_SHAPE, "ldx < Q*d");
    if (ldh < h->M) return fail(h, ELMRNN_ERR_SHAPE, "ldh < M");
    if (Yfb && ldy < h->Q) return fail(h, ELMRNN_ERR_SHAPE, "ldy < Q");
    if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(H)) & 3)
        return fail(h, ELMRNN_ERR_SHAPE, "pointers must be 4-byte aligned");
    return build_impl(h, X, ldx, Yfb, ldy, N, H, ldh);
}

elmrnn_status elmrnn_build_H_ef(elmrnn_t h, const float* X, int64_t ldx, const float* Yfb, int64_t ldy,
                                const float* Ef, int64_t lde, int64_t N, float* H, int64_t ldh) {
    if (!h) return ELMRNN_ERR_ARG;
    if (Ef && h->arch != ELMRNN_NARMAX) return fail(h, ELMRNN_ERR_ARG, "error feedback is a NARMAX input");
    if (Ef && lde < h->Q) return fail(h, ELMRNN_ERR_SHAPE, "lde < Q");
    if (Ef && (reinterpret_cast<uintptr_t>(Ef) & 3)) return fail(h, ELMRNN_ERR_SHAPE, "Ef must be 4-byte aligned");
    if (N < 0) return fail(h, ELMRNN_ERR_ARG, "N < 0");
    if (N == 0) return ELMRNN_OK;
    if (!X || !H) return fail(h, ELMRNN_ERR_ARG, "X or H is NULL");
    if (ldx < (int64_t)h->Q * h->S) return fail(h, ELMRNN_ERR_SHAPE, "ldx < Q*d");
    if (ldh < h->M) return fail(h, ELMRNN_ERR_SHAPE, "ldh < M");
    if (Yfb && ldy < h->Q) return fail(h, ELMRNN_ERR_SHAPE, "ldy < Q");
    if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(H)) & 3)
        return fail(h, ELMRNN_ERR_SHAPE, "pointers must be 4-byte aligned");
    return build_impl(h, X, ldx, Yfb, ldy, N, H, ldh, Ef, lde);
}

elmrnn_status elmrnn_error_windows(elmrnn_t h, const float* H, int64_t ldh, const float* Y, int64_t N,
                                   const double* beta, float* Ef, int64_t lde) {
    if (!h) return ELMRNN_ERR_ARG;
    if (N < 0) return fail(h, ELMRNN_ERR_ARG, "N < 0");
    if (N == 0) return ELMRNN_OK;
    if (!H || !Y || !beta || !Ef) return fail(h, ELMRNN_ERR_ARG, "NULL pointer");
    if (ldh < h->M) return fail(h, ELMRNN_ERR_SHAPE, "ldh < M");
    if (lde < h->Q) return fail(h, ELMRNN_ERR_SHAPE, "lde < Q");
    cudaError_t e;
    if (N > h->rws_rows) {
        if (h->rws) cudaFree(h->rws);
        h->rws = nullptr;
        h->rws_rows = 0;
        if ((e = cudaMalloc(&h->rws, sizeof(float) * N))) return cuda_fail(h, e, "error-window workspace");
        h->rws_rows = N;
    }
    if ((e = launch_error_windows(h, H, ldh, Y, N, beta, Ef, lde))) return cuda_fail(h, e, "error_windows");
    return ELMRNN_OK;
}

// Read the device diagnostics (synchronises the stream) and clear the sticky
// non-finite flag that asynchronous solves accumulate.
static cudaError_t read_solve_dev(elmrnn* h) {
    cudaError_t e;
    if ((e = cudaMemcpyAsync(h->shost, h->sdev, sizeof(SolveDev), cudaMemcpyDeviceToHost, h->stream)) ||
        (e = cudaMemsetAsync(&h->sdev->nf_sticky, 0, sizeof(int), h->stream)) ||
        (e = cudaStreamSynchronize(h->stream)))
        return e;
    return cudaSuccess;
}

static elmrnn_status finish_solve(elmrnn* h, elmrnn_solve_info* info) {
    cudaError_t e;
    if (!info) {
        if ((e = cudaGetLastError())) return cuda_fail(h, e, "solve");
        return ELMRNN_OK;
    }
    if ((e = read_solve_dev(h))) return cuda_fail(h, e, "solve");
    const SolveDev& s = *h->shost;
    info->rho = s.rho; info->rmse = s.rmse; info->rdiag_min_abs = s.dmin; info->rdiag_max_abs = s.dmax;
    info->ridge_lambda = s.lambda; info->rank_flag = s.rank_flag; info->n_total = s.n_total;
    if (s.nonfinite) return fail(h, ELMRNN_ERR_NONFINITE, "NaN or Inf in H or Y");
    return s.rank_flag ? ELMRNN_WARN_RIDGE : ELMRNN_OK;
}

elmrnn_status elmrnn_solve_beta(elmrnn_t h, const float* H, int64_t ldh, const float* Y, int64_t N, double* beta,
                                elmrnn_solve_info* info) {
    if (!h) return ELMRNN_ERR_ARG;
    if (!H || !Y || !beta) return fail(h, ELMRNN_ERR_ARG, "NULL pointer");
    if (ldh < h->M) return fail(h, ELMRNN_ERR_SHAPE, "ldh < M");
    if (N < h->M) return fail(h, ELMRNN_ERR_UNDERDETERMINED, "N < M");
    cudaError_t e;
    if ((e = tsqr_factor(h, H, ldh, Y, 1, N))) return cuda_fail(h, e, "tsqr_factor");
    if ((e = tsqr_solve(h, N, beta))) return cuda_fail(h, e, "tsqr_solve");
    return finish_solve(h, info);
}

elmrnn_status elmrnn_solve_beta_multi(elmrnn_t h, const float* H, int64_t ldh, const float* Y, int64_t ldy, int P,
                                      int64_t N, double* beta, double* rmse, elmrnn_solve_info* info) {
    if (!h) return ELMRNN_ERR_ARG;
    if (!H || !Y || !beta || P < 1) return fail(h, ELMRNN_ERR_ARG, "NULL pointer or P < 1");
    if (ldh < h->M) return fail(h, ELMRNN_ERR_SHAPE, "ldh < M");
    if (ldy < P) return fail(h, ELMRNN_ERR_SHAPE, "ldy < P");
    if (h->M + P > 1536) return fail(h, ELMRNN_ERR_UNSUPPORTED, "M + P <= 1536 (one 16-row WY tile in shared memory)");
    if (N < h->M) return fail(h, ELMRNN_ERR_UNDERDETERMINED, "N < M");
    cudaError_t e;
    if (P > h->rho_multi_len) {
        if (h->rho_multi) cudaFree(h->rho_multi);
        h->rho_multi = nullptr;
        h->rho_multi_len = 0;
        if ((e = cudaMalloc(&h->rho_multi, sizeof(double) * P))) return cuda_fail(h, e, "workspace");
        h->rho_multi_len = P;
    }
    struct Nrhs { elmrnn* h; ~Nrhs() { h->nrhs = 1; } } guard{h};
    h->nrhs = P;
    if ((e = tsqr_factor(h, H, ldh, Y, ldy, N))) return cuda_fail(h, e, "tsqr_factor");
    if ((e = tsqr_solve(h, N, beta))) return cuda_fail(h, e, "tsqr_solve");
    elmrnn_solve_info tmp;
    elmrnn_solve_info* ip = info ? info : (rmse ? &tmp : nullptr);
    const elmrnn_status st = finish_solve(h, ip);
    if (st < 0 || !rmse) return st;
    if (P == 1) {   // a single output may take the per-column-fold solve, which reports through info
        rmse[0] = ip->rmse;
        return st;
    }
    std::vector<double> rho(P);
    if ((e = cudaMemcpyAsync(rho.data(), h->rho_multi, sizeof(double) * P, cudaMemcpyDeviceToHost, h->stream)) ||
        (e = cudaStreamSynchronize(h->stream)))
        return cuda_fail(h, e, "solve");
    for (int p = 0; p < P; ++p) rmse[p] = rho[p] / std::sqrt((double)N);
    return st;
}

elmrnn_status elmrnn_solve_local(elmrnn_t h, const float* H, int64_t ldh, const float* Y, int64_t N, double* Rpk) {
    if (!h) return ELMRNN_ERR_ARG;
    if (!Rpk || N < 0 || (N > 0 && (!H || !Y))) return fail(h, ELMRNN_ERR_ARG, "bad argument");
    if (ldh < h->M) return fail(h, ELMRNN_ERR_SHAPE, "ldh < M");
    cudaError_t e;
    if ((e = tsqr_factor(h, H, ldh, Y, 1, N))) return cuda_fail(h, e, "tsqr_factor");
    if ((e = tsqr_pack(h, Rpk))) return cuda_fail(h, e, "tsqr_pack");
    return ELMRNN_OK;
}

elmrnn_status elmrnn_solve_merge(elmrnn_t h, const double* Rpk_all, int P, int64_t N_total, double* beta,
                                 elmrnn_solve_info* info) {
    if (!h) return ELMRNN_ERR_ARG;
    if (!Rpk_all || !beta || P < 1) return fail(h, ELMRNN_ERR_ARG, "bad argument");
    if (N_total < h->M) return fail(h, ELMRNN_ERR_UNDERDETERMINED, "N_total < M");
    cudaError_t e;
    if ((e = tsqr_merge_packed(h, Rpk_all, P))) return cuda_fail(h, e, "tsqr_merge");
    if ((e = tsqr_solve(h, N_total, beta))) return cuda_fail(h, e, "tsqr_solve");
    return finish_solve(h, info);
}

elmrnn_status elmrnn_sync(elmrnn_t h) {
    if (!h) return ELMRNN_ERR_ARG;
    cudaError_t e;
    if ((e = cudaStreamSynchronize(h->stream))) return cuda_fail(h, e, "sync");
    if (!h->sdev) return ELMRNN_OK;   // no solve has run on this handle
    if ((e = read_solve_dev(h))) return cuda_fail(h, e, "sync");
    if (h->shost->nf_sticky)
        return fail(h, ELMRNN_ERR_NONFINITE, "NaN or Inf in H or Y in an asynchronous solve since the last check");
    return ELMRNN_OK;
}

// Fused readout (Eq. 4): the builder runs with the
// readout sink set, so it writes no H(Q) -- only the fp64 partial products of
// its H(Q) row segments with beta (4 or fewer slots per row, elmrnn::ro_slots) --
// and k_readout_finish sums each row's slots in a fixed order.  With w != null
// the finish also shifts the forecast window (reading R31).
static elmrnn_status readout_impl(elmrnn* h, const float* X, int64_t ldx, const float* Yfb, int64_t ldy, int64_t N,
                                  const double* beta, float* yout, int64_t ldyo, float* w = nullptr,
                                  int64_t ldw = 0) {
    cudaError_t e;
    const int64_t need = (int64_t)elm::ro_max_slots(h->arch, h->M) * N;
    if (need > h->ypws_len) {
        if (h->ypws) cudaFree(h->ypws);
        h->ypws = nullptr;
        h->ypws_len = 0;
        if ((e = cudaMalloc(&h->ypws, sizeof(double) * need))) return cuda_fail(h, e, "readout workspace");
        h->ypws_len = need;
    }
    h->ro_beta = beta;
    h->ro_yp = h->ypws;
    h->ro_slots = 0;
    elmrnn_status st = build_impl(h, X, ldx, Yfb, ldy, N, nullptr, 0);
    h->ro_beta = nullptr;
    h->ro_yp = nullptr;
    if (st != ELMRNN_OK) return st;
    if (h->ro_slots == 0) return fail(h, ELMRNN_ERR_CUDA, "builder without a readout sink");
    if ((e = launch_readout_finish(h, h->ypws, N, h->ro_slots, yout, ldyo, w, ldw))) return cuda_fail(h, e, "readout");
    return ELMRNN_OK;
}

static cudaError_t ensure_hws(elmrnn* h, int64_t N) {
    if (N <= h->Hws_rows) return cudaSuccess;
    if (h->Hws) cudaFree(h->Hws);
    h->Hws = nullptr;
    h->Hws_rows = 0;
    cudaError_t e = cudaMalloc(&h->Hws, sizeof(float) * N * h->M);
    if (!e) h->Hws_rows = N;
    return e;
}

// Alg. 1 lines 2-3 in one call.  Cell-independent archs on
// the per-column TSQR path: fused build -> leaf, H never exists.  Others: H in a
// library workspace, then the solve.
static elmrnn_status train_factor(elmrnn* h, const float* X, int64_t ldx, const float* Yfb, int64_t ldy,
                                  const float* Y, int64_t N) {
    if (!X || !Y) return fail(h, ELMRNN_ERR_ARG, "NULL pointer");
    if (ldx < (int64_t)h->Q * h->S) return fail(h, ELMRNN_ERR_SHAPE, "ldx < Q*d");
    if (Yfb && ldy < h->Q) return fail(h, ELMRNN_ERR_SHAPE, "ldy < Q");
    cudaError_t e;
    if (h->fused_train && tsqr_fused_supported(h)) {
        if ((e = tsqr_factor_fused(h, X, ldx, Yfb, ldy, Y, N))) return cuda_fail(h, e, "train (fused)");
        return ELMRNN_OK;
    }
    if ((e = ensure_hws(h, N))) return cuda_fail(h, e, "train workspace");
    elmrnn_status st = build_impl(h, X, ldx, Yfb, ldy, N, h->Hws, h->M);
    if (st != ELMRNN_OK) return st;
    if ((e = tsqr_factor(h, h->Hws, h->M, Y, 1, N))) return cuda_fail(h, e, "tsqr_factor");
    return ELMRNN_OK;
}

elmrnn_status elmrnn_train(elmrnn_t h, const float* X, int64_t ldx, const float* Yfb, int64_t ldy, const float* Y,
                           int64_t N, double* beta, elmrnn_solve_info* info) {
    if (!h) return ELMRNN_ERR_ARG;
    if (!beta) return fail(h, ELMRNN_ERR_ARG, "NULL pointer");
    if (N < h->M) return fail(h, ELMRNN_ERR_UNDERDETERMINED, "N < M");
    elmrnn_status st = train_factor(h, X, ldx, Yfb, ldy, Y, N);
    if (st != ELMRNN_OK) return st;
    cudaError_t e;
    if ((e = tsqr_solve(h, N, beta))) return cuda_fail(h, e, "tsqr_solve");
    return finish_solve(h, info);
}

elmrnn_status elmrnn_train_local(elmrnn_t h, const float* X, int64_t ldx, const float* Yfb, int64_t ldy,
                                 const float* Y, int64_t N, double* Rpk) {
    if (!h) return ELMRNN_ERR_ARG;
    if (!Rpk || N < 0) return fail(h, ELMRNN_ERR_ARG, "bad argument");
    cudaError_t e;
    if (N == 0) {
        if ((e = tsqr_factor(h, nullptr, h->M, nullptr, 1, 0))) return cuda_fail(h, e, "tsqr_factor");
    } else {
        elmrnn_status st = train_factor(h, X, ldx, Yfb, ldy, Y, N);
        if (st != ELMRNN_OK) return st;
    }
    if ((e = tsqr_pack(h, Rpk))) return cuda_fail(h, e, "tsqr_pack");
    return ELMRNN_OK;
}

int elmrnn_train_fused(elmrnn_t h) { return h && h->fused_train && tsqr_fused_supported(h) ? 1 : 0; }

elmrnn_status elmrnn_solve_local_multi(elmrnn_t h, const float* H, int64_t ldh, const float* Y, int64_t ldy, int P,
                                       int64_t N, double* Rpk) {
    if (!h) return ELMRNN_ERR_ARG;
    if (!Rpk || N < 0 || P < 1 || (N > 0 && (!H || !Y))) return fail(h, ELMRNN_ERR_ARG, "bad argument");
    if (ldh < h->M) return fail(h, ELMRNN_ERR_SHAPE, "ldh < M");
    if (ldy < P) return fail(h, ELMRNN_ERR_SHAPE, "ldy < P");
    if (h->M + P > 1536) return fail(h, ELMRNN_ERR_UNSUPPORTED, "M + P <= 1536 (one 16-row WY tile in shared memory)");
    struct Nrhs { elmrnn* h; ~Nrhs() { h->nrhs = 1; } } guard{h};
    h->nrhs = P;
    cudaError_t e;
    if ((e = tsqr_factor(h, H, ldh, Y, ldy, N))) return cuda_fail(h, e, "tsqr_factor");
    if ((e = tsqr_pack(h, Rpk))) return cuda_fail(h, e, "tsqr_pack");
    return ELMRNN_OK;
}

elmrnn_status elmrnn_solve_merge_multi(elmrnn_t h, const double* Rpk_all, int ranks, int P, int64_t N_total,
                                       double* beta, double* rmse, elmrnn_solve_info* info) {
    if (!h) return ELMRNN_ERR_ARG;
    if (!Rpk_all || !beta || ranks < 1 || P < 1) return fail(h, ELMRNN_ERR_ARG, "bad argument");
    if (h->M + P > 1536) return fail(h, ELMRNN_ERR_UNSUPPORTED, "M + P <= 1536");
    if (N_total < h->M) return fail(h, ELMRNN_ERR_UNDERDETERMINED, "N_total < M");
    cudaError_t e;
    if (P > h->rho_multi_len) {
        if (h->rho_multi) cudaFree(h->rho_multi);
        h->rho_multi = nullptr;
        h->rho_multi_len = 0;
        if ((e = cudaMalloc(&h->rho_multi, sizeof(double) * P))) return cuda_fail(h, e, "workspace");
        h->rho_multi_len = P;
    }
    struct Nrhs { elmrnn* h; ~Nrhs() { h->nrhs = 1; } } guard{h};
    h->nrhs = P;
    if ((e = tsqr_merge_packed(h, Rpk_all, ranks))) return cuda_fail(h, e, "tsqr_merge");
    if ((e = tsqr_solve(h, N_total, beta))) return cuda_fail(h, e, "tsqr_solve");
    elmrnn_solve_info tmp;
    elmrnn_solve_info* ip = info ? info : (rmse ? &tmp : nullptr);
    const elmrnn_status st = finish_solve(h, ip);
    if (st < 0 || !rmse) return st;
    if (P == 1) {
        rmse[0] = ip->rmse;
        return st;
    }
    std::vector<double> rho(P);
    if ((e = cudaMemcpyAsync(rho.data(), h->rho_multi, sizeof(double) * P, cudaMemcpyDeviceToHost, h->stream)) ||
        (e = cudaStreamSynchronize(h->stream)))
        return cuda_fail(h, e, "solve");
    for (int p = 0; p < P; ++p) rmse[p] = rho[p] / std::sqrt((double)N_total);
    return st;
}

int64_t elmrnn_packed_r_len_multi(elmrnn_t h, int P) {
    if (!h || P < 1) return -1;
    return (int64_t)(h->M + P) * (h->M + P + 1) / 2;
}

int64_t elmrnn_packed_r_len(elmrnn_t h) {
    if (!h) return -1;
    return (int64_t)(h->M + 1) * (h->M + 2) / 2;
}


elmrnn_status elmrnn_predict(elmrnn_t h, const float* X, int64_t ldx, const float* Yfb, int64_t ldy, int64_t N,
                             const double* beta, float* Yhat) {
    if (!h) return ELMRNN_ERR_ARG;
    if (N < 0) return fail(h, ELMRNN_ERR_ARG, "N < 0");
    if (N == 0) return ELMRNN_OK;
    if (!X || !beta || !Yhat) return fail(h, ELMRNN_ERR_ARG, "NULL pointer");
    if (ldx < (int64_t)h->Q * h->S) return fail(h, ELMRNN_ERR_SHAPE, "ldx < Q*d");
    if (Yfb && ldy < h->Q) return fail(h, ELMRNN_ERR_SHAPE, "ldy < Q");
    return readout_impl(h, X, ldx, Yfb, ldy, N, beta, Yhat, 1);
}

static int64_t forecast_ldw(const elmrnn* h) { return (h->Q + 3) & ~3; }   // 16-B aligned window rows

elmrnn_status elmrnn_forecast(elmrnn_t h, const float* X, int64_t ldx, int64_t N, const double* beta, int K,
                              float* Yhat, int64_t ldyh) {
    if (!h) return ELMRNN_ERR_ARG;
    if (h->S != 1) return fail(h, ELMRNN_ERR_UNSUPPORTED, "free-running forecast needs a univariate window (d = 1)");
    if (h->Q > 128) return fail(h, ELMRNN_ERR_UNSUPPORTED, "forecast supports Q <= 128");
    if (N < 0 || K < 0) return fail(h, ELMRNN_ERR_ARG, "N < 0 or K < 0");
    if (N == 0 || K == 0) return ELMRNN_OK;
    if (!X || !beta || !Yhat) return fail(h, ELMRNN_ERR_ARG, "NULL pointer");
    if (ldx < h->Q) return fail(h, ELMRNN_ERR_SHAPE, "ldx < Q");
    if (ldyh < K) return fail(h, ELMRNN_ERR_SHAPE, "ldyh < K");
    cudaError_t e;
    const int64_t ldw = forecast_ldw(h);
    if (N > h->fws_rows) {
        if (h->fws) cudaFree(h->fws);
        h->fws = nullptr;
        h->fws_rows = 0;
        if ((e = cudaMalloc(&h->fws, sizeof(float) * N * (ldw + 1)))) return cuda_fail(h, e, "forecast workspace");
        h->fws_rows = N;
    }
    if ((e = launch_window_init(h, X, ldx, N, h->fws, ldw))) return cuda_fail(h, e, "forecast");
    // per step: the fused readout of the current windows, then the window shift (in the finish)
    for (int k = 0; k < K; ++k) {
        elmrnn_status st = readout_impl(h, h->fws, ldw, nullptr, 0, N, beta, Yhat + k, ldyh, h->fws, ldw);
        if (st != ELMRNN_OK) return st;
    }
    return ELMRNN_OK;
}

elmrnn_status elmrnn_test_rmse(elmrnn_t h, const float* X, int64_t ldx, const float* Yfb, int64_t ldy,
                               const float* Y, int64_t N, const double* beta, double* rmse) {
    if (!h) return ELMRNN_ERR_ARG;
    if (N < 1) return fail(h, ELMRNN_ERR_ARG, "N < 1");
    if (!X || !Y || !beta || !rmse) return fail(h, ELMRNN_ERR_ARG, "NULL pointer");
    if (ldx < (int64_t)h->Q * h->S) return fail(h, ELMRNN_ERR_SHAPE, "ldx < Q*d");
    if (Yfb && ldy < h->Q) return fail(h, ELMRNN_ERR_SHAPE, "ldy < Q");
    cudaError_t e;
    if (N > h->fws_rows) {
        if (h->fws) cudaFree(h->fws);
        h->fws = nullptr;
        h->fws_rows = 0;
        if ((e = cudaMalloc(&h->fws, sizeof(float) * N * (forecast_ldw(h) + 1)))) return cuda_fail(h, e, "workspace");
        h->fws_rows = N;
    }
    if (!h->dscr && (e = cudaMalloc(&h->dscr, sizeof(double)))) return cuda_fail(h, e, "workspace");
    float* yhat = h->fws + (size_t)N * forecast_ldw(h);
    elmrnn_status st = elmrnn_predict(h, X, ldx, Yfb, ldy, N, beta, yhat);
    if (st != ELMRNN_OK) return st;
    if ((e = launch_rmse(h, yhat, Y, N, h->dscr))) return cuda_fail(h, e, "test_rmse");
    if ((e = cudaMemcpyAsync(rmse, h->dscr, sizeof(double), cudaMemcpyDeviceToHost, h->stream)) ||
        (e = cudaStreamSynchronize(h->stream)))
        return cuda_fail(h, e, "test_rmse");
    return ELMRNN_OK;
}

int64_t elmrnn_weight_block_len(elmrnn_t h, int block_id) {
    if (!h) return -1;
    return logical_block_len(h, block_id);
}

elmrnn_status elmrnn_get_weights(elmrnn_t h, int block_id, float* host_dst, int64_t count) {
    if (!h) return ELMRNN_ERR_ARG;
    int64_t len = logical_block_len(h, block_id);
    if (len < 0 || !host_dst || count != len) return fail(h, ELMRNN_ERR_ARG, "bad block id or count");
    if (len == 0) return ELMRNN_OK;
    float* tmp = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&tmp, sizeof(float) * len))) return cuda_fail(h, e, "get_weights");
    int64_t n = 0;
    e = gen_logical_block(h, block_id, tmp, &n);
    if (!e) e = cudaMemcpyAsync(host_dst, tmp, sizeof(float) * len, cudaMemcpyDeviceToHost, h->stream);
    if (!e) e = cudaStreamSynchronize(h->stream);
    cudaFree(tmp);
    if (e) return cuda_fail(h, e, "get_weights");
    return ELMRNN_OK;
}

int elmrnn_path(elmrnn_t h) { return h ? h->path : 0; }

int64_t elmrnn_launch_count(elmrnn_t h) { return h ? h->launches : -1; }

const char* elmrnn_last_error(elmrnn_t h) { return h ? h->err.c_str() : g_init_error.c_str(); }

void elmrnn_destroy(elmrnn_t h) {
    if (!h) return;
    cudaFree(h->W); cudaFree(h->b); cudaFree(h->rec); cudaFree(h->tc_ops);
    cudaFree(h->Rws); cudaFree(h->sdev); cudaFree(h->flag); cudaFree(h->Hws); cudaFree(h->prog); cudaFree(h->rho_multi); cudaFree(h->rws); cudaFree(h->fws); cudaFree(h->dscr); cudaFree(h->scratch); cudaFree(h->ypws);
    if (h->shost) cudaFreeHost(h->shost);
    delete h;
}

}  // extern "C"
