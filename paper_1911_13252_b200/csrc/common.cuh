// common.cuh -- internal declarations of libelmrnn (not part of the ABI).
// The public contract is include/elmrnn.h; citations "P:n" = PAPER.md line n.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include <vector>

#include "elmrnn.h"

namespace elm {

constexpr int kArchElman = 0, kArchJordan = 1, kArchNarmax = 2, kArchFC = 3, kArchLSTM = 4, kArchGRU = 5;
constexpr int kArchLSTMDiag = 6, kArchGRUDiag = 7, kArchFCEq8 = 8;   // paper-literal per-cell variants

inline int gates_of(int arch) {
    return (arch == kArchLSTM || arch == kArchLSTMDiag) ? 4 : ((arch == kArchGRU || arch == kArchGRUDiag) ? 3 : 1);
}

// Device-side solve diagnostics (copied to the host struct on request).
struct SolveDev {
    double rho, rmse, dmin, dmax, lambda;
    int rank_flag;
    int nonfinite;
    long long n_total;
    int nf_sticky;   // OR of `nonfinite` over the solves since the last synchronising check
};

// Tuning overrides: defaults are the measured choices; a test may override them
// through the environment ONLY when ELMRNN_TESTING=1 is set, and they are read
// once, at elmrnn_init_ex (never on the solve path).
struct Tune {
    int tsqr_wy = -1;   // ELMRNN_TSQR_WY: 1 force the blocked-WY TSQR, 0 force the per-column fold
    int wy_rows = 0;    // ELMRNN_TSQR_WY_ROWS: WY leaf tile rows (8..96)
    int pw_mode = -1;   // ELMRNN_PW_MODE: WY leaf panel warp 0 rotate SMSPs per CTA, 1 pin to SMSP 0 (-1: by tile)
    int wy_nw = 0;      // ELMRNN_WY_NW: WY leaf/merge warps per CTA (4 or 8; 0 = by n)
    int max_slabs = 0;  // ELMRNN_TSQR_MAXSLABS: cap on the TSQR leaf count (0 = by size)
    int wy_2phase = 1;  // ELMRNN_WY_2PHASE: 0 = single-chain WY leaf only; 2 = two-phase also for n <= 320
    int merge_small = 1; // ELMRNN_MERGE_SMALL: 0 = top tree levels keep the tall merge tiles
    int wide_pair = 1;   // ELMRNN_WIDE_PAIR: 0 = wide LSTM MMA units of one 32-neuron chunk (N = 128)
};

}  // namespace elm

// The opaque handle.  Weights are stored in kernel-friendly packed layouts
// (DESIGN.md "Data layout in HBM"); the logical blocks are regenerated on
// demand by elmrnn_get_weights.
struct elmrnn {
    int arch, S, M, Q, F, R, act, fc_lags, rec_scale, weight_grid, force_path, fused_train;
    int G;                // gate blocks
    uint64_t seed;
    int device, sm_count;
    cudaStream_t stream;
    int path;             // 1 FMA, 2 tensor cores
    // packed weights (device)
    float* W;             // [S][G*M]
    float* b;             // [G*M]
    float* rec;           // Elman/Jordan alpha^T [Q][M]; NARMAX W'^T [F][M] | W''^T [R][M]; FC A [L][M][M];
                          // LSTM/GRU U_cat [M][G*M] (U_cat[k][g*M+j] = U_g[k][j])
    int64_t rec_len;
    // tensor-core operands (device; only when path == 2)
    void* tc_ops;
    size_t tc_ops_bytes;
    float tc_inv_scale;       // 2^-sigma of the scaled fp16 U images
    std::vector<float> tc_wb; // host copy of W | b (kernel parameter block)
    // solve workspace (device)
    double* Rws;          // slabs of n^2 doubles, n = M + nrhs
    int64_t Rws_slabs;
    int Rws_n;            // n the slabs were allocated for
    int nrhs;             // outputs in the current solve (1; P inside elmrnn_solve_beta_multi)
    double* rho_multi;    // device [P] per-output residual norms (multi-output solve)
    int* prog;            // pipelined-merge progress counters [pairs][128]
    int64_t prog_pairs;
    int rho_multi_len;
    elm::SolveDev* sdev;  // device diagnostics
    int* flag;            // device non-finite flag
    elm::SolveDev* shost; // pinned host mirror
    float* Hws;           // predict scratch
    float* rws;           // error-window scratch: residual per row (N floats)
    int64_t rws_rows;
    float* fws;           // forecast window buffer [N][ldw] + predict output [N]
    int64_t fws_rows;
    double* dscr;         // device scalar (held-out RMSE)
    int64_t Hws_rows;
    float* scratch;       // builder scratch (FC history ring)
    size_t scratch_bytes;
    // fused readout sink (Eq. 4): while ro_beta is set, a builder
    // writes no H(Q) but the fp64 partial dot products of its H(Q) row segments with
    // beta, slot s of row i at ro_yp[s * N + i]; the launcher reports the slot layout
    // in ro_slots (K > 0: K slots per row; kRoCellSlots: the 32-cell warp groups a row
    // spans) and elm::launch_readout_finish sums the slots in a fixed order
    const double* ro_beta;
    double* ro_yp;
    int ro_slots;
    double* ypws;         // readout slot workspace
    int64_t ypws_len;
    int64_t launches;
    elm::Tune tune;
    std::string err;
};

namespace elm {

// ---- weights (weights.cu) -------------------------------------------------
cudaError_t gen_weights(elmrnn* h);
cudaError_t gen_logical_block(elmrnn* h, int block_id, float* dst_dev, int64_t* count);
int64_t logical_block_len(const elmrnn* h, int block_id);
int num_blocks(int arch);

// ---- H builders --------------------------------------------------------------
cudaError_t launch_elman(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh);
cudaError_t launch_diag_gated(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh);
cudaError_t launch_teacher_forced(elmrnn* h, const float* X, int64_t ldx, const float* Yfb, int64_t ldy,
                                  int64_t N, float* H, int64_t ldh, const float* Ef = nullptr, int64_t lde = 0);
cudaError_t launch_window_init(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* w, int64_t ldw);
cudaError_t launch_rmse(elmrnn* h, const float* yhat, const float* y, int64_t N, double* out);
cudaError_t launch_error_windows(elmrnn* h, const float* H, int64_t ldh, const float* Y, int64_t N,
                                 const double* beta, float* Ef, int64_t lde);
cudaError_t launch_dense_fma(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh);
bool elman_supported(int Q);

// ---- tensor-core builder (hbuild_dense_tc.cu) -----------------------------
bool tc_supported(const elmrnn* h);
cudaError_t tc_prepare(elmrnn* h);
cudaError_t launch_dense_tc(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh);
bool gru_tc_supported(const elmrnn* h);
cudaError_t gru_tc_prepare(elmrnn* h);
cudaError_t launch_gru_tc(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh);
bool lstm_wide_supported(const elmrnn* h);
bool lstm_wide_pair(const elmrnn* h);
bool gru_wide_supported(const elmrnn* h);
cudaError_t gru_wide_prepare(elmrnn* h);
cudaError_t launch_gru_wide(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh);
size_t lstm_wide_wb_offset(const elmrnn* h);
cudaError_t launch_lstm_wide(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh);
bool fc_tc_supported(const elmrnn* h);
cudaError_t fc_tc_prepare(elmrnn* h);
cudaError_t launch_fc_tc(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh);

// ---- TSQR (tsqr.cu) ------------------------------------------------------------
// Fold [H | Y] rows into per-CTA R slabs and reduce them to slab 0 (full storage).
cudaError_t tsqr_factor(elmrnn* h, const float* H, int64_t ldh, const float* Y, int64_t ldy, int64_t N);
cudaError_t tsqr_pack(elmrnn* h, double* Rpk);
bool tsqr_fused_supported(const elmrnn* h);
cudaError_t tsqr_factor_fused(elmrnn* h, const float* X, int64_t ldx, const float* Yfb, int64_t ldyfb, const float* Y,
                              int64_t N);
cudaError_t tsqr_merge_packed(elmrnn* h, const double* Rpk_all, int P);
cudaError_t tsqr_solve(elmrnn* h, int64_t n_total, double* beta);
cudaError_t ensure_solve_ws(elmrnn* h, int64_t slabs);
int64_t tsqr_leaf_slabs(const elmrnn* h, int64_t N);

// ---- fused readout (readout.cu) ---------------------------------------------------
constexpr int kRoCellSlots = -1;   // slot = 32-cell group index - first group of the row
// slots per row: the flattened-cell builders (Elman / FC by Eq. 8 / diagonal LSTM-GRU)
// one per 32-cell warp group the row spans; the tile builders at most 4
inline int ro_max_slots(int arch, int M) {
    const bool cell = arch == kArchElman || arch == kArchFCEq8 || arch == kArchLSTMDiag || arch == kArchGRUDiag;
    return cell ? (M + 31) / 32 + 1 : 4;
}
// yhat_i = fp32(sum of row i's slots, in slot order); with w != null also
// w_i <- (w_i[1:], yhat_i) (the free-running forecast step, reading R31)
cudaError_t launch_readout_finish(elmrnn* h, const double* yp, int64_t N, int slots, float* yout, int64_t ldyo,
                                  float* w, int64_t ldw);

}  // namespace elm

// ---- small device helpers ------------------------------------------------------
#ifdef __CUDACC__
namespace elm {
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// Activations (R3).  The H builders use the accurate forms: the beta of an
// ill-conditioned [H|Y] (cond(H) ~ 1e6 on smooth series) amplifies every ulp
// of H, so H is kept within ~1-2 ulp of the rounded fp64 value.
//   sigma(a) = 1 / (1 + e^-a)  (expf: <= 2 ulp; IEEE division)
//   tanh(a)  = tanhf(a)        (<= 2 ulp)
__device__ __forceinline__ float sigmoidf_(float a) { return 1.0f / (1.0f + expf(-a)); }
__device__ __forceinline__ float tanhf_(float a) { return tanhf(a); }
__device__ __forceinline__ float act_g(float a, int act) { return act == 1 ? tanhf_(a) : sigmoidf_(a); }
// fp64 forms for the latency-bound per-cell builders
__device__ __forceinline__ double sigmoid64(double a) { return 1.0 / (1.0 + exp(-a)); }
__device__ __forceinline__ double act_g64(double a, int act) { return act == 1 ? tanh(a) : sigmoid64(a); }
// Gate forms of the tensor-core epilogues, from exp2-domain arguments (the
// gate's log2(e) factor and the 2^-sigma operand scale are folded into the
// accumulator scale and W|b on the host):
//   sig_e2(a2)  = 1 / (1 + 2^a2)            = sigma(x) for a2 = -log2(e) x
//   tanh_e2(a2) = tanh(a2 / (2 log2(e)))    = tanh(x)  for a2 = 2 log2(e) x
// Accuracy matters more than MUFU count here: a shared reciprocal of 2-4 gate
// denominators and tanh(x) as 1 - 2/(1 + e^2x) left a systematic bias in H
// (mean -7e-9, measured) that ill-conditioned solves amplify into beta (6-7x
// the fp32-rounding floor; DESIGN R26).  ex2.approx + rcp.approx with one
// Newton step is correctly rounded in practice (bitwise equal to
// 1.0f / (1.0f + exp2f(a2)) on the parity cases), tanhf is libm's (<= 2 ulp).
__device__ __forceinline__ float sig_e2(float a2) {
    const float d = 1.0f + ex2_approx(fminf(a2, 80.0f));   // sigma(x < -55) ~ 0 (< 1e-24), never inf/NaN
    const float r = rcp_approx(d);
    return fmaf(r, fmaf(-d, r, 1.0f), r);
}
__device__ __forceinline__ float tanh_e2(float a2) { return tanhf(a2 * 0.34657359027997264f); }
__device__ __forceinline__ float tanh_acc(float x) { return tanhf(x); }
// tanh(x) = 2 sigma(2x) - 1 with the correctly rounded sigma: unbiased, absolute
// error ~1 ulp(1) near 0.  The GRU candidate uses it: measured beta deviation
// 4.3 vs 3.8 floors with tanhf at 10% less build time (C3 GRU); the LSTM keeps
// tanhf (2.1-2.3 vs 3.9-5.8 floors with this form).
__device__ __forceinline__ float tanh_e2_sig(float a2) { return fmaf(2.0f, sig_e2(-a2), -1.0f); }

// Fused readout of the flattened-cell builders (cell c = i*M + j, 32 consecutive
// cells per warp): per row segment of the warp, sum v over its lanes (fixed
// shuffle order: deterministic) and store it from the segment's first lane into
// slot (c/32 - (i*M)/32) of row i (kRoCellSlots layout).  All 32 lanes must call.
__device__ __forceinline__ void ro_cell_store(double v, int64_t cell, int64_t N, int M, double* yp) {
    const int lane = threadIdx.x & 31;
    const int64_t i = cell / M;
    const int64_t last = min((i + 1) * (int64_t)M, N * (int64_t)M) - 1;   // last cell of row i
    const int seg_end = (int)min((int64_t)31, (last - cell) + lane);       // lane of that cell in this warp
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double t = __shfl_down_sync(0xffffffffu, v, off);
        if (lane + off <= seg_end) v += t;
    }
    const bool head = lane == 0 || cell % M == 0;
    if (head && cell < N * (int64_t)M) yp[(cell / 32 - (i * M) / 32) * N + i] = v;
}

// Fast MUFU forms (ex2.approx / rcp.approx, ~2 ulp each) for epilogues that
// are MUFU bound; accuracy validated by the parity tests of the kernel using them.
__device__ __forceinline__ float sigmoid_fast(float a) {
    return rcp_approx(1.0f + ex2_approx(-1.4426950408889634f * a));
}
__device__ __forceinline__ float tanh_fast(float a) {
    return 1.0f - 2.0f * rcp_approx(1.0f + ex2_approx(2.8853900817779268f * a));
}
}  // namespace elm
#endif
