// tsqr.cu -- fp64 Householder tall-skinny QR of [H | Y], Q^T Y by the same
// reflectors, and back substitution: S4.2 of the paper, "H = QR,
// z = Q^T Y, R beta = z by back substitution".  The paper delegates this to a
// Numba/NumPy library call; here it is three kernels:
//
//  k_tsqr_leaf   persistent CTAs, each owning a contiguous row block and an
//                (M+1)x(M+1) R slab (full storage, L2 resident).  Row tiles of
//                P*TR rows are folded in: R <- R-factor of [R; tile] by the
//                structured Householder sweep (LAPACK tpqrt semantics).  The
//                tile lives in registers: the P threads of column j (adjacent
//                lanes) hold TR rows each of tile column j, and they own column
//                j of R, so R needs no inter-thread synchronisation; partial
//                dot products of a column pair combine with one shuffle.  The
//                reflector v of column k is broadcast through shared memory,
//                one barrier per column, with one-column look-ahead (the owner
//                of k+1 builds its reflector right after its own update).
//  k_tsqr_merge  one level of a binary tree: slab c absorbs slab c+stride by
//                folding it in (P*TR)-row tiles, skipping the zero columns
//                left of each tile's diagonal.
//  k_tsqr_solve  one CTA: sign normalisation (R18), rank check + ridge
//                fallback by folding sqrt(lambda) (I|0) rows (R19), back
//                substitution, rho = ||R_aug [beta; -1]|| = ||H beta - Y||.
//
// All arithmetic is fp64 (reading R20: an fp32 streaming fold breaks the beta
// tolerance); H and Y are read as fp32 and widened exactly.
#include <cfloat>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <type_traits>

#include "common.cuh"
#include "cell.cuh"

namespace elm {

// TR rows per thread, P threads per column (1 or 2): tile = P*TR rows.
template <int TR, int P>
struct Fold {
    static constexpr int ROWS = TR * P;
    // register budget (16K registers per SM sub-partition): 2*TR registers of
    // tile per thread plus ~40; 576 threads -> 96 registers, 1024 -> 64
    static constexpr int MAX_THREADS = (P == 2 && (TR == 24 || TR == 16)) ? 576 : (TR >= 32 ? 256 : 1024);
};

// Fast fp64 reciprocal / square root: hardware approximation + Newton steps
// (the reflector is on the per-column critical path; IEEE div/sqrt sequences
// cost hundreds of cycles of dependent latency).  Outside a safe exponent
// range the IEEE forms are used.
__device__ __forceinline__ double rcp_fast(double d) {
#ifdef ELM_TSQR_IEEE
    return 1.0 / d;
#endif
    const double ad = fabs(d);
    if (!(ad > 1e-250 && ad < 1e250)) return 1.0 / d;
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}
__device__ __forceinline__ double sqrt_fast(double t) {
#ifdef ELM_TSQR_IEEE
    return sqrt(t);
#endif
    if (!(t > 1e-250 && t < 1e250)) return sqrt(t);
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t));
    y = y * fma(-0.5 * t * y, y, 1.5);
    double s = t * y;
    return fma(0.5 * y, fma(-s, s, t), s);
}

// Reflector of column k from x0 = R[k][k] and the tile column a (this thread's
// TR rows; the partner lane holds the rest), in the unnormalised form
//   H = I + g u u^T,  u = [x0 - beta; a],  g = 1 / (beta (x0 - beta)),
//   beta = -sign(x0) ||(x0, a)||,  sign(0) = +1,
// which equals LAPACK's I - tau v v^T (v = u / u0, tau = (beta - x0)/beta)
// with one reciprocal and no scaling of u.  ||a|| = 0 gives H = I (g = 0).
// Both threads of the column compute it; half 0 publishes (g, u0) and R[k][k].
template <int TR, int P>
__device__ __forceinline__ void make_reflector(const double (&a)[TR], double x0, double* v, double* coef, double* Rkk,
                                               int half, unsigned mask) {
    double p0 = 0.0, p1 = 0.0, p2 = 0.0, p3 = 0.0;
#pragma unroll
    for (int i = 0; i < TR; i += 4) {
        p0 = fma(a[i], a[i], p0);
        p1 = fma(a[i + 1], a[i + 1], p1);
        p2 = fma(a[i + 2], a[i + 2], p2);
        p3 = fma(a[i + 3], a[i + 3], p3);
    }
    double s2 = (p0 + p1) + (p2 + p3);
    if (P == 2) s2 += __shfl_xor_sync(mask, s2, 1);
    if (s2 == 0.0) {
        if (half == 0) coef[0] = 0.0;
        return;
    }
    const double beta = -(x0 >= 0.0 ? 1.0 : -1.0) * sqrt_fast(fma(x0, x0, s2));
    const double u0 = x0 - beta;
    // A reflector of a column whose norm is at rounding-noise-of-noise level
    // (trailing rows of rank-deficient partial R factors) would overflow
    // 1/(beta u0); such a column is treated as already reduced (H = I), as
    // LAPACK's dlarfg guards with safmin.
    if (!(fabs(beta * u0) > 1e-280)) {
        if (half == 0) coef[0] = 0.0;
        return;
    }
#pragma unroll
    for (int i = 0; i < TR; ++i) v[half * TR + i] = a[i];
    if (half == 0) {
        coef[0] = rcp_fast(beta * u0);
        coef[1] = u0;
        *Rkk = beta;
    }
}

// Column owned by this thread (adjacent lanes share a column when P = 2).
// A reversed mapping (look-ahead column in the highest warp) was measured
// slower (2200 vs 2055 cycles per column), so columns map in order.
template <int P>
__device__ __forceinline__ int col_of(int n) {
    return (int)(threadIdx.x / P);
}

// Optional event trace of CTA 0 (testing aid, ELMRNN_TRACE_QR): per column,
// clock at loop top (thread 0), after the update of thread k+1, after its
// reflector, and after the barrier.
__device__ unsigned long long* g_qr_trace = nullptr;
__device__ __forceinline__ void qr_ev_t(int slot, int k) {   // globaltimer (ns) variant
#ifdef ELM_QR_TRACE
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    if (g_qr_trace && blockIdx.x == 0 && k < 4096) g_qr_trace[k * 8 + slot] = t;
#endif
}
__device__ __forceinline__ void qr_ev(int slot, int k) {
#ifdef ELM_QR_TRACE   // compiled in only for tracing builds: the pointer load sits on the critical path
    if (g_qr_trace && blockIdx.x == 0 && k < 4096) g_qr_trace[k * 8 + slot] = clock64();
#endif
}

// Fold the register tile (thread (j, half) holds rows half*TR.. of column j)
// into R (n x n, full storage), columns k0..n-1.  vbuf: 2*ROWS doubles of
// shared memory (u tails), coefs: 2 x (g, u0).
template <int TR, int P>
__device__ void fold_tile(double (&a)[TR], int n, int k0, double* __restrict__ R, double* vbuf, double* coefs) {
    constexpr int ROWS = TR * P;
    const int j = col_of<P>(n), half = threadIdx.x % P;
    const bool own = j >= 0 && j < n;
    // R[k][j] for the next three rows are prefetched into registers: the
    // reflector of column k+1 needs R[k+1][k+1] right after its own update,
    // so its L2 latency must be hidden two columns ahead.
    const double* Rj = R + j;
    auto ld = [&](int row) -> double { return (own && row < n && j >= row) ? Rj[(size_t)row * n] : 0.0; };
    double rq0 = ld(k0), rq1 = ld(k0 + 1), rq2 = ld(k0 + 2);
    {
        const unsigned m = __ballot_sync(0xffffffffu, j == k0);
        if (j == k0)
            make_reflector<TR, P>(a, rq0, vbuf + (k0 & 1) * ROWS, coefs + 2 * (k0 & 1), R + (size_t)k0 * n + k0,
                                  half, m);
    }
    __syncthreads();
    for (int k = k0; k < n; ++k) {
        if (threadIdx.x == 0) qr_ev(0, k);
        const double rkj = rq0;
        rq0 = rq1;
        rq1 = rq2;
        rq2 = ld(k + 3);
        const double g = coefs[2 * (k & 1)], u0 = coefs[2 * (k & 1) + 1];
        const bool upd = own && j > k && g != 0.0;
        const unsigned mu = __ballot_sync(0xffffffffu, upd);
        if (upd) {
            const double2* v = reinterpret_cast<const double2*>(vbuf + (k & 1) * ROWS + half * TR);
            double w0 = (half == 0) ? u0 * rkj : 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
#pragma unroll
            for (int i = 0; i < TR; i += 4) {
                const double2 va = v[i / 2], vb = v[i / 2 + 1];
                w0 = fma(va.x, a[i], w0);
                w1 = fma(va.y, a[i + 1], w1);
                w2 = fma(vb.x, a[i + 2], w2);
                w3 = fma(vb.y, a[i + 3], w3);
            }
            double w = (w0 + w1) + (w2 + w3);
            if (P == 2) w += __shfl_xor_sync(mu, w, 1);
            const double f = g * w;                      // x_j += f u
            if (half == 0) R[(size_t)k * n + j] = fma(f, u0, rkj);
#pragma unroll
            for (int i = 0; i < TR; i += 2) {
                const double2 vv = v[i / 2];
                a[i] = fma(f, vv.x, a[i]);
                a[i + 1] = fma(f, vv.y, a[i + 1]);
            }
        }
        const bool nxt = j == k + 1 && k + 1 < n;
        if (nxt && half == 0) qr_ev(1, k);
        const unsigned mr = __ballot_sync(0xffffffffu, nxt);
        if (nxt)
            make_reflector<TR, P>(a, rq0, vbuf + ((k + 1) & 1) * ROWS, coefs + 2 * ((k + 1) & 1),
                                  R + (size_t)(k + 1) * n + (k + 1), half, mr);
        if (nxt && half == 0) qr_ev(2, k);
        __syncthreads();
        if (threadIdx.x == 0) qr_ev(3, k);
    }
}


// Leaf element sources: H loaded from memory, or computed per cell (fused
// build -> leaf, elmrnn_train; cell.cuh).  KIND 0: H; 1: Elman (QMAX >= Q);
// 2: Jordan / NARMAX teacher forced.
template <int KIND, int QMAX>
struct LeafSrc {
    const float* H;
    int64_t ldh;
    CellSrc cell;
    __device__ __forceinline__ float at(int64_t row, int j) const {
        if constexpr (KIND == 0) return __ldg(H + row * ldh + j);
        else if constexpr (KIND == 1) return cell_elman<QMAX>(cell, row, j);
        else return cell_tf(cell, row, j);
    }
};

template <int TR, int P, int KIND = 0, int QMAX = 1>
__global__ void __launch_bounds__(Fold<TR, P>::MAX_THREADS, 1)
    k_tsqr_leaf(const LeafSrc<KIND, QMAX> src, const float* __restrict__ Y, int64_t ldy, int64_t N, int M,
                double* __restrict__ Rws, int64_t rows_per_cta, int* __restrict__ flag) {
    constexpr int ROWS = TR * P;
    __shared__ __align__(16) double vbuf[2 * ROWS];
    __shared__ double coefs[4];
    const int n = M + 1, j = col_of<P>(n), half = threadIdx.x % P;
    double* R = Rws + (size_t)blockIdx.x * n * n;
    if (j >= 0 && j < n)
        for (int k = half; k < n; k += P) R[(size_t)k * n + j] = 0.0;   // column j is private to its threads
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
    const int64_t r1 = min(N, r0 + rows_per_cta);
    bool bad = false;
    for (int64_t base = r0; base < r1; base += ROWS) {
        double a[TR];
#pragma unroll
        for (int i = 0; i < TR; ++i) {
            const int64_t row = base + half * TR + i;
            float v = 0.0f;
            if (row < r1 && j >= 0 && j < n) v = (j < M) ? src.at(row, j) : __ldg(Y + row * ldy);
            bad |= !isfinite(v);
            a[i] = (double)v;
        }
        fold_tile<TR, P>(a, n, 0, R, vbuf, coefs);
    }
    if (bad) atomicOr(flag, 1);
}

template <int TR, int P>
__global__ void __launch_bounds__(Fold<TR, P>::MAX_THREADS, 1)
    k_tsqr_merge(double* __restrict__ Rws, int64_t slabs, int64_t stride, int n) {
    constexpr int ROWS = TR * P;
    __shared__ __align__(16) double vbuf[2 * ROWS];
    __shared__ double coefs[4];
    const int64_t c = (int64_t)blockIdx.x * 2 * stride, partner = c + stride;
    if (partner >= slabs) return;
    double* Ra = Rws + (size_t)c * n * n;
    const double* Rb = Rws + (size_t)partner * n * n;
    const int j = col_of<P>(n), half = threadIdx.x % P;
    for (int s = 0; s * ROWS < n; ++s) {
        double a[TR];
#pragma unroll
        for (int i = 0; i < TR; ++i) {
            const int row = s * ROWS + half * TR + i;
            a[i] = (row < n && j >= 0 && j < n && j >= row) ? Rb[(size_t)row * n + j] : 0.0;
        }
        fold_tile<TR, P>(a, n, s * ROWS, Ra, vbuf, coefs);
    }
}

// Unpack P packed R factors (row k holds R[k][k..n-1]) into full slabs.
__global__ void k_unpack(const double* __restrict__ Rpk, int P, int n, double* __restrict__ Rws) {
    const int64_t len = (int64_t)n * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)P * len;
         e += (int64_t)gridDim.x * blockDim.x) {
        int64_t p = e / len, rem = e - p * len;
        int k = (int)(rem / n), j = (int)(rem - (int64_t)k * n);
        double v = 0.0;
        if (j >= k) v = Rpk[p * ((int64_t)n * (n + 1) / 2) + (int64_t)k * n - (int64_t)k * (k - 1) / 2 + (j - k)];
        Rws[e] = v;
    }
}

__global__ void k_pack(const double* __restrict__ R, int n, double* __restrict__ Rpk, const int* __restrict__ flag,
                       SolveDev* __restrict__ sdev) {
    const int64_t len = (int64_t)n * (n + 1) / 2;
    if (blockIdx.x == 0 && threadIdx.x == 0 && *flag) sdev->nf_sticky = 1;   // reported by elmrnn_sync
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len; e += (int64_t)gridDim.x * blockDim.x) {
        // row k starts at k*n - k(k-1)/2; find k by bisection (n <= 1024)
        int lo = 0, hi = n - 1;
        while (lo < hi) {
            int mid = (lo + hi + 1) / 2;
            if ((int64_t)mid * n - (int64_t)mid * (mid - 1) / 2 <= e) lo = mid; else hi = mid - 1;
        }
        int k = lo;
        int j = k + (int)(e - ((int64_t)k * n - (int64_t)k * (k - 1) / 2));
        Rpk[e] = R[(size_t)k * n + j];
    }
}

__device__ double block_sum(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < nw; ++i) s += red[i];
    __syncthreads();
    return s;
}
__device__ double block_min(double v, double* red) {
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = INFINITY;
    for (int i = 0; i < nw; ++i) s = fmin(s, red[i]);
    __syncthreads();
    return s;
}
__device__ double block_max(double v, double* red) { return -block_min(-v, red); }

// Final solve on slab 0 (one CTA of P*n threads).  R0 is copied to Rorig
// before a ridge refactorisation so rho is measured on the unregularised R.
template <int TR, int P>
__global__ void __launch_bounds__(Fold<TR, P>::MAX_THREADS, 1)
    k_tsqr_solve(double* __restrict__ Rg, double* __restrict__ Rorig, int M, long long n_total,
                 const int* __restrict__ flag, double* __restrict__ beta, SolveDev* __restrict__ out, int r_smem) {
    constexpr int ROWS = TR * P;
    __shared__ __align__(16) double vbuf[2 * ROWS];
    __shared__ double coefs[4];
    __shared__ double red[32];
    extern __shared__ __align__(16) double zs[];   // [3][n] signs / rhs, R_kk, beta; then R when r_smem
    const int n = M + 1, j = col_of<P>(n), half = threadIdx.x % P;
    const bool own = j >= 0 && j < n && half == 0;
    // small n: the whole R in shared memory (one coalesced copy in and out), so the
    // column walks below (sign flips, norms, the ridge fold) are not chains of L2 loads
    double* R = Rg;
    if (r_smem) {
        R = zs + 3 * ((n + 1) & ~1);
        for (int e = threadIdx.x; e < n * n; e += blockDim.x) R[e] = Rg[e];
        __syncthreads();
    }
    // sign normalisation: flip row k when R_kk < 0 (signs read into smem first)
    if (own) zs[j] = R[(size_t)j * n + j] < 0.0 ? -1.0 : 1.0;
    __syncthreads();
    if (own)
        for (int k = 0; k <= j; ++k) R[(size_t)k * n + j] *= zs[k];
    __syncthreads();
    const bool diag = own && j < M;
    double d = diag ? fabs(R[(size_t)j * n + j]) : INFINITY;
    const double dmin = block_min(d, red);
    const double dmax = block_max(diag ? d : 0.0, red);
    double f2 = 0.0;
    if (diag)
        for (int k = 0; k <= j; ++k) f2 += R[(size_t)k * n + j] * R[(size_t)k * n + j];
    const double fro2 = block_sum(f2, red);
    const bool ridge = !(dmin > DBL_EPSILON * (double)M * dmax);
    double lambda = 0.0;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) Rorig[e] = R[e];   // sign-normalised, pre-ridge
    if (ridge) {
        lambda = 1e-8 * fro2 / (double)M;
        const double sl = sqrt(lambda);
        for (int s = 0; s * ROWS < M; ++s) {
            double a[TR];
#pragma unroll
            for (int i = 0; i < TR; ++i) {
                const int row = s * ROWS + half * TR + i;
                a[i] = (row < M && j == row) ? sl : 0.0;
            }
            fold_tile<TR, P>(a, n, s * ROWS, R, vbuf, coefs);
        }
        if (own) zs[j] = R[(size_t)j * n + j] < 0.0 ? -1.0 : 1.0;
        __syncthreads();
        if (own)
            for (int k = 0; k <= j; ++k) R[(size_t)k * n + j] *= zs[k];
        __syncthreads();
    }
    // back substitution, one barrier per step: thread (i, 0) owns z_i and reads
    // row i of R (R[i][k] at step k) through a 4-deep register prefetch queue, so
    // the L2 latency of R is off the step chain; the diagonal sits in shared
    // memory and every thread forms b_k = z_k / R_kk itself (no broadcast step).
    double* rdg = zs + n;       // [n] R_kk
    double* bs = zs + 2 * n;    // [n] beta
    if (diag) {
        zs[j] = R[(size_t)j * n + M];
        rdg[j] = R[(size_t)j * n + j];
    }
    __syncthreads();
    auto rowv = [&](int k) { return (diag && k > j) ? R[(size_t)j * n + k] : 0.0; };
    double q0 = rowv(M - 1), q1 = rowv(M - 2), q2 = rowv(M - 3), q3 = rowv(M - 4);
    for (int k = M - 1; k >= 0; --k) {
        const double rjk = q0;
        q0 = q1;
        q1 = q2;
        q2 = q3;
        q3 = rowv(k - 4);
        const double b = zs[k] / rdg[k];   // zs[k] is final: its last update was in step k+1
        if (diag && j < k) zs[j] -= rjk * b;
        if (diag && j == k) bs[k] = b;
        __syncthreads();
    }
    if (diag) beta[j] = bs[j];
    // rho = || R_orig [beta; -1] ||
    double s = 0.0;
    if (own) {
        for (int c = j; c < M; ++c) s += Rorig[(size_t)j * n + c] * bs[c];
        s -= Rorig[(size_t)j * n + M];
    }
    const double rho2 = block_sum(own ? s * s : 0.0, red);
    if (r_smem)
        for (int e = threadIdx.x; e < n * n; e += blockDim.x) Rg[e] = R[e];
    if (threadIdx.x == 0) {
        out->rho = sqrt(rho2);
        out->rmse = sqrt(rho2) / sqrt((double)n_total);
        out->dmin = dmin;
        out->dmax = dmax;
        out->lambda = lambda;
        out->rank_flag = ridge ? 1 : 0;
        out->nonfinite = *flag;
        if (*flag) out->nf_sticky = 1;
        out->n_total = n_total;
    }
}

// ---- wide solve (n = M+1 > 1024: more columns than threads in a CTA) ---------------------
// Same steps as k_tsqr_solve, with each thread owning the columns j = tid,
// tid + nt, ...; the ridge rows sqrt(lambda)(I|0) are written to slab 1 and
// folded into slab 0 by k_tsqr_merge_wy (a zero slab folds as the identity:
// every reflector has s2 = 0, g = 0), then k_solve_wide_finish re-normalises
// the signs and back-substitutes.  Reading R18/R19 as in k_tsqr_solve.
__device__ void wide_sign_normalise(double* __restrict__ R, int n, double* zs) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) zs[j] = R[(size_t)j * n + j] < 0.0 ? -1.0 : 1.0;
    __syncthreads();
    for (int j = threadIdx.x; j < n; j += blockDim.x)
        for (int k = 0; k <= j; ++k) R[(size_t)k * n + j] *= zs[k];
    __syncthreads();
}

__global__ void __launch_bounds__(1024, 1)
    k_solve_wide_prep(double* __restrict__ R, double* __restrict__ Rridge, double* __restrict__ Rorig, int M, int n,
                      SolveDev* __restrict__ out) {
    extern __shared__ __align__(16) double zs[];
    __shared__ double red[32];
    wide_sign_normalise(R, n, zs);
    double dmn = INFINITY, dmx = 0.0, f2 = 0.0;
    for (int j = threadIdx.x; j < M; j += blockDim.x) {
        const double d = fabs(R[(size_t)j * n + j]);
        dmn = fmin(dmn, d);
        dmx = fmax(dmx, d);
        for (int k = 0; k <= j; ++k) f2 += R[(size_t)k * n + j] * R[(size_t)k * n + j];
    }
    const double dmin = block_min(dmn, red), dmax = block_max(dmx, red), fro2 = block_sum(f2, red);
    const bool ridge = !(dmin > DBL_EPSILON * (double)M * dmax);
    const double lambda = ridge ? 1e-8 * fro2 / (double)M : 0.0;
    const double sl = sqrt(lambda);
    for (int64_t e = threadIdx.x; e < (int64_t)n * n; e += blockDim.x) {
        Rorig[e] = R[e];
        const int64_t k = e / n, j = e % n;
        Rridge[e] = (k == j && k < M) ? sl : 0.0;
    }
    if (threadIdx.x == 0) {
        out->dmin = dmin;
        out->dmax = dmax;
        out->lambda = lambda;
        out->rank_flag = ridge ? 1 : 0;
    }
}

// P = n - M outputs: beta[p*M + j]; rho of output p to rho_multi[p] (when non-null), output 0
// also to out->rho / out->rmse.
__global__ void __launch_bounds__(1024, 1)
    k_solve_wide_finish(double* __restrict__ R, const double* __restrict__ Rorig, int M, int n, long long n_total,
                        const int* __restrict__ flag, double* __restrict__ beta, SolveDev* __restrict__ out,
                        double* __restrict__ rho_multi) {
    extern __shared__ __align__(16) double zs[];
    __shared__ double red[32];
    __shared__ double bk;
    wide_sign_normalise(R, n, zs);
    for (int p = 0; p < n - M; ++p) {
        const int col = M + p;
        for (int j = threadIdx.x; j < M; j += blockDim.x) zs[j] = R[(size_t)j * n + col];
        __syncthreads();
        for (int k = M - 1; k >= 0; --k) {
            if (threadIdx.x == 0) bk = zs[k] / R[(size_t)k * n + k];
            __syncthreads();
            for (int j = threadIdx.x; j < k; j += blockDim.x) zs[j] -= R[(size_t)j * n + k] * bk;
            if (threadIdx.x == 0) zs[k] = bk;
            __syncthreads();
        }
        double s2 = 0.0;
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            double s = 0.0;
            for (int c = j; c < M; ++c) s += Rorig[(size_t)j * n + c] * zs[c];
            s -= Rorig[(size_t)j * n + col];
            s2 += s * s;
            if (j < M) beta[(size_t)p * M + j] = zs[j];
        }
        const double rho2 = block_sum(s2, red);   // ends with a barrier: zs may be reused
        if (threadIdx.x == 0) {
            if (rho_multi) rho_multi[p] = sqrt(rho2);
            if (p == 0) {
                out->rho = sqrt(rho2);
                out->rmse = sqrt(rho2) / sqrt((double)n_total);
            }
        }
    }
    if (threadIdx.x == 0) {
        out->nonfinite = *flag;
        if (*flag) out->nf_sticky = 1;
        out->n_total = n_total;
    }
}

// ---- blocked compact-WY fold (k_tsqr_leaf_wy / k_tsqr_merge_wy) ------------------------
// The north star's "blocked Householder TSQR: panel factorisation with warp-level
// reductions, trailing update as a blocked-reflector update".  A tile of ROWS
// rows lives in SHARED memory as fp64 (so 2-4 CTAs fit per SM and one CTA's
// latency-bound panel overlaps another's FMA-bound trailing update); R stays
// in its L2-resident slab.  Per panel of kNBW = 16 columns:
//  1. warp 0 factors [R diag block; tile panel] column by column in registers
//     (lane = (rg, column pair); reductions are 4-lane butterflies over rg;
//     no block barrier inside the panel) and leaves the reflector tails v_i in
//     the tile's panel columns, (g_i, u0_i) and the R block in shared memory;
//  2. all threads form G = striu(V^T V);
//  3. every trailing column pair applies Q^T = I + U T'^T U^T at once:
//     W = U^T C,  W' = T'^T W,  C_R += u0 W',  C_A += V W',  where the
//     UT transform gives T'^T = (diag(1/g) - striu(U^T U))^{-T}, so W' follows
//     from a 16-step forward substitution per column and T' is never formed
//     (u_a^T u_b = v_a^T v_b for a != b: the R parts of u are distinct unit rows).
constexpr int kNBW = 16;

__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Shared-memory load the compiler may not hoist (keeps the 16 u0 / G values
// out of registers across the trailing loops).
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ double lds_nohoist(const double* p) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)));
    return v;
}

__host__ __device__ constexpr int wy_ldc(int n) { return (n + 7) & ~7; }   // >= n, whole 8-column MMA tiles
__host__ __device__ constexpr size_t wy_smem_bytes(int rows, int n) {
    return ((size_t)rows * wy_ldc(n) + kNBW * kNBW * 3 + 4 * kNBW) * sizeof(double);
}

// rsqrt / rcp: hardware approximation + two Newton steps (full fp64 accuracy;
// measured ~15% shorter than IEEE sqrt + div on the panel's critical path).
// Operands here are norms of H-sized data, far from the approximation's
// exponent limits (the 1e-280 guard above keeps beta*u0 normal).
__device__ __forceinline__ double rsqrt_nr(double t) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t));
    y = y * fma(-0.5 * t * y, y, 1.5);
    return y * fma(-0.5 * t * y, y, 1.5);
}
__device__ __forceinline__ double rcp_nr(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
    e = fma(-d, r, 1.0);
    return fma(r, e, r);
}

// fp64 warp shuffles as two explicit 32-bit halves (the generic double
// shuffle made ptxas land the halves swapped and fix them with three dependent
// LOP3 XORs per value -- on the panel's critical path; profiles/r02).
__device__ __forceinline__ double shfl_idx_d(double v, int src) {
    const int lo = __shfl_sync(0xffffffffu, __double2loint(v), src);
    const int hi = __shfl_sync(0xffffffffu, __double2hiint(v), src);
    return __hiloint2double(hi, lo);
}
__device__ __forceinline__ double shfl_xor_d(double v, int m) {
    const int lo = __shfl_xor_sync(0xffffffffu, __double2loint(v), m);
    const int hi = __shfl_xor_sync(0xffffffffu, __double2hiint(v), m);
    return __hiloint2double(hi, lo);
}

// Panel factorisation by one warp.  Lane = (row group rg, column pair cp):
// rows rg, rg+4, ... of panel columns 2cp, 2cp+1 in registers.  Per column i
// the critical path is ONE shuffle round (v = column i from its owner lanes)
// and ONE 2-level butterfly that reduces |v|^2 and both dot products v^T a
// together; every lane then forms the reflector itself from identical bits
// (commutative butterfly sums), so g, u0 and beta need no broadcast.  Columns
// are processed in pairs with the parity a compile-time constant (no per-column
// register selects), and the per-column stores (Gram entries, R row, the
// coefficients) are predicated, off the dependency chain.
template <int ROWS>
__device__ __noinline__ void wy_panel(double* __restrict__ C, int LDC, int p, int nbp, double* Rd, double* cgv,
                                      double* cuv, double* Gp) {
    constexpr int RPL = ROWS / 4;   // rows per lane: rows rg, rg+4, ... (interleaved: no bank conflicts)
    const int lane = threadIdx.x & 31, rg = lane >> 3, cp = lane & 7;
    const int c0 = 2 * cp, c1 = c0 + 1;
    double a[2][RPL];
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
        const double* row = C + (size_t)(rg + 4 * r) * LDC + p;
        a[0][r] = c0 < nbp ? row[c0] : 0.0;
        a[1][r] = c1 < nbp ? row[c1] : 0.0;
    }
    // Gram matrix G = striu(V^T V) of this panel for the trailing update: zero here,
    // strict-upper entries filled below from the butterfly sums (see w[0] / w[1])
#pragma unroll
    for (int t = 0; t < kNBW * kNBW / 32; ++t) Gp[lane + 32 * t] = 0.0;
    __syncwarp();
    double* const g_row0 = Gp + c0 * kNBW;   // G[c0][.], G[c1][.] = g_row0[kNBW + .]
    double* const rd_c = Rd + c0;            // R[i][c0] = rd_c[i * kNBW], R[i][c1] = rd_c[i * kNBW + 1]
    // R entries of row i are read one column ahead: row i+1 is untouched until reflector i+1
    double x0n = Rd[0], rdn[2] = {rd_c[0], rd_c[1]};

    auto step = [&](auto par, const int i) {
        constexpr int PAR = decltype(par)::value;   // column i = 2 * (i >> 1) + PAR
        const int src = (lane & 24) | (i >> 1);     // owner lane of column i with this lane's rows
        const double x0 = x0n, rd0 = rdn[0], rd1 = rdn[1];
        if (i + 1 < kNBW) {
            x0n = Rd[(i + 1) * (kNBW + 1)];
            rdn[0] = rd_c[(i + 1) * kNBW];
            rdn[1] = rd_c[(i + 1) * kNBW + 1];
        }
        double v[RPL];
#pragma unroll
        for (int r = 0; r < RPL; ++r) v[r] = shfl_idx_d(a[PAR][r], src);
        double s2a = 0.0, s2b = 0.0, w0 = 0.0, w0b = 0.0, w1 = 0.0, w1b = 0.0;
#pragma unroll
        for (int r = 0; r < RPL; r += 2) {
            s2a = fma(v[r], v[r], s2a);
            s2b = fma(v[r + 1], v[r + 1], s2b);
            w0 = fma(v[r], a[0][r], w0);
            w0b = fma(v[r + 1], a[0][r + 1], w0b);
            w1 = fma(v[r], a[1][r], w1);
            w1b = fma(v[r + 1], a[1][r + 1], w1b);
        }
        double s2 = s2a + s2b;
        w0 += w0b;
        w1 += w1b;
        s2 += shfl_xor_d(s2, 8);
        w0 += shfl_xor_d(w0, 8);
        w1 += shfl_xor_d(w1, 8);
        s2 += shfl_xor_d(s2, 16);
        w0 += shfl_xor_d(w0, 16);
        w1 += shfl_xor_d(w1, 16);
        // columns c < i hold their final reflector vectors, so w = v_c . v_i = G[c][i]
        if (rg == 0 && c0 < i) g_row0[i] = w0;
        if (rg == 0 && c1 < i) g_row0[kNBW + i] = w1;
        // ---- reflector of panel column i (make_reflector semantics): s2 == 0 or
        // t <= 1e-280 is H = I (|beta u0| lies in [t, 2t]); testing t also keeps a
        // subnormal t away from rsqrt.approx.ftz, which would flush it to 0 (NaN
        // reflector) -- it occurs in deep noise cascades of rank-deficient partial R.
        // Branch-free (every lane takes the same path): evaluate on a safe t, then
        // select H = I.
        const double t = fma(x0, x0, s2);
        const bool refl_ok = s2 != 0.0 && t > 1e-280;
        const double ts = refl_ok ? t : 1.0;
        const double rs = rsqrt_nr(ts);
        const double bt = -(x0 >= 0.0 ? 1.0 : -1.0) * (ts * rs);
        const double uu = x0 - bt;
        const bool app = refl_ok && fabs(bt * uu) > 1e-280;
        const double gg = -rs * rs * rcp_nr(1.0 + fabs(x0) * rs);   // = 1 / (beta u0)
        const double g = app ? gg : 0.0, u0 = app ? uu : 0.0;
        if (lane == 0) {   // coefficients and R_ii (off the chain: nothing reads them in this panel)
            cgv[i] = g;
            cuv[i] = u0;
            if (app) Rd[i * (kNBW + 1)] = bt;
        }
        // ---- apply H_i to the panel columns right of i: W_j = u0 R[i][j] + v^T a_j
        // (unconditionally: f = 0 when H_i = I or the column is not right of i)
        const bool l0 = c0 > i && c0 < nbp, l1 = c1 > i && c1 < nbp;
        const double f0 = l0 ? g * fma(u0, rd0, w0) : 0.0;
        const double f1 = l1 ? g * fma(u0, rd1, w1) : 0.0;
#pragma unroll
        for (int r = 0; r < RPL; ++r) {
            a[0][r] = fma(f0, v[r], a[0][r]);
            a[1][r] = fma(f1, v[r], a[1][r]);
        }
        if (rg == 0 && app && l0) rd_c[i * kNBW] = fma(f0, u0, rd0);
        if (rg == 0 && app && l1) rd_c[i * kNBW + 1] = fma(f1, u0, rd1);
    };
#pragma unroll 1
    for (int i = 0; i < nbp; i += 2) {
        step(std::integral_constant<int, 0>{}, i);
        if (i + 1 < nbp) step(std::integral_constant<int, 1>{}, i + 1);
    }
    // the reflector vectors: lane (rg, cp) holds final columns 2cp, 2cp+1 of its rows
#pragma unroll
    for (int r = 0; r < RPL; ++r) {
        double* row = C + (size_t)(rg + 4 * r) * LDC + p;
        if (c0 < nbp) row[c0] = a[0][r];
        if (c1 < nbp) row[c1] = a[1][r];
    }
    __syncwarp();
}

// f64 tensor-core MMA, m8n8k4: A row-major 8x4 (lane: A[lane/4][lane%4]), B col 4x8
// (lane: B[lane%4][lane/4]), C/D 8x8 (lane: D[lane/4][2(lane%4) + {0,1}]).
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// Trailing update of columns [pe, n) by the panel's block reflector, on the
// f64 tensor cores: each warp takes 8-column tiles;
//   GEMM 1  W (16 x 8) = u0 o R[p.., j] + V^T C        (K = ROWS)
//   solve   W' = T'^T W (16-step forward substitution across the 8 lanes of a column)
//   R[p+i][j] += u0_i W'_i
//   GEMM 2  C (ROWS x 8) += V W'                        (K = 16)
// A warp with two or more tiles left runs two of them in lockstep (NT = 2): each
// tile is a latency-bound chain (8 dependent MMA k-steps, the 16-step
// substitution, 4 more), so two interleaved chains nearly double the warp's
// throughput (measured: the first panel steps of a fold are trailing bound).
template <int ROWS, int NT>
__device__ __forceinline__ void wy_trailing_tiles(double* __restrict__ C, int LDC, int n, int p, const int (&j0)[NT],
                                                  const bool (&ok)[NT], double* __restrict__ R, const double* Gs,
                                                  const double* cgv, const double (&u0r)[2]) {
    constexpr int KS1 = ROWS / 4, MT2 = ROWS / 8;
    const int lane = threadIdx.x & 31;
    const int gid = lane >> 2, tig = lane & 3;
    const double* Vt = C + p;   // V[r][i] = Vt[r * LDC + i]
    double rcur[NT][2][2], d[NT][2][2];
#pragma unroll
    for (int q = 0; q < NT; ++q)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int j = j0[q] + 2 * tig + e;
                rcur[q][mt][e] = (ok[q] && j < n) ? __ldcg(R + (size_t)(p + 8 * mt + gid) * n + j) : 0.0;
                d[q][mt][e] = 0.0;   // the R term joins after GEMM 1: its L2 latency overlaps the MMAs
            }
#pragma unroll 4
    for (int ks = 0; ks < KS1; ++ks) {
        const double va = Vt[(size_t)(4 * ks + tig) * LDC + gid], vb = Vt[(size_t)(4 * ks + tig) * LDC + 8 + gid];
#pragma unroll
        for (int q = 0; q < NT; ++q) {
            const double b = C[(size_t)(4 * ks + tig) * LDC + j0[q] + gid];
            dmma(d[q][0], va, b);
            dmma(d[q][1], vb, b);
        }
    }
#pragma unroll
    for (int q = 0; q < NT; ++q)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int e = 0; e < 2; ++e) d[q][mt][e] = fma(u0r[mt], rcur[q][mt][e], d[q][mt][e]);
    // W'_l = g_l (W_l + sum_{m<l} G[m][l] W'_m): finalise row l, push it down
#pragma unroll
    for (int l = 0; l < kNBW; ++l) {
        const int mt = l >> 3;
        if (gid == (l & 7)) {
            const double gl = lds_nohoist(cgv + l);
#pragma unroll
            for (int q = 0; q < NT; ++q) {
                d[q][mt][0] *= gl;
                d[q][mt][1] *= gl;
            }
        }
        if (l + 1 < kNBW) {
            double w0[NT], w1[NT];
#pragma unroll
            for (int q = 0; q < NT; ++q) {
                w0[q] = __shfl_sync(0xffffffffu, d[q][mt][0], (l & 7) * 4 + tig);
                w1[q] = __shfl_sync(0xffffffffu, d[q][mt][1], (l & 7) * 4 + tig);
            }
#pragma unroll
            for (int m2 = mt; m2 < 2; ++m2) {
                const int i = 8 * m2 + gid;
                if (i > l) {
                    const double gg = lds_nohoist(Gs + l * kNBW + i);
#pragma unroll
                    for (int q = 0; q < NT; ++q) {
                        d[q][m2][0] = fma(gg, w0[q], d[q][m2][0]);
                        d[q][m2][1] = fma(gg, w1[q], d[q][m2][1]);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < NT; ++q)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int j = j0[q] + 2 * tig + e;
                if (ok[q] && j < n) R[(size_t)(p + 8 * mt + gid) * n + j] = fma(u0r[mt], d[q][mt][e], rcur[q][mt][e]);
            }
    // B fragments of W': B[k][n] = W'[4 kt + k][n], lane (k = tig, n = gid); W' row
    // i = 4 kt + tig lives in D tile kt/2 on lanes (i % 8) * 4 + n / 2, element n % 2
    double b2[NT][4];
#pragma unroll
    for (int kt = 0; kt < 4; ++kt) {
        const int srcl = ((4 * kt + tig) & 7) * 4 + (gid >> 1);
#pragma unroll
        for (int q = 0; q < NT; ++q) {
            const double x0 = __shfl_sync(0xffffffffu, d[q][kt >> 1][0], srcl);
            const double x1 = __shfl_sync(0xffffffffu, d[q][kt >> 1][1], srcl);
            b2[q][kt] = (gid & 1) ? x1 : x0;
        }
    }
#pragma unroll 2
    for (int mt = 0; mt < MT2; ++mt) {
        const double* vrow = Vt + (size_t)(8 * mt + gid) * LDC + tig;
        double vk[4];
#pragma unroll
        for (int kt = 0; kt < 4; ++kt) vk[kt] = vrow[4 * kt];
#pragma unroll
        for (int q = 0; q < NT; ++q) {
            if (!ok[q]) continue;
            double2* cp2 = reinterpret_cast<double2*>(C + (size_t)(8 * mt + gid) * LDC + j0[q] + 2 * tig);
            const double2 cv = *cp2;
            double acc[2] = {cv.x, cv.y};
#pragma unroll
            for (int kt = 0; kt < 4; ++kt) dmma(acc, vk[kt], b2[q][kt]);
            *cp2 = make_double2(acc[0], acc[1]);
        }
    }
}

template <int ROWS, bool ILP2>
__device__ __forceinline__ void wy_trailing(double* __restrict__ C, int LDC, int n, int p, int pe, int jend,
                                            int warp, int nw, double* __restrict__ R, const double* Gs,
                                            const double* cgv, const double* cuv) {
    const int gid = (threadIdx.x & 31) >> 2;
    const double u0r[2] = {cuv[gid], cuv[8 + gid]};
    int j0 = pe + 8 * warp;
    if constexpr (ILP2) {
        for (; j0 + 8 * nw < jend; j0 += 16 * nw) {   // two tiles in lockstep
            const int jj[2] = {j0, j0 + 8 * nw};
            const bool ok[2] = {true, true};
            wy_trailing_tiles<ROWS, 2>(C, LDC, n, p, jj, ok, R, Gs, cgv, u0r);
        }
    }
    for (; j0 < jend; j0 += 8 * nw) {
        const int jj[1] = {j0};
        const bool ok[1] = {true};
        wy_trailing_tiles<ROWS, 1>(C, LDC, n, p, jj, ok, R, Gs, cgv, u0r);
    }
}

// Fold the shared-memory tile C (ROWS x n, columns < k0 zero) into R (n x n),
// with one-panel look-ahead: while warps 1.. apply panel p's block reflector to
// columns beyond panel p+1, warp 0 applies it to panel p+1's 16 columns and
// factors panel p+1 -- the latency-bound panel chain overlaps the FMA-bound
// trailing update.  Coefficients and G = striu(V^T V) (written by the panel
// warp from its butterfly sums) are double-buffered by panel parity.  (wy_fold
// follows the R diagonal-block helpers below.)

// R diagonal block of panel p (16 x 16, upper part) <-> registers / shared memory.
// The panel warp reads the NEXT panel's block one step early (its R rows are
// not touched by the current step), so the load latency leaves the panel chain.
__device__ __forceinline__ void rd_load(const double* __restrict__ R, int n, int p, double (&rr)[8]) {
    const int lane = threadIdx.x & 31, nbp = min(kNBW, n - p);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        const int e = lane + 32 * t, i = e / kNBW, c = e % kNBW;
        rr[t] = (p < n && i < nbp && c < nbp && c >= i) ? __ldcg(R + (size_t)(p + i) * n + p + c) : 0.0;
    }
}
__device__ __forceinline__ void rd_put(double* Rd, const double (&rr)[8]) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int t = 0; t < 8; ++t) Rd[lane + 32 * t] = rr[t];
    __syncwarp();
}

template <int ROWS>
__device__ __forceinline__ void wy_panel_rd(double* C, int LDC, int n, int p, double* __restrict__ R, double* Rd,
                                            double* cgv, double* cuv, double* Gp) {
    const int lane = threadIdx.x & 31, nbp = min(kNBW, n - p);
    wy_panel<ROWS>(C, LDC, p, nbp, Rd, cgv, cuv, Gp);
    for (int e = lane; e < kNBW * kNBW; e += 32) {
        const int i = e / kNBW, c = e % kNBW;
        if (i < nbp && c < nbp && c >= i) R[(size_t)(p + i) * n + p + c] = Rd[e];
    }
}

// A warp group that runs one fold: threads [base, base + threads) of the CTA,
// its own named barriers (step barrier: 0 = the whole CTA via __syncthreads),
// and the exclusive end of the panels it factors (p_end = n: the whole fold).
struct WyGroup {
    int base, threads, bar_step, bar_la, p_end;
};
__device__ __forceinline__ WyGroup wy_whole_cta(int n) { return WyGroup{0, (int)blockDim.x, 0, 1, n}; }

// ILP2: two trailing tiles per warp in lockstep (measured per kernel shape: faster
// for the 32-row single-chain leaf (C4 77.1 -> 76.0 ms) and the 16-row two-phase
// leaf (2M x 1025: 918 -> 854 ms); slower for 32-row two-phase CTAs and 64/96-row tiles)
template <int ROWS, bool ILP2 = false>
__device__ void wy_fold(double* __restrict__ C, int LDC, int n, int k0, double* __restrict__ R, double* Gs,
                        double* Rd, double* cgv, double* cuv, int pw, const int* pred_prog = nullptr,
                        int* my_prog = nullptr, bool la_wait = false, WyGroup grp = WyGroup{0, 0, 0, 1, -1}) {
    if (grp.threads == 0) grp = wy_whole_cta(n);
    const int gtid = (int)threadIdx.x - grp.base;
    const int warp = gtid >> 5, nw = grp.threads >> 5;
    const int tw = warp < pw ? warp : warp - 1;
    const bool lane0 = (gtid & 31) == 0 && warp == pw;
    auto step_sync = [&]() {
        if (grp.bar_step == 0) __syncthreads();
        else named_bar_sync(grp.bar_step, grp.threads);
    };
    // Pipelined merge (k_tsqr_merge_wy_par): the fold of the previous row chunk into
    // the same R publishes the number of panel steps it has completed; step p of
    // this fold touches R rows p .. p+47 (trailing rows, look-ahead panel, diagonal
    // prefetch), which the predecessor no longer writes once it has completed
    // panel step p/16 + 2.
    const int npan = (n + kNBW - 1) / kNBW;
    auto wait_pred = [&](int need) {
        if (!pred_prog) return;
        need = min(need, npan);
        if (gtid == 0)
            while (ld_acquire_gpu(pred_prog) < need) __nanosleep(64);
        step_sync();
    };
    auto publish = [&](int v) {
        if (my_prog && gtid == 0) {
            __threadfence();
            st_release_gpu(my_prog, v);
        }
    };
    // the R diagonal block of panel q is read only for panels this group factors
    auto rd_next = [&](int q, double (&rr)[8]) {
        if (q < grp.p_end) rd_load(R, n, q, rr);
    };
    int p = k0, buf = 0;
    double rdn[8];   // panel warp: next panel's R diagonal block
    wait_pred(k0 / kNBW + 2);
    if (warp == pw) {
        rd_load(R, n, p, rdn);
        rd_put(Rd, rdn);
        rd_next(p + kNBW, rdn);
        wy_panel_rd<ROWS>(C, LDC, n, p, R, Rd, cgv, cuv, Gs);
    }
    step_sync();
    for (;;) {
        const int pe = p + min(kNBW, n - p);
        if (pe >= n) break;   // no trailing columns (so below nbp == kNBW)
        const bool fact = pe < grp.p_end;   // does this group factor panel pe (look-ahead)?
        wait_pred(p / kNBW + 3);
        if (lane0) qr_ev(0, p);
        const int nbn = min(kNBW, n - pe);
        double *G0 = Gs + buf * kNBW * kNBW, *g0 = cgv + buf * kNBW, *u0 = cuv + buf * kNBW;
        if (nw == 1) {
            wy_trailing<ROWS, ILP2>(C, LDC, n, p, pe, n, 0, 1, R, G0, g0, u0);
            __syncwarp();
            if (fact) {
                rd_put(Rd, rdn);
                rd_next(pe + kNBW, rdn);
                wy_panel_rd<ROWS>(C, LDC, n, pe, R, Rd, cgv + (buf ^ 1) * kNBW, cuv + (buf ^ 1) * kNBW,
                                  Gs + (buf ^ 1) * kNBW * kNBW);
            }
        } else if (warp == pw) {
            // look-ahead: wait until panel p+1's columns carry panel p's update, factor it
            if (fact) {
                rd_put(Rd, rdn);
                rd_next(pe + kNBW, rdn);
            }
            named_bar_sync(grp.bar_la, grp.threads);
            if (lane0) qr_ev(1, p);
            if (fact)
                wy_panel_rd<ROWS>(C, LDC, n, pe, R, Rd, cgv + (buf ^ 1) * kNBW, cuv + (buf ^ 1) * kNBW,
                                  Gs + (buf ^ 1) * kNBW * kNBW);
            if (lane0) qr_ev(5, p);
        } else {
            wy_trailing<ROWS, ILP2>(C, LDC, n, p, pe, pe + nbn, tw, nw - 1, R, G0, g0, u0);   // panel p+1's columns first
            if (tw == 0 && (gtid & 31) == 0) qr_ev(3, p);
            __threadfence_block();
            // warps without a look-ahead tile wait with the panel warp so the
            // look-ahead chain is not slowed by their trailing work
            if (la_wait && 8 * tw >= nbn) named_bar_sync(grp.bar_la, grp.threads);
            else named_bar_arrive(grp.bar_la, grp.threads);
            wy_trailing<ROWS, ILP2>(C, LDC, n, p, pe + nbn, n, tw, nw - 1, R, G0, g0, u0);
            if (tw == 0 && (gtid & 31) == 0) qr_ev(4, p);
        }
        step_sync();
        if (lane0) qr_ev(2, p);
        publish(p / kNBW + 1);
        if (!fact) break;     // phase end: panels >= p_end belong to the next group
        p = pe;
        buf ^= 1;   // the panel warp wrote G of the new panel p with its reflectors
    }
    publish(npan);
}

// Panel warp of this CTA.  mode 1 (default): the warp of this CTA that sits on
// SM sub-partition 0 (%warpid & 3 == 0), so the latency-bound panels of all
// co-resident CTAs share SMSP 0 and no trailing update's DMMA stream (16 FP64-pipe
// cycles per m8n8k4) delays their dependent DFMA/MUFU chain; the trailing warps
// own SMSPs 1-3.  mode 0: co-resident CTAs take distinct warp indices (per-SM
// arrival counters, sm_slot zeroed before the launch), one panel per SMSP.
__device__ __forceinline__ int wy_panel_warp(int* sm_slot, int mode) {
    __shared__ int pw_s;
    const int nw = (int)(blockDim.x >> 5);
    if (threadIdx.x == 0) pw_s = nw;
    __syncthreads();
    if (mode == 1) {
        unsigned wid;
        asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
        if ((threadIdx.x & 31) == 0 && (wid & 3) == 0) atomicMin(&pw_s, (int)(threadIdx.x >> 5));
        __syncthreads();
        const int pw = pw_s;
        __syncthreads();
        if (pw < nw) return pw;
    }
    if (threadIdx.x == 0) {
        int local = (int)blockIdx.x;
        if (sm_slot) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            local = atomicAdd(sm_slot + (smid & 1023), 1);
        }
        pw_s = local % nw;
    }
    __syncthreads();
    return pw_s;
}

// NW = 4 warps (n <= 320): 3 CTAs of 32-row tiles share an SM, so the register
// cap is 65536 / 384 = 168 (the 2-CTA bound of 128 spilled the panel warp's R
// prefetch to local memory right behind its load: measured, profiles/r02).
template <int ROWS, int NW>
__global__ void __launch_bounds__(32 * NW, (NW == 4 && ROWS <= 32) ? 3 : ((NW <= 6 && (ROWS == 48 || ROWS == 40)) ? 2 : 1))
    k_tsqr_leaf_wy(const float* __restrict__ H, int64_t ldh, const float* __restrict__ Y, int64_t ldy, int P,
                   int64_t N, int M, double* __restrict__ Rws, int64_t rows_per_cta, int* __restrict__ flag,
                   int* sm_slot, int la_wait, int pw_mode) {
    extern __shared__ __align__(16) double wsm[];
    // columns [0, M) of the tile are H, [M, M + P) the P outputs Y[row][0..P-1] (row stride ldy)
    const int n = M + P, LDC = wy_ldc(n), tid = threadIdx.x, nt = blockDim.x;
    double* C = wsm;
    double* Gs = C + (size_t)ROWS * LDC;     // [2][16][16]
    double* Rd = Gs + 2 * kNBW * kNBW;       // [16][16]
    double* cgv = Rd + kNBW * kNBW;          // [2][16]
    double* cuv = cgv + 2 * kNBW;            // [2][16]
    double* R = Rws + (size_t)blockIdx.x * n * n;
    for (int64_t e = tid; e < (int64_t)n * n; e += nt) R[e] = 0.0;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
    const int64_t r1 = min(N, r0 + rows_per_cta);
    bool bad = false;
    const int pw = wy_panel_warp(sm_slot, pw_mode);
    // 16-B vector loads of H when rows allow it, issued in batches of 8 per
    // thread so the tile load is not a chain of dependent HBM round trips
    const bool vec = (M % 4 == 0) && (ldh % 4 == 0) && ((reinterpret_cast<uintptr_t>(H) & 15) == 0);
    const int M4 = M / 4, tail = LDC - M;
    for (int64_t base = r0; base < r1; base += ROWS) {
        if (vec) {
            constexpr int B = 8;
            for (int e0 = tid; e0 < ROWS * M4; e0 += nt * B) {
                float4 v[B];
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const int e = e0 + b * nt, r = e / M4, q = e - r * M4;
                    v[b] = (e < ROWS * M4 && base + r < r1)
                               ? __ldcs(reinterpret_cast<const float4*>(H + (base + r) * ldh) + q)
                               : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int b = 0; b < B; ++b) {
                    const int e = e0 + b * nt, r = e / M4, q = e - r * M4;
                    if (e < ROWS * M4) {
                        bad |= !(isfinite(v[b].x) && isfinite(v[b].y) && isfinite(v[b].z) && isfinite(v[b].w));
                        double2* d = reinterpret_cast<double2*>(C + (size_t)r * LDC + 4 * q);
                        d[0] = make_double2(v[b].x, v[b].y);
                        d[1] = make_double2(v[b].z, v[b].w);
                    }
                }
            }
            for (int e = tid; e < ROWS * tail; e += nt) {   // Y columns, zero padding
                const int r = e / tail, c = M + (e - r * tail);
                const int64_t row = base + r;
                const float x = (c < n && row < r1) ? __ldg(Y + row * ldy + (c - M)) : 0.0f;
                bad |= !isfinite(x);
                C[(size_t)r * LDC + c] = (double)x;
            }
        } else {
            for (int r = 0; r < ROWS; ++r) {
                const int64_t row = base + r;
                for (int c = tid; c < LDC; c += nt) {
                    float x = 0.0f;
                    if (row < r1 && c < n) x = c < M ? __ldg(H + row * ldh + c) : __ldg(Y + row * ldy + (c - M));
                    bad |= !isfinite(x);
                    C[(size_t)r * LDC + c] = (double)x;
                }
            }
        }
        __syncthreads();
#ifdef ELM_WY48_NO_ILP
        wy_fold<ROWS, ROWS == 32>(C, LDC, n, 0, R, Gs, Rd, cgv, cuv, pw, nullptr, nullptr, la_wait != 0);
#else
        wy_fold<ROWS, ROWS == 32 || ROWS == 48 || ROWS == 40 || ROWS == 24>(C, LDC, n, 0, R, Gs, Rd, cgv, cuv, pw,
                                                                             nullptr, nullptr, la_wait != 0);
#endif
    }
    if (bad) atomicOr(flag, 1);
}

// ---- two-phase pipelined WY leaf ----------------------------------------------------
// The fold of a tile is a chain of npan panel steps (the panel warp's dependency
// latency); the trailing warps wait on it most of the time, and one 32-row fp64
// tile per chain fills a third of shared memory.  Split the chain: group A
// factors panels [0, p_split) of tile k (trailing updates over all columns)
// while group B factors panels [p_split, n) of tile k-1 -- the two touch
// disjoint R rows, so they need no synchronisation until the period ends.  A
// tile past phase A only needs its columns >= p_split, so group B's buffer is
// half the size: two chains for 1.5 tiles of shared memory.
__host__ __device__ constexpr int wy2_split(int n) { return 16 * (((n + kNBW - 1) / kNBW + 1) / 2); }
__host__ __device__ constexpr size_t wy2_aux_doubles() { return (size_t)kNBW * kNBW * 3 + 4 * kNBW; }
__host__ __device__ constexpr size_t wy2_smem_bytes(int rows, int n) {
    return ((size_t)rows * wy_ldc(n) + (size_t)rows * wy_ldc(n - wy2_split(n)) + 2 * wy2_aux_doubles()) * sizeof(double);
}

template <int ROWS, int NWA, int NWB>
__global__ void __launch_bounds__(32 * (NWA + NWB), (NWA + NWB) * 32 * 168 * 2 <= 65536 ? 2 : 1)
    k_tsqr_leaf_wy2(const float* __restrict__ H, int64_t ldh, const float* __restrict__ Y, int64_t ldy, int P,
                    int64_t N, int M, double* __restrict__ Rws, int64_t rows_per_cta, int* __restrict__ flag,
                    int la_wait) {
    extern __shared__ __align__(16) double wsm[];
    const int n = M + P, LDC = wy_ldc(n), ps = wy2_split(n), LDCB = wy_ldc(n - ps);
    double* bufA = wsm;
    double* auxA = bufA + (size_t)ROWS * LDC;
    double* bufB = auxA + wy2_aux_doubles();
    double* auxB = bufB + (size_t)ROWS * LDCB;
    // aux: Gs [2][16][16] | Rd [16][16] | cgv [2][16] | cuv [2][16]
    auto Gs = [](double* a) { return a; };
    auto Rd = [](double* a) { return a + 2 * kNBW * kNBW; };
    auto cg = [](double* a) { return a + 3 * kNBW * kNBW; };
    auto cu = [](double* a) { return a + 3 * kNBW * kNBW + 2 * kNBW; };
    constexpr int TA = 32 * NWA, TB = 32 * NWB;
    const WyGroup gA{0, TA, 2, 1, ps}, gB{TA, TB, 4, 3, n};
    const bool inA = (int)threadIdx.x < TA;
    double* R = Rws + (size_t)blockIdx.x * n * n;
    for (int64_t e = threadIdx.x; e < (int64_t)n * n; e += blockDim.x) R[e] = 0.0;
    const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
    const int64_t r1 = min(N, r0 + rows_per_cta);
    const int64_t ntiles = r1 > r0 ? (r1 - r0 + ROWS - 1) / ROWS : 0;
    bool bad = false;
    const bool vec = (M % 4 == 0) && (ldh % 4 == 0) && ((reinterpret_cast<uintptr_t>(H) & 15) == 0);
    const int M4 = M / 4, tail = LDC - M;
    __syncthreads();
    for (int64_t k = 0; k <= ntiles; ++k) {
        if (inA) {
            if (k < ntiles) {
                const int tid = threadIdx.x, nt = TA;
                const int64_t base = r0 + k * ROWS;
                if (vec) {   // 16-B evict-first loads, 8 in flight per thread
                    constexpr int B = 8;
                    for (int e0 = tid; e0 < ROWS * M4; e0 += nt * B) {
                        float4 v[B];
#pragma unroll
                        for (int b = 0; b < B; ++b) {
                            const int e = e0 + b * nt, r = e / M4, q = e - r * M4;
                            v[b] = (e < ROWS * M4 && base + r < r1)
                                       ? __ldcs(reinterpret_cast<const float4*>(H + (base + r) * ldh) + q)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
#pragma unroll
                        for (int b = 0; b < B; ++b) {
                            const int e = e0 + b * nt, r = e / M4, q = e - r * M4;
                            if (e < ROWS * M4) {
                                bad |= !(isfinite(v[b].x) && isfinite(v[b].y) && isfinite(v[b].z) && isfinite(v[b].w));
                                double2* d = reinterpret_cast<double2*>(bufA + (size_t)r * LDC + 4 * q);
                                d[0] = make_double2(v[b].x, v[b].y);
                                d[1] = make_double2(v[b].z, v[b].w);
                            }
                        }
                    }
                    for (int e = tid; e < ROWS * tail; e += nt) {   // Y columns, zero padding
                        const int r = e / tail, c = M + (e - r * tail);
                        const int64_t row = base + r;
                        const float x = (c < n && row < r1) ? __ldg(Y + row * ldy + (c - M)) : 0.0f;
                        bad |= !isfinite(x);
                        bufA[(size_t)r * LDC + c] = (double)x;
                    }
                } else {
                    for (int r = 0; r < ROWS; ++r) {
                        const int64_t row = base + r;
                        for (int c = tid; c < LDC; c += nt) {
                            float x = 0.0f;
                            if (row < r1 && c < n) x = c < M ? __ldg(H + row * ldh + c) : __ldg(Y + row * ldy + (c - M));
                            bad |= !isfinite(x);
                            bufA[(size_t)r * LDC + c] = (double)x;
                        }
                    }
                }
                named_bar_sync(gA.bar_step, TA);
                wy_fold<ROWS, ROWS == 16>(bufA, LDC, n, 0, R, Gs(auxA), Rd(auxA), cg(auxA), cu(auxA), 0, nullptr, nullptr,
                              la_wait != 0, gA);
            }
        } else if (k >= 1) {
            // columns >= ps of tile k-1 live in bufB (column c at bufB[r * LDCB + c - ps])
            wy_fold<ROWS, ROWS == 16>(bufB - ps, LDCB, n, ps, R, Gs(auxB), Rd(auxB), cg(auxB), cu(auxB), 0, nullptr, nullptr,
                          la_wait != 0, gB);
        }
        __syncthreads();
        if (k < ntiles) {   // tile k moves on to phase B
            const int w = LDC - ps;
            for (int e = threadIdx.x; e < ROWS * w; e += blockDim.x) {
                const int r = e / w, c = e - r * w;
                bufB[(size_t)r * LDCB + c] = bufA[(size_t)r * LDC + ps + c];
            }
        }
        __syncthreads();
    }
    if (bad) atomicOr(flag, 1);
}

template <int ROWS, int NW>
__global__ void __launch_bounds__(32 * NW, (NW == 4 && ROWS <= 32) ? 3 : 1)
    k_tsqr_merge_wy(double* __restrict__ Rws, int64_t slabs, int64_t stride, int n, const int* gate = nullptr) {
    extern __shared__ __align__(16) double wsm[];
    const int64_t c = (int64_t)blockIdx.x * 2 * stride, partner = c + stride;
    if (partner >= slabs) return;
    if (gate && *gate == 0) return;   // wide solve: no ridge rows to fold (rank_flag == 0)
    const int LDC = wy_ldc(n), tid = threadIdx.x, nt = blockDim.x;
    double* C = wsm;
    double* Gs = C + (size_t)ROWS * LDC;     // [2][16][16]
    double* Rd = Gs + 2 * kNBW * kNBW;       // [16][16]
    double* cgv = Rd + kNBW * kNBW;          // [2][16]
    double* cuv = cgv + 2 * kNBW;            // [2][16]
    double* Ra = Rws + (size_t)c * n * n;
    const double* Rb = Rws + (size_t)partner * n * n;
    for (int s = 0; s * ROWS < n; ++s) {
        for (int r = 0; r < ROWS; ++r) {
            const int row = s * ROWS + r;
            for (int cc = tid; cc < LDC; cc += nt)
                C[(size_t)r * LDC + cc] = (row < n && cc < n && cc >= row) ? Rb[(size_t)row * n + cc] : 0.0;
        }
        __syncthreads();
        wy_fold<ROWS>(C, LDC, n, s * ROWS, Ra, Gs, Rd, cgv, cuv, (int)(blockIdx.x % (blockDim.x >> 5)));
    }
}

// Pipelined merge: P CTAs share one pair (R_a <- qr_r([R_a; R_b])); CTA pc folds
// the ROWS-row chunks s = pc, pc + P, ... of R_b in order, each fold waiting on
// the progress counter of chunk s - 1 (a wavefront one to three panel steps
// apart) instead of for the whole previous chunk.  All CTAs of the grid must be
// co-resident: launched cooperatively.  prog: [pairs][kMaxChunks] zeroed ints.
constexpr int kMaxChunks = 128;
template <int ROWS, int NW>
__global__ void __launch_bounds__(32 * NW, (NW == 4 && ROWS <= 32) ? 3 : 1)
    k_tsqr_merge_wy_par(double* __restrict__ Rws, int64_t slabs, int64_t stride, int n, int P, int* prog) {
    extern __shared__ __align__(16) double wsm[];
    const int64_t m = blockIdx.x / P;
    const int pc = (int)(blockIdx.x % P);
    const int64_t c = m * 2 * stride, partner = c + stride;
    if (partner >= slabs) return;
    const int LDC = wy_ldc(n), tid = threadIdx.x, nt = blockDim.x;
    double* C = wsm;
    double* Gs = C + (size_t)ROWS * LDC;     // [2][16][16]
    double* Rd = Gs + 2 * kNBW * kNBW;       // [16][16]
    double* cgv = Rd + kNBW * kNBW;          // [2][16]
    double* cuv = cgv + 2 * kNBW;            // [2][16]
    double* Ra = Rws + (size_t)c * n * n;
    const double* Rb = Rws + (size_t)partner * n * n;
    int* pg = prog + m * kMaxChunks;
    for (int s = pc; s * ROWS < n; s += P) {
        for (int r = 0; r < ROWS; ++r) {
            const int row = s * ROWS + r;
            for (int cc = tid; cc < LDC; cc += nt)
                C[(size_t)r * LDC + cc] = (row < n && cc < n && cc >= row) ? Rb[(size_t)row * n + cc] : 0.0;
        }
        __syncthreads();
        wy_fold<ROWS>(C, LDC, n, s * ROWS, Ra, Gs, Rd, cgv, cuv, (int)(blockIdx.x % (blockDim.x >> 5)),
                      s > 0 ? pg + s - 1 : nullptr, pg + s);
    }
}

// ---- host side ---------------------------------------------------------------------

// Per-column fold variants (n <= 128 by default; any n when forced): n <= 288:
// 2 threads x 24 rows per column (48-row tiles, <= 576 threads); n <= 512:
// 2 x 12 (24-row tiles, <= 1024 threads); else 1 x 12.
enum class Var { P2T24, P2T12, P1T12 };
static Var pick_var(int n) { return n <= 288 ? Var::P2T24 : (n <= 512 ? Var::P2T12 : Var::P1T12); }
static int var_rows(Var v) { return v == Var::P2T24 ? 48 : (v == Var::P2T12 ? 24 : 12); }
static int var_p(Var v) { return v == Var::P1T12 ? 1 : 2; }
static int var_threads(Var v, int n) { return (var_p(v) * n + 31) / 32 * 32; }

template <class F>
static auto dispatch(Var v, F&& f) {
    switch (v) {
    case Var::P2T24: return f(std::integral_constant<int, 24>{}, std::integral_constant<int, 2>{});
    case Var::P2T12: return f(std::integral_constant<int, 12>{}, std::integral_constant<int, 2>{});
    default: return f(std::integral_constant<int, 12>{}, std::integral_constant<int, 1>{});
    }
}

// n = M+1 above this takes the WY leaf/merge and the wide solve (columns > threads).
constexpr int kWideN = 1024;
// Blocked compact-WY leaf + merge (wy_fold).  ELMRNN_TSQR_WY=0/1 overrides the default.
static bool use_wy(const elmrnn* h, int n) {
    if (n > kWideN) return true;   // the only leaf/merge for more columns than CTA threads
    if (h->tune.tsqr_wy >= 0) return h->tune.tsqr_wy != 0;   // testing knob (elmrnn_init_ex)
    // measured (tools/qr_time.py, B200): M = 128 x 1M rows WY 8.6 vs per-column fold
    // 10.4 ms; M = 64 x 100k rows 1.22 vs 0.93 ms
    return n > 128;
}
// Look-ahead isolation in the leaf: trailing warps without a look-ahead tile
// wait for the look-ahead columns with the panel warp instead of competing with
// that chain (measured C4 shape 81.6 -> 80.3 ms; neutral at 8 warps, n > 320).
static int wy_la_wait(int n) { return n <= 320 ? 1 : 0; }
// multi-output [H | Y_1..Y_P] (P > 1) always takes the WY leaf/merge and the wide solve
static bool use_wy_h(const elmrnn* h) { return h->nrhs > 1 || use_wy(h, h->M + h->nrhs); }
static bool wide_solve(const elmrnn* h) { return h->nrhs > 1 || h->M + h->nrhs > kWideN; }
// 448 < n with a 24-row tile within shared memory: the single-chain 12-warp leaf
static bool wide_single(int n) { return n > 448 && wy_smem_bytes(24, n) <= 220 * 1024; }
static int wy_rows(const elmrnn* h, int n) {
    if (const int r = h->tune.wy_rows) {   // testing knob (elmrnn_init_ex)
        if ((r == 96 || r == 64 || r == 48 || r == 40 || r == 32 || r == 24 || r == 16 || r == 8) &&
            wy_smem_bytes(r, n) <= 220 * 1024)
            return r;
    }
    // n <= 160: 64-row tiles (measured M = 128 x 2M rows: 12.9 vs 14.3 ms with 32);
    // 160 < n <= ~288: 48-row tiles, two 6-warp CTAs per SM (1 panel + 5 trailing
    // warps each, panel warps on different SM sub-partitions): C4 shape 75.5 -> 67.3 ms,
    // 500k x 257 13.9 -> 12.2, 2M x 193 25.2 -> 24.0 (tools/qr_time.py knobs; 40-row tiles
    // and 5-warp CTAs slower); larger n: 32-row tiles, 3 CTAs per SM (16/24-row tiles
    // and 4-warp CTAs measured slower at n = 257, 513, 1025: tools/wy_variants.sh)
    if (n <= 160) return 64;
    if (2 * wy_smem_bytes(48, n) <= 227 * 1024) return 48;
    // wide n, single-chain 12-warp CTAs (one per SM) with the tallest tile that fits:
    // 2M x 513 48 rows 135.6 vs two-phase 32-row 140.3 ms; 2M x 1025 24 rows 690 vs
    // two-phase 16-row 849 ms (tools/qr_time.py with the ELMRNN_TSQR_WY_ROWS / ELMRNN_WY_NW knobs); n = 401 keeps the two-phase leaf
    if (wide_single(n)) return wy_smem_bytes(48, n) <= 220 * 1024 ? 48 : 24;
    return wy_smem_bytes(32, n) <= 220 * 1024 ? 32 : 16;
}
// Leaf dynamic shared memory: the tile + coefficients.
static size_t wy_leaf_smem(int rows, int n) { return std::min(wy_smem_bytes(rows, n), (size_t)227 * 1024); }
static int wy_nw(int n) { return n <= 320 ? 4 : 8; }
static int wy_threads(int n) { return 32 * wy_nw(n); }
// leaf warps per CTA: by n, or the testing override
static int wy_leaf_nw(const elmrnn* h, int n) {
    if (h->tune.wy_nw >= 4 && h->tune.wy_nw <= 16) return h->tune.wy_nw;
    return (wide_single(n) && !h->tune.wy_rows) ? 12 : wy_nw(n);
}
template <int RW, class F>
static auto wy_nw_dispatch(int nw, F& f) {
    if (nw == 4) return f(std::integral_constant<int, RW>{}, std::integral_constant<int, 4>{});
    return f(std::integral_constant<int, RW>{}, std::integral_constant<int, 8>{});
}
template <class F>
static auto wy_dispatch(const elmrnn* h, int n, F&& f) {
    const int nw = wy_leaf_nw(h, n);
    switch (wy_rows(h, n)) {
    case 96:
        if (nw == 12) return f(std::integral_constant<int, 96>{}, std::integral_constant<int, 12>{});
        return wy_nw_dispatch<96>(nw, f);
    case 64:
        if (nw == 12) return f(std::integral_constant<int, 64>{}, std::integral_constant<int, 12>{});
        return wy_nw_dispatch<64>(nw, f);
    case 48:   // 2 CTAs x 5-6 warps (n <= ~280), or one 12-warp CTA
        if (nw == 5) return f(std::integral_constant<int, 48>{}, std::integral_constant<int, 5>{});
        if (nw == 12) return f(std::integral_constant<int, 48>{}, std::integral_constant<int, 12>{});
        if (nw == 16) return f(std::integral_constant<int, 48>{}, std::integral_constant<int, 16>{});
        return f(std::integral_constant<int, 48>{}, std::integral_constant<int, 6>{});
    case 40:
        if (nw == 5) return f(std::integral_constant<int, 40>{}, std::integral_constant<int, 5>{});
        return f(std::integral_constant<int, 40>{}, std::integral_constant<int, 6>{});
    case 32: return wy_nw_dispatch<32>(nw, f);
    case 24:
        if (nw == 12) return f(std::integral_constant<int, 24>{}, std::integral_constant<int, 12>{});
        if (nw == 16) return f(std::integral_constant<int, 24>{}, std::integral_constant<int, 16>{});
        return wy_nw_dispatch<24>(nw, f);
    case 8: return wy_nw_dispatch<8>(nw, f);
    default: return wy_nw_dispatch<16>(nw, f);
    }
}

template <class F>
static auto wy_dispatch_merge(int n, F&& f) {
    const int nw = wy_nw(n);
    // n > ~568 (no 32-row tile fits): 24-row 12-warp CTAs like the wide leaf (2M x 1025
    // 667.5 -> 660.6 ms; at n = 513 the 32-row 8-warp merges stay: 135.5 vs 137.6 ms)
    if (wide_single(n) && wy_smem_bytes(32, n) > 220 * 1024)
        return f(std::integral_constant<int, 24>{}, std::integral_constant<int, 12>{});
    if (wy_smem_bytes(96, n) <= 220 * 1024) return wy_nw_dispatch<96>(nw, f);
    if (wy_smem_bytes(64, n) <= 220 * 1024) return wy_nw_dispatch<64>(nw, f);
    if (wy_smem_bytes(32, n) <= 220 * 1024) return wy_nw_dispatch<32>(nw, f);
    return wy_nw_dispatch<16>(nw, f);
}

// Two-phase pipelined WY leaf (k_tsqr_leaf_wy2) for n > 160 when its two tile
// buffers fit: (rows, warps of phase A, warps of phase B).  0 rows: not used.
struct Wy2Cfg { int rows, nwa, nwb; };
static Wy2Cfg wy2_cfg(const elmrnn* h, int n) {
    // n <= 320: the single-chain leaf with 3 CTAs/SM measured faster (C4 shape 67.7
    // vs 77.4 ms with 4+2-warp two-phase CTAs); n = 401: 46.6 vs 56.6 ms, n = 513:
    // 135.5 vs 155.1, n = 1025: 789 vs 803 (tools/wy_variants.sh)
    if (h->tune.wy_2phase == 0 || n <= 160 || h->tune.wy_rows) return {0, 0, 0};
    if (n <= 320) return h->tune.wy_2phase == 2 ? Wy2Cfg{32, 4, 2} : Wy2Cfg{0, 0, 0};
    if (wide_single(n) && h->tune.wy_2phase != 3) return {0, 0, 0};   // 3: force two-phase (testing)
    if (wy2_smem_bytes(32, n) <= 220 * 1024) return {32, 8, 4};
    if (wy2_smem_bytes(16, n) <= 220 * 1024) return {16, 8, 4};
    return {0, 0, 0};
}
template <class F>
static auto wy2_dispatch(const Wy2Cfg& c, F&& f) {
    if (c.rows == 32 && c.nwa == 4) return f(std::integral_constant<int, 32>{}, std::integral_constant<int, 4>{},
                                             std::integral_constant<int, 2>{});
    if (c.rows == 32) return f(std::integral_constant<int, 32>{}, std::integral_constant<int, 8>{},
                               std::integral_constant<int, 4>{});
    return f(std::integral_constant<int, 16>{}, std::integral_constant<int, 8>{}, std::integral_constant<int, 4>{});
}

int64_t tsqr_leaf_slabs(const elmrnn* h, int64_t N) {
    const int n = h->M + h->nrhs;
    const Var v = pick_var(n);
    const int threads = var_threads(v, n);
    const Wy2Cfg c2 = use_wy_h(h) ? wy2_cfg(h, n) : Wy2Cfg{0, 0, 0};
    int per_sm = c2.rows ? wy2_dispatch(c2, [&](auto rows, auto na, auto nb) {
        constexpr int RW = decltype(rows)::value, NA = decltype(na)::value, NB = decltype(nb)::value;
        const size_t sm = wy2_smem_bytes(RW, n);
        cudaFuncSetAttribute(k_tsqr_leaf_wy2<RW, NA, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        int ps = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, k_tsqr_leaf_wy2<RW, NA, NB>, 32 * (NA + NB), sm);
        return ps < 1 ? 1 : ps;
    }) : use_wy_h(h) ? wy_dispatch(h, n, [&](auto rows, auto nwc) {
        constexpr int RW = decltype(rows)::value, NW = decltype(nwc)::value;
        const size_t sm = wy_leaf_smem(RW, n);
        cudaFuncSetAttribute(k_tsqr_leaf_wy<RW, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        int ps = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, k_tsqr_leaf_wy<RW, NW>, 32 * NW, sm);
        return ps < 1 ? 1 : ps;
    }) : dispatch(v, [&](auto tr, auto p) {
        int ps = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, k_tsqr_leaf<decltype(tr)::value, decltype(p)::value, 0, 1>,
                                                      threads, 0);
        return ps < 1 ? 1 : ps;
    });
    int64_t maxc = (int64_t)per_sm * h->sm_count;
    if (h->tune.max_slabs >= 1 && h->tune.max_slabs < maxc) maxc = h->tune.max_slabs;
    // at least n rows per leaf: a leaf R with fewer rows is rank deficient
    // and its noise rows only cost merges (and risk underflow cascades)
    int64_t byrows = N / n;
    // per-column path: at least ~128 rows per leaf, so a small N does not buy a deep
    // merge tree of short leaves (C1, 1000 x 21: 47 -> 8 slabs, 133 -> 123 us; C2 unchanged)
    if (!use_wy_h(h) && h->tune.max_slabs < 1) byrows = std::min(byrows, (N + 127) / 128);
    int64_t g = byrows < maxc ? byrows : maxc;
    return g < 1 ? 1 : g;
}

cudaError_t ensure_solve_ws(elmrnn* h, int64_t slabs) {
    cudaError_t e;
    const int n = h->M + h->nrhs;
    if (slabs + 1 > h->Rws_slabs || n != h->Rws_n) {   // +1: Rorig copy for the final solve
        if (h->Rws) cudaFree(h->Rws);
        h->Rws = nullptr;
        h->Rws_slabs = 0;
        if ((e = cudaMalloc(&h->Rws, (size_t)(slabs + 1) * n * n * sizeof(double)))) return e;
        h->Rws_slabs = slabs + 1;
        h->Rws_n = n;
    }
    if ((slabs + 1) / 2 > h->prog_pairs) {   // progress counters of the pipelined merge
        if (h->prog) cudaFree(h->prog);
        h->prog = nullptr;
        h->prog_pairs = 0;
        const int64_t pairs = (slabs + 1) / 2;
        if ((e = cudaMalloc(&h->prog, sizeof(int) * pairs * kMaxChunks))) return e;
        h->prog_pairs = pairs;
    }
    if (!h->sdev) {   // SolveDev + 1024 ints of per-SM counters (k_tsqr_leaf_wy)
        if ((e = cudaMalloc(&h->sdev, sizeof(SolveDev) + 1024 * sizeof(int)))) return e;
        if ((e = cudaMemsetAsync(h->sdev, 0, sizeof(SolveDev), h->stream))) return e;
        if ((e = cudaMalloc(&h->flag, sizeof(int)))) return e;
        if ((e = cudaMallocHost(&h->shost, sizeof(SolveDev)))) return e;
    }
    return cudaSuccess;
}

// One tree level of the WY merge: P CTAs per pair (pipelined chunks, cooperative
// launch) when P >= 2, else one CTA per pair.
template <int RW, int NW>
static cudaError_t wy_merge_level(elmrnn* h, int64_t slabs, int64_t stride, int n, int64_t pairs, int P) {
    const size_t sm = wy_smem_bytes(RW, n);
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_tsqr_merge_wy<RW, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)))
        return e;
    if ((e = cudaFuncSetAttribute(k_tsqr_merge_wy_par<RW, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)))
        return e;
    if (P >= 2) {
        if ((e = cudaMemsetAsync(h->prog, 0, sizeof(int) * pairs * kMaxChunks, h->stream))) return e;
        double* rws = h->Rws;
        int64_t sl = slabs, sd = stride;
        int nn = n;
        int* pg = h->prog;
        void* args[] = {&rws, &sl, &sd, &nn, &P, &pg};
        e = cudaLaunchCooperativeKernel((const void*)k_tsqr_merge_wy_par<RW, NW>, dim3((unsigned)(pairs * P)),
                                        dim3(32 * NW), args, sm, h->stream);
    } else {
        k_tsqr_merge_wy<RW, NW><<<(unsigned)pairs, 32 * NW, sm, h->stream>>>(h->Rws, slabs, stride, n);
        e = cudaGetLastError();
    }
    h->launches++;
    return e;
}

template <int RW, int NW>
static int64_t wy_merge_resident(const elmrnn* h, int n) {
    const size_t sm = wy_smem_bytes(RW, n);
    cudaFuncSetAttribute(k_tsqr_merge_wy_par<RW, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tsqr_merge_wy_par<RW, NW>, 32 * NW, sm);
    return (int64_t)occ * h->sm_count;
}

static cudaError_t tree(elmrnn* h, int64_t slabs) {
    const int n = h->M + h->nrhs;
    const Var v = pick_var(n);
    const int threads = var_threads(v, n);
    const int64_t max_stride = slabs;
    if (use_wy_h(h)) {
        // merges are latency-bound (few pairs at the top of the tree): the
        // tallest tile that fits means the fewest panel steps per fold, and the
        // SMs a level leaves idle pipeline each pair's row chunks
        // (k_tsqr_merge_wy_par).  Levels with so few pairs that every pair can
        // pipeline ALL its short chunks (32 rows; 16 when n > 320) on its own CTAs
        // take those instead: a chunk trails its predecessor by two panel steps,
        // so a chunk's fold is shorter (measured at n = 257: 0.46-0.47 -> 0.41 ms
        // per top level; the lag between chunks compounds, DESIGN 6.4b)
        const bool small32 = wy_smem_bytes(32, n) <= 220 * 1024;
        const int rws = small32 ? 32 : 16, nchs = (n + rws - 1) / rws;
        const int64_t res_s = small32 ? wy_merge_resident<32, 4>(h, n) : wy_merge_resident<16, 8>(h, n);
        return wy_dispatch_merge(n, [&](auto rows, auto nwc) {
            constexpr int RW = decltype(rows)::value, NW = decltype(nwc)::value;
            const int64_t resident = wy_merge_resident<RW, NW>(h, n);
            const int nch = (n + RW - 1) / RW;
            for (int64_t stride = 1; stride < slabs && stride < max_stride; stride *= 2) {
                const int64_t pairs = (slabs + 2 * stride - 1) / (2 * stride);
                cudaError_t e;
                if (h->tune.merge_small != 0 && RW > rws && nchs <= kMaxChunks && pairs <= h->prog_pairs &&
                    pairs * nchs <= res_s) {
                    e = small32 ? wy_merge_level<32, 4>(h, slabs, stride, n, pairs, nchs)
                                : wy_merge_level<16, 8>(h, slabs, stride, n, pairs, nchs);
                } else {
                    int P = (int)std::min<int64_t>(nch, resident / std::max<int64_t>(pairs, 1));
                    if (!(P >= 2 && nch <= kMaxChunks && pairs <= h->prog_pairs)) P = 1;
                    e = wy_merge_level<RW, NW>(h, slabs, stride, n, pairs, P);
                }
                if (e) return e;
            }
            return cudaSuccess;
        });
    }
    // 48 < n <= 72 (C2: n = 65): one 72-row chunk per merge (36 rows per thread) instead
    // of 48 + 17 rows, i.e. n column steps per tree level instead of n + (n - 48)
    if (n > 48 && n <= 72 && h->tune.merge_small != 0) {
        for (int64_t stride = 1; stride < slabs && stride < max_stride; stride *= 2) {
            int64_t pairs = (slabs + 2 * stride - 1) / (2 * stride);
            k_tsqr_merge<36, 2><<<(unsigned)pairs, threads, 0, h->stream>>>(h->Rws, slabs, stride, n);
            h->launches++;
        }
        return cudaGetLastError();
    }
    return dispatch(v, [&](auto tr, auto p) {
        for (int64_t stride = 1; stride < slabs && stride < max_stride; stride *= 2) {
            int64_t pairs = (slabs + 2 * stride - 1) / (2 * stride);
            k_tsqr_merge<decltype(tr)::value, decltype(p)::value>
                <<<(unsigned)pairs, threads, 0, h->stream>>>(h->Rws, slabs, stride, n);
            h->launches++;
        }
        return cudaGetLastError();
    });
}

cudaError_t tsqr_factor(elmrnn* h, const float* H, int64_t ldh, const float* Y, int64_t ldy, int64_t N) {
    const int n = h->M + h->nrhs;
    const Var v = pick_var(n);
    const int64_t slabs = tsqr_leaf_slabs(h, N);
    cudaError_t e;
    if ((e = ensure_solve_ws(h, wide_solve(h) && slabs < 2 ? 2 : slabs))) return e;   // wide solve: slab 1 = ridge rows
    if ((e = cudaMemsetAsync(h->flag, 0, sizeof(int), h->stream))) return e;
    const Wy2Cfg c2 = use_wy_h(h) ? wy2_cfg(h, n) : Wy2Cfg{0, 0, 0};
    const int rows_tile = c2.rows ? c2.rows : use_wy_h(h) ? wy_rows(h, n) : var_rows(v);
    int64_t rows = (N + slabs - 1) / slabs;
    rows = (rows + rows_tile - 1) / rows_tile * rows_tile;
    const int threads = var_threads(v, n);
    if (c2.rows) {
        e = wy2_dispatch(c2, [&](auto rws, auto na, auto nb) {
            constexpr int RW = decltype(rws)::value, NA = decltype(na)::value, NB = decltype(nb)::value;
            const size_t sm = wy2_smem_bytes(RW, n);
            cudaFuncSetAttribute(k_tsqr_leaf_wy2<RW, NA, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            k_tsqr_leaf_wy2<RW, NA, NB><<<(unsigned)slabs, 32 * (NA + NB), sm, h->stream>>>(
                H, ldh, Y, ldy, h->nrhs, N, h->M, h->Rws, rows, h->flag, wy_la_wait(n));
            h->launches++;
            return cudaGetLastError();
        });
        if (e) return e;
        return tree(h, slabs);
    }
    if (use_wy_h(h)) {
        e = wy_dispatch(h, n, [&](auto rws, auto nwc) {
            constexpr int RW = decltype(rws)::value, NW = decltype(nwc)::value;
            const size_t sm = wy_leaf_smem(RW, n);
            cudaFuncSetAttribute(k_tsqr_leaf_wy<RW, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            int* slot = reinterpret_cast<int*>(h->sdev + 1);   // per-SM arrival counters (ensure_solve_ws)
            cudaMemsetAsync(slot, 0, 1024 * sizeof(int), h->stream);
#ifdef ELM_QR_TRACE   // tracing build: per panel step clocks of CTA 0's last tile -> $ELMRNN_TRACE_QR
            const char* tpath = std::getenv("ELMRNN_TRACE_QR");
            unsigned long long* tb = nullptr;
            if (tpath) {
                cudaMalloc(&tb, 4096 * 8 * sizeof(unsigned long long));
                cudaMemset(tb, 0, 4096 * 8 * sizeof(unsigned long long));
                cudaMemcpyToSymbol(g_qr_trace, &tb, sizeof(tb));
            }
#endif
            k_tsqr_leaf_wy<RW, NW><<<(unsigned)slabs, 32 * NW, sm, h->stream>>>(
                H, ldh, Y, ldy, h->nrhs, N, h->M, h->Rws, rows, h->flag, slot, wy_la_wait(n),
                h->tune.pw_mode >= 0 ? h->tune.pw_mode : (RW == 48 ? 0 : 1));
            h->launches++;
#ifdef ELM_QR_TRACE
            if (tb) {
                std::vector<unsigned long long> hb(4096 * 8);
                cudaStreamSynchronize(h->stream);
                cudaMemcpy(hb.data(), tb, hb.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
                unsigned long long* z = nullptr;
                cudaMemcpyToSymbol(g_qr_trace, &z, sizeof(z));
                cudaFree(tb);
                if (FILE* f = std::fopen(tpath, "w")) {
                    for (int k = 0; k < 4096; ++k) {
                        bool any = false;
                        for (int c = 0; c < 8; ++c) any |= hb[k * 8 + c] != 0;
                        if (!any) continue;
                        std::fprintf(f, "%d", k);
                        for (int c = 0; c < 8; ++c) std::fprintf(f, ",%llu", hb[k * 8 + c]);
                        std::fprintf(f, "\n");
                    }
                    std::fclose(f);
                }
            }
#endif
            return cudaGetLastError();
        });
        if (e) return e;
        return tree(h, slabs);
    }
    e = dispatch(v, [&](auto tr, auto p) {
        LeafSrc<0, 1> src{H, ldh, {}};
        k_tsqr_leaf<decltype(tr)::value, decltype(p)::value, 0, 1>
            <<<(unsigned)slabs, threads, 0, h->stream>>>(src, Y, ldy, N, h->M, h->Rws, rows, h->flag);
        h->launches++;
        return cudaGetLastError();
    });
    if (e) return e;
    return tree(h, slabs);
}

// Fused build -> leaf (elmrnn_train): the per-column leaf
// computes each H element of the cell-independent archs where it would load it.
bool tsqr_fused_supported(const elmrnn* h) {
    const int n = h->M + 1;
    if (use_wy(h, n)) return false;   // the per-column fold's thread = column layout only
    if (h->arch == kArchElman) return h->Q <= 32;
    return h->arch == kArchJordan || h->arch == kArchNarmax;
}

cudaError_t tsqr_factor_fused(elmrnn* h, const float* X, int64_t ldx, const float* Yfb, int64_t ldyfb,
                              const float* Y, int64_t N) {
    const int n = h->M + 1;
    const Var v = pick_var(n);
    const int64_t slabs = tsqr_leaf_slabs(h, N);
    cudaError_t e;
    if ((e = ensure_solve_ws(h, slabs))) return e;
    if ((e = cudaMemsetAsync(h->flag, 0, sizeof(int), h->stream))) return e;
    int64_t rows = (N + slabs - 1) / slabs;
    rows = (rows + var_rows(v) - 1) / var_rows(v) * var_rows(v);
    const int threads = var_threads(v, n);
    int nlag = h->Q - 1;
    if (h->arch == kArchNarmax) nlag = h->F < h->Q - 1 ? h->F : h->Q - 1;
    const CellSrc cs{X, ldx, Yfb, ldyfb, h->S, h->M, h->Q, h->act, nlag, h->W, h->b, h->rec};
    e = dispatch(v, [&](auto tr, auto p) {
        constexpr int TRv = decltype(tr)::value, Pv = decltype(p)::value;
        if (h->arch == kArchElman) {
            if (h->Q <= 16) {
                LeafSrc<1, 16> src{nullptr, 0, cs};
                k_tsqr_leaf<TRv, Pv, 1, 16><<<(unsigned)slabs, threads, 0, h->stream>>>(src, Y, 1, N, h->M, h->Rws, rows, h->flag);
            } else {
                LeafSrc<1, 32> src{nullptr, 0, cs};
                k_tsqr_leaf<TRv, Pv, 1, 32><<<(unsigned)slabs, threads, 0, h->stream>>>(src, Y, 1, N, h->M, h->Rws, rows, h->flag);
            }
        } else {
            LeafSrc<2, 1> src{nullptr, 0, cs};
            k_tsqr_leaf<TRv, Pv, 2, 1><<<(unsigned)slabs, threads, 0, h->stream>>>(src, Y, 1, N, h->M, h->Rws, rows, h->flag);
        }
        h->launches++;
        return cudaGetLastError();
    });
    if (e) return e;
    return tree(h, slabs);
}

cudaError_t tsqr_pack(elmrnn* h, double* Rpk) {
    const int n = h->M + h->nrhs;
    int64_t len = (int64_t)n * (n + 1) / 2;
    int blocks = (int)((len + 255) / 256);
    if (blocks > 1024) blocks = 1024;
    k_pack<<<blocks, 256, 0, h->stream>>>(h->Rws, n, Rpk, h->flag, h->sdev);
    h->launches++;
    return cudaGetLastError();
}

cudaError_t tsqr_merge_packed(elmrnn* h, const double* Rpk_all, int P) {
    const int n = h->M + h->nrhs;
    cudaError_t e;
    if ((e = ensure_solve_ws(h, wide_solve(h) && P < 2 ? 2 : P))) return e;
    if ((e = cudaMemsetAsync(h->flag, 0, sizeof(int), h->stream))) return e;
    int64_t total = (int64_t)P * n * n;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 4096) blocks = 4096;
    k_unpack<<<blocks, 256, 0, h->stream>>>(Rpk_all, P, n, h->Rws);
    h->launches++;
    if ((e = cudaGetLastError())) return e;
    return tree(h, P);
}

cudaError_t tsqr_solve(elmrnn* h, int64_t n_total, double* beta) {
    const int n = h->M + h->nrhs;
    const Var v = pick_var(n);
    const int threads = var_threads(v, n);
    double* Rorig = h->Rws + (size_t)(h->Rws_slabs - 1) * n * n;
    if (wide_solve(h)) {
        const size_t zsm = ((n + 1) & ~1) * sizeof(double);
        k_solve_wide_prep<<<1, 1024, zsm, h->stream>>>(h->Rws, h->Rws + (size_t)n * n, Rorig, h->M, n, h->sdev);
        h->launches++;
        cudaError_t e = wy_dispatch_merge(n, [&](auto rows, auto nwc) {
            constexpr int RW = decltype(rows)::value, NW = decltype(nwc)::value;
            const size_t sm = wy_smem_bytes(RW, n);
            cudaFuncSetAttribute(k_tsqr_merge_wy<RW, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            // the ridge rows are folded only when k_solve_wide_prep found R rank deficient
            k_tsqr_merge_wy<RW, NW><<<1, wy_threads(n), sm, h->stream>>>(h->Rws, 2, 1, n, &h->sdev->rank_flag);
            h->launches++;
            return cudaGetLastError();
        });
        if (e) return e;
        k_solve_wide_finish<<<1, 1024, zsm, h->stream>>>(h->Rws, Rorig, h->M, n, (long long)n_total, h->flag, beta,
                                                          h->sdev, h->nrhs > 1 ? h->rho_multi : nullptr);
        h->launches++;
        return cudaGetLastError();
    }
    size_t smem = 3 * ((n + 1) & ~1) * sizeof(double);   // z, R_kk, beta
    const int r_smem = smem + (size_t)n * n * sizeof(double) <= 160 * 1024 ? 1 : 0;   // R resident (n <= ~140)
    if (r_smem) smem += (size_t)n * n * sizeof(double);
    return dispatch(v, [&](auto tr, auto p) {
        auto kern = k_tsqr_solve<decltype(tr)::value, decltype(p)::value>;
        if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<1, threads, smem, h->stream>>>(h->Rws, Rorig, h->M, (long long)n_total, h->flag, beta, h->sdev, r_smem);
        h->launches++;
        return cudaGetLastError();
    });
}

}  // namespace elm
