// hbuild_dense_fma.cu -- FP32-FMA H builder for the dense-recurrence
// architectures: fully connected (S2.2.4, prose reading R9), LSTM
// (S2.2.5) and GRU (S2.2.6) with dense U (R10, R11).
//
// Unlike Elman, these are NOT cell independent: step t needs the whole
// h(t-1) of the sample, so the unit of parallel work is a tile of T samples
// whose state stays resident in shared memory across all Q steps (the paper's
// "H_loc" idea of Alg. 3, carried to the whole state), and each step is
// a small GEMM  a(t) = h(t-1) [T x K] . U [K x G*M] + x(t) W + b  with the gate
// epilogue fused.  Thread layout: warp w = row group (RT rows), lane = neuron
// within a 32-neuron chunk, all G gates of that neuron in registers, so the
// gate nonlinearities and the c/h update are thread local.  U K-slices are
// staged through shared memory once per CTA; h rows are warp-broadcast reads.
// This is the small-M path and the reference path for every shape; the
// tcgen05 builder (hbuild_dense_tc.cu) takes over at large M.
#include <algorithm>

#include "common.cuh"

namespace elm {

struct DenseParams {
    const float* X;
    int64_t ldx, N;
    int S, M, Q, G, act, L;
    const float* W;   // [S][G*M]
    const float* b;   // [G*M]
    const float* U;   // LSTM/GRU U_cat [M][G*M]; FC A [L*M][M]
    float* H;
    int64_t ldh;
    float* ring_global;  // FC history ring in global memory (nullptr: shared)
    const double* rbeta; // fused readout (Eq. 4): no H store, ryp[i] = H_i . beta
    double* ryp;
    int T;               // rows per tile (= 8 * RT)
    int64_t ntiles;
};

constexpr int kNJ = 32;   // neurons per chunk (one per lane)
constexpr int kKC = 16;   // K rows per staged U slice

template <int RT>
__device__ __forceinline__ void load_rows(const float* src, float (&v)[RT]) {
    if constexpr (RT % 4 == 0) {
#pragma unroll
        for (int q = 0; q < RT / 4; ++q) {
            float4 f = *reinterpret_cast<const float4*>(src + 4 * q);
            v[4 * q] = f.x; v[4 * q + 1] = f.y; v[4 * q + 2] = f.z; v[4 * q + 3] = f.w;
        }
    } else {
#pragma unroll
        for (int q = 0; q < RT; ++q) v[q] = src[q];
    }
}

// acc[rr][g] += sum_k A[k][row0+rr] * B[k][g*ldgate + j]  over k in [0, K)
// A row k is at a_of(k) (a [T]-vector); B row k at b_of(k).
// A_STAGE: the A rows live in global memory (FC history ring in L2) and are
// staged through shared memory slice by slice together with B.
template <int RT, int GG, bool A_STAGE = false, class AOf, class BOf>
__device__ __forceinline__ void tile_contract(float (&acc)[RT][GG], int K, int c0, int M, AOf a_of, BOf b_of,
                                              float* us, int rbase, float* as = nullptr) {
    const int tid = threadIdx.x, lane = tid & 31;
    constexpr int T = 8 * RT;
    for (int k0 = 0; k0 < K; k0 += kKC) {
        for (int e = tid; e < kKC * GG * kNJ; e += blockDim.x) {
            int kk = e / (GG * kNJ), rem = e - kk * (GG * kNJ), g = rem / kNJ, jj = rem - g * kNJ;
            int k = k0 + kk, j = c0 + jj;
            us[e] = (k < K && j < M) ? __ldg(b_of(k) + g * M + j) : 0.0f;
        }
        if constexpr (A_STAGE) {
            for (int e = tid; e < kKC * T; e += blockDim.x) {
                int kk = e / T, rr = e - kk * T;
                as[e] = (k0 + kk < K) ? a_of(k0 + kk)[rr] : 0.0f;
            }
        }
        __syncthreads();
        int kmax = min(kKC, K - k0);
        for (int kk = 0; kk < kmax; ++kk) {
            float hv[RT];
            if constexpr (A_STAGE)
                load_rows<RT>(as + kk * T + rbase, hv);
            else
                load_rows<RT>(a_of(k0 + kk) + rbase, hv);
            float u[GG];
#pragma unroll
            for (int g = 0; g < GG; ++g) u[g] = us[(kk * GG + g) * kNJ + lane];
#pragma unroll
            for (int rr = 0; rr < RT; ++rr)
#pragma unroll
                for (int g = 0; g < GG; ++g) acc[rr][g] = fmaf(hv[rr], u[g], acc[rr][g]);
        }
        __syncthreads();
    }
}

template <int ARCH, int RT>
__global__ void __launch_bounds__(256) k_dense_fma(DenseParams p) {
    extern __shared__ float4 smem4[];
    float* sm = reinterpret_cast<float*>(smem4);
    constexpr int GG = (ARCH == kArchLSTM) ? 4 : (ARCH == kArchGRU ? 2 : 1);
    const int T = 8 * RT, M = p.M, S = p.S, GM = p.G * p.M;
    const int nslots = (ARCH == kArchFC) ? p.L + 1 : 2;
    const int tid = threadIdx.x, lane = tid & 31, rg = tid >> 5, rbase = rg * RT;
    const size_t MT = (size_t)M * T;

    float* xs = sm;                                           // [T][S]
    float* us = xs + ((T * S + 3) & ~3);                      // [KC][GG][NJ]
    float* as = us + kKC * 4 * kNJ;                           // [KC][T] staged A (FC, global ring)
    float* cur = as + kKC * T;
    float* ring;
    if (p.ring_global) {
        ring = p.ring_global + (size_t)blockIdx.x * nslots * MT;
    } else {
        ring = cur;
        cur += nslots * MT;
    }
    float* cs = cur;        // LSTM c(t) / GRU z, [M][T]
    float* rhs = cur + MT;  // GRU r o h(t-1), [M][T]

    for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
        const int64_t row0 = tile * T;
        if (ARCH != kArchFC)
            for (size_t e = tid; e < MT; e += blockDim.x) ring[e] = 0.0f;   // h(0) = 0 (R13)
        if (ARCH == kArchLSTM)
            for (size_t e = tid; e < MT; e += blockDim.x) cs[e] = 0.0f;     // c(0) = 0
        for (int t = 1; t <= p.Q; ++t) {
            for (int e = tid; e < T * S; e += blockDim.x) {
                int r = e / S, s = e - r * S;
                int64_t i = row0 + r;
                xs[e] = (i < p.N) ? __ldg(p.X + i * p.ldx + (int64_t)(t - 1) * S + s) : 0.0f;
            }
            __syncthreads();
            const float* hprev = ring + (size_t)((t - 1) % nslots) * MT;
            float* hcur = ring + (size_t)(t % nslots) * MT;
            for (int c0 = 0; c0 < M; c0 += kNJ) {
                const int j = c0 + lane;
                const bool jv = j < M;
                float acc[RT][GG];
#pragma unroll
                for (int g = 0; g < GG; ++g) {
                    float bg = jv ? __ldg(p.b + g * M + j) : 0.0f;
#pragma unroll
                    for (int rr = 0; rr < RT; ++rr) acc[rr][g] = bg;
                }
                for (int s = 0; s < S; ++s) {
#pragma unroll
                    for (int g = 0; g < GG; ++g) {
                        float wv = jv ? __ldg(p.W + (int64_t)s * GM + g * M + j) : 0.0f;
#pragma unroll
                        for (int rr = 0; rr < RT; ++rr) acc[rr][g] = fmaf(xs[(rbase + rr) * S + s], wv, acc[rr][g]);
                    }
                }
                if (ARCH == kArchFC) {
                    const int nl = min(t - 1, p.L);
                    auto aof = [&](int k) { int lag = k / M + 1, m = k - (lag - 1) * M;
                                            return ring + (size_t)((t - lag) % nslots) * MT + (size_t)m * T; };
                    auto bof = [&](int k) { return p.U + (size_t)k * M; };
                    if (p.ring_global)
                        tile_contract<RT, GG, true>(acc, nl * M, c0, M, aof, bof, us, rbase, as);
                    else
                        tile_contract<RT, GG>(acc, nl * M, c0, M, aof, bof, us, rbase);
                } else {
                    tile_contract<RT, GG>(
                        acc, M, c0, M, [&](int k) { return hprev + (size_t)k * T; },
                        [&](int k) { return p.U + (size_t)k * GM; }, us, rbase);
                }
                if (jv) {
#pragma unroll
                    for (int rr = 0; rr < RT; ++rr) {
                        const size_t o = (size_t)j * T + rbase + rr;
                        if (ARCH == kArchFC) {
                            hcur[o] = act_g(acc[rr][0], p.act);
                        } else if (ARCH == kArchLSTM) {
                            // gates (o, c, lambda, in) = 0..3
                            float c = sigmoidf_(acc[rr][2]) * cs[o] + sigmoidf_(acc[rr][3]) * tanhf_(acc[rr][1]);
                            cs[o] = c;
                            hcur[o] = sigmoidf_(acc[rr][0]) * tanhf_(c);
                        } else {
                            // GRU phase 1: z, r = 0, 1
                            cs[o] = sigmoidf_(acc[rr][0]);
                            rhs[o] = sigmoidf_(acc[rr][1]) * hprev[o];
                        }
                    }
                }
            }
            __syncthreads();
            if (ARCH == kArchGRU) {
                // phase 2: n = tanh(x W_f + (r o h) U_f + b_f); h = (1 - z) h + z n
                for (int c0 = 0; c0 < M; c0 += kNJ) {
                    const int j = c0 + lane;
                    const bool jv = j < M;
                    float acc[RT][1];
                    float bg = jv ? __ldg(p.b + 2 * M + j) : 0.0f;
#pragma unroll
                    for (int rr = 0; rr < RT; ++rr) acc[rr][0] = bg;
                    for (int s = 0; s < S; ++s) {
                        float wv = jv ? __ldg(p.W + (int64_t)s * GM + 2 * M + j) : 0.0f;
#pragma unroll
                        for (int rr = 0; rr < RT; ++rr) acc[rr][0] = fmaf(xs[(rbase + rr) * S + s], wv, acc[rr][0]);
                    }
                    tile_contract<RT, 1>(
                        acc, M, c0, M, [&](int k) { return rhs + (size_t)k * T; },
                        [&](int k) { return p.U + (size_t)k * GM + 2 * M; }, us, rbase);
                    if (jv) {
#pragma unroll
                        for (int rr = 0; rr < RT; ++rr) {
                            const size_t o = (size_t)j * T + rbase + rr;
                            float z = cs[o];
                            hcur[o] = (1.0f - z) * hprev[o] + z * tanhf_(acc[rr][0]);
                        }
                    }
                }
                __syncthreads();
            }
        }
        const float* hQ = ring + (size_t)(p.Q % nslots) * MT;
        if (p.rbeta) {   // one warp per row: lanes over neurons, fixed shuffle-tree order
            const int lane = tid & 31;
            for (int r = tid >> 5; r < T; r += (int)(blockDim.x >> 5)) {
                double v = 0.0;
                for (int j = lane; j < M; j += 32) v = fma((double)hQ[(size_t)j * T + r], __ldg(p.rbeta + j), v);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0 && row0 + r < p.N) p.ryp[row0 + r] = v;
            }
        } else {
            for (int e = tid; e < T * M; e += blockDim.x) {
                int r = e / M, j = e - r * M;
                int64_t i = row0 + r;
                if (i < p.N) p.H[i * p.ldh + j] = hQ[(size_t)j * T + r];
            }
        }
        __syncthreads();
    }
}

// Shared-memory floats the kernel needs for a given tile height.
static size_t dense_smem_floats(int arch, int T, int S, int M, int L, bool ring_in_smem) {
    size_t MT = (size_t)M * T;
    size_t f = ((size_t)T * S + 3) / 4 * 4 + (size_t)kKC * 4 * kNJ + (size_t)kKC * T;
    int nslots = arch == kArchFC ? L + 1 : 2;
    if (ring_in_smem) f += nslots * MT;
    if (arch == kArchLSTM) f += MT;
    if (arch == kArchGRU) f += 2 * MT;
    return f;
}

template <int ARCH>
static cudaError_t launch_arch(elmrnn* h, DenseParams& p, int RT, size_t smem) {
    auto pick = [&](auto kern) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e) return e;
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
        if (e) return e;
        if (per_sm < 1) return cudaErrorInvalidConfiguration;
        int64_t grid = std::min<int64_t>(p.ntiles, (int64_t)per_sm * h->sm_count);
        if (p.ring_global) {
            size_t need = (size_t)grid * (p.L + 1) * (size_t)p.M * p.T * sizeof(float);
            if (need > h->scratch_bytes) {
                if (h->scratch) cudaFree(h->scratch);
                h->scratch = nullptr;
                h->scratch_bytes = 0;
                if ((e = cudaMalloc(&h->scratch, need))) return e;
                h->scratch_bytes = need;
            }
            p.ring_global = h->scratch;
        }
        kern<<<(unsigned)grid, 256, smem, h->stream>>>(p);
        h->launches++;
        return cudaGetLastError();
    };
    switch (RT) {
    case 8: return pick(k_dense_fma<ARCH, 8>);
    case 4: return pick(k_dense_fma<ARCH, 4>);
    case 2: return pick(k_dense_fma<ARCH, 2>);
    default: return pick(k_dense_fma<ARCH, 1>);
    }
}

cudaError_t launch_dense_fma(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    const size_t kMaxSmem = 220 * 1024;
    DenseParams p{};
    p.X = X; p.ldx = ldx; p.N = N; p.S = h->S; p.M = h->M; p.Q = h->Q; p.G = h->G; p.act = h->act;
    p.L = h->fc_lags; p.W = h->W; p.b = h->b; p.U = h->rec; p.H = H; p.ldh = ldh;
    p.rbeta = h->ro_beta; p.ryp = h->ro_yp;
    h->ro_slots = 1;
    int RT = 8;
    bool ring_smem = true;
    for (;;) {
        size_t f = dense_smem_floats(h->arch, 8 * RT, h->S, h->M, h->fc_lags, ring_smem);
        if (f * sizeof(float) <= kMaxSmem) break;
        if (RT > 1) { RT /= 2; continue; }
        if (ring_smem && h->arch == kArchFC) { ring_smem = false; RT = 8; continue; }
        return cudaErrorInvalidConfiguration;  // state does not fit: caller reports UNSUPPORTED
    }
    // FC with a ring in global memory: prefer the tallest tile that keeps reuse high.
    p.T = 8 * RT;
    p.ntiles = (N + p.T - 1) / p.T;
    p.ring_global = ring_smem ? nullptr : reinterpret_cast<float*>(1);  // allocated in launch_arch
    size_t smem = dense_smem_floats(h->arch, p.T, h->S, h->M, h->fc_lags, ring_smem) * sizeof(float);
    switch (h->arch) {
    case kArchFC: return launch_arch<kArchFC>(h, p, RT, smem);
    case kArchLSTM: return launch_arch<kArchLSTM>(h, p, RT, smem);
    case kArchGRU: return launch_arch<kArchGRU>(h, p, RT, smem);
    }
    return cudaErrorInvalidValue;
}

}  // namespace elm
