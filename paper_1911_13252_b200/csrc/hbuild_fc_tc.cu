// hbuild_fc_tc.cu -- tcgen05 tensor-core H builder for the fully connected
// RNN (S2.2.4, prose reading R9), M = 128:
//   a(t) = x(t) W + b + sum_{k=1}^{min(t-1,L)} h(t-k) A_k,   h(t) = g(a(t))
// The lag sum is a K = min(t-1,L)*M contraction per step; it runs on the 5th
// generation tensor cores (3-pass fp16 hi/lo split into one fp32 TMEM
// accumulator, A_k pre-scaled by 2^sigma, as in the LSTM builder), x W + b and
// g on the CUDA cores.
//
// The history h(t-1..t-L) does not fit on chip (L x 64 KB per 128-row tile),
// so each CTA keeps a private ring of NS = min(L, Q-1) + 1 history slots in
// global memory, stored directly as the MMA's SW128 K-major fp16 hi|lo images.
// Per step the bulk-copy producer streams (history slot K-slice, A_k K-slice)
// pairs through a 3-stage shared-memory ring, OLDEST lag first: only the lag-1
// slot depends on the previous step's epilogue, so step t+1's lags >= 2 run
// on the tensor cores while the epilogue of step t is still computing h(t).
//
//   smem: 3 stages x [A = history hi|lo 32 KB, B = A_k hi|lo 32 KB]
//   TMEM: 2 x 128 accumulator columns (double buffered across steps)
//   warps 0..15 epilogue (warp w: TMEM lane quadrant w % 4, neurons
//   32 (w / 4) .. +31), 16 producer + TMEM allocator, 17 MMA issuer.
//   The epilogue writes h(t) to the ring with generic stores, then
//   fence.proxy.async.global + an mbarrier arrive hand it to the producer.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace elm {

namespace {

constexpr int kFM = 128;                         // hidden size handled by this kernel
constexpr int kFRows = 128;
constexpr int kFKS = kFM / 64;                   // K slices per lag
constexpr int kFStages = 3;
constexpr int kFTile = 128 * 64 * 2;             // one 128 x 64 fp16 SW128 tile (16 KB)
constexpr int kFPair = 2 * kFTile;               // hi + lo
constexpr int kFStageBytes = 2 * kFPair;         // history pair + A_k pair
constexpr int kFSlotBytes = kFKS * kFPair;       // one history slot: h(t) hi|lo, 64 KB
constexpr int kFEpiWarps = 16;
constexpr int kFProdWarp = kFEpiWarps, kFMmaWarp = kFEpiWarps + 1;
constexpr int kFThreads = (kFEpiWarps + 2) * 32;
constexpr int kFSmem = 1024 + kFStages * kFStageBytes + 256;
constexpr int kFWbMax = 1024;

struct FcParams {
    const float* X;
    int64_t ldx, N;
    float* H;
    int64_t ldh;
    const uint8_t* Aimg;   // [Leff][KS][hi|lo][16 KB]: B images of A_k (row j, K index m)
    uint8_t* hist;         // [grid][NS][KS][hi|lo][16 KB]: A images of h(tau)
    int S, Q, L, NS, act;
    int two_pass;          // 1: A_k on the fp16 grid (weight_grid = 1), A_lo = 0 -> hi.hi + lo.hi only
    int64_t ntiles;
    uint32_t xbytes;       // a1: bytes of a tile's X block staged by cp.async.bulk (0: x(t) via L1)
    const double* rbeta;   // fused readout (Eq. 4): no H store; ryp[u * N + row] = H[row][u's neurons] . beta
    double* ryp;
    float k_act;           // sigmoid: -log2(e) 2^-sigma; tanh: 2 log2(e) 2^-sigma
    float wb[kFWbMax];     // per neuron j: [b, W_0..W_{S-1}] x 2^sigma
};

__device__ __forceinline__ void tmem_ld16f(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int SS>
__global__ void __launch_bounds__(kFThreads, 1) k_fc_tc(const __grid_constant__ FcParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stages = smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(stages + kFStages * kFStageBytes);
    uint64_t* full = bars;                        // [kFStages]
    uint64_t* empty = bars + kFStages;            // [kFStages]
    uint64_t* acc_full = bars + 2 * kFStages;     // [2]
    uint64_t* acc_empty = acc_full + 2;           // [2]
    uint64_t* hist_ready = acc_empty + 2;         // h(t) is in the ring (t < Q)
    uint64_t* x_full = hist_ready + 1;            // the tile's X block has landed
    uint64_t* x_empty = x_full + 1;               // every epilogue warp has read its last x(t)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(x_empty + 1);
    float* xbuf = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);   // the tile's X block

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kFStages; ++i) {
            ptx::mbar_init(full + i, 1);
            ptx::mbar_init(empty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(acc_full + i, 1);
            ptx::mbar_init(acc_empty + i, kFEpiWarps);
        }
        ptx::mbar_init(hist_ready, kFEpiWarps);
        ptx::mbar_init(x_full, 1);
        ptx::mbar_init(x_empty, kFEpiWarps);
        ptx::fence_mbar_init();
    }
    if (warp == kFProdWarp) {
        ptx::tmem_alloc(tmem_slot, 256);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    uint8_t* hist = p.hist + (size_t)blockIdx.x * p.NS * kFSlotBytes;

    if (warp == kFProdWarp) {
        // ---------------- producer: per step t >= 2, lags min(t-1,L)..1
        uint32_t st = 0, ph = 0, hph = 0, xph = 0;
        for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            if (ptx::xstage_tile(p.xbytes, tile, p.N))   // the tile's X block (a1)
                ptx::xstage_issue(xbuf, p.X, p.ldx, tile, p.xbytes, x_full, x_empty, xph);
            for (int t = 2; t <= p.Q; ++t) {
                const int nl = min(t - 1, p.L);
                for (int k = nl; k >= 1; --k) {
                    const uint8_t* slot = hist + (size_t)((t - k) % p.NS) * kFSlotBytes;
                    for (int ks = 0; ks < kFKS; ++ks) {
                        if (k == 1 && ks == 0) {   // h(t-1) comes from the previous step's epilogue
                            ptx::mbar_wait(hist_ready, hph);
                            hph ^= 1;
                            fence_proxy_async_global();
                        }
                        ptx::mbar_wait(empty + st, ph ^ 1);
                        if (ptx::elect_one()) {
                            uint8_t* sb = stages + st * kFStageBytes;
                            const uint32_t bb = p.two_pass ? kFTile : kFPair;   // A_k hi only when A_lo = 0
                            ptx::mbar_arrive_expect_tx(full + st, kFPair + bb);
                            ptx::bulk_g2s(sb, slot + ks * kFPair, kFPair, full + st);
                            ptx::bulk_g2s(sb + kFPair, p.Aimg + (size_t)((k - 1) * kFKS + ks) * kFPair, bb, full + st);
                        }
                        __syncwarp();
                        if (++st == kFStages) { st = 0; ph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == kFMmaWarp) {
        // ---------------- MMA issuer: 12 SS MMAs (4 K-steps x 3 passes) per stage
        constexpr uint32_t idesc = ptx::idesc_f16(128, kFM);
        const uint64_t dbase = ptx::desc_sw128_kmajor(ptx::smem_u32(stages));
        const bool two = p.two_pass != 0;
        uint32_t st = 0, ph = 0, ach = 0, aph = 0;
        for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            for (int t = 2; t <= p.Q; ++t) {
                const int nl = min(t - 1, p.L);
                ptx::mbar_wait(acc_empty + ach, aph ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + ach * kFM;
                for (int k = nl; k >= 1; --k) {
                    for (int ks = 0; ks < kFKS; ++ks) {
                        ptx::mbar_wait(full + st, ph);
                        ptx::tc_fence_after();
                        const uint64_t ah = dbase + (uint64_t)((st * kFStageBytes) >> 4);
                        const uint64_t al = ah + (uint64_t)(kFTile >> 4);
                        const uint64_t bh = ah + (uint64_t)(kFPair >> 4);
                        const uint64_t bl = bh + (uint64_t)(kFTile >> 4);
                        const bool first = (k == nl) && (ks == 0);
                        if (ptx::elect_one()) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                ptx::mma_f16_ss(d, ah + 2 * kk, bh + 2 * kk, idesc, (first && kk == 0) ? 0u : 1u);
                                if (!two) ptx::mma_f16_ss(d, ah + 2 * kk, bl + 2 * kk, idesc, 1u);
                                ptx::mma_f16_ss(d, al + 2 * kk, bh + 2 * kk, idesc, 1u);
                            }
                            ptx::mma_commit(empty + st);
                            if (k == 1 && ks == kFKS - 1) ptx::mma_commit(acc_full + ach);
                        }
                        __syncwarp();
                        if (++st == kFStages) { st = 0; ph ^= 1; }
                    }
                }
                if (++ach == 2) { ach = 0; aph ^= 1; }
            }
        }
    } else {
        // ---------------- epilogue: h(t) = g(acc 2^-sigma + x W + b), ring write, H(Q)
        const int q = warp & 3, u = warp >> 2;
        const int r = 32 * q + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
        const float kA = p.k_act;
        const bool is_tanh = p.act == 1;
        uint32_t ach = 0, aph = 0, xph = 0;
        for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            const int64_t row = tile * kFRows + r;
            const bool valid = row < p.N;
            const bool xst = ptx::xstage_tile(p.xbytes, tile, p.N);
            const float* xrow = xst ? xbuf + (int64_t)r * p.ldx : p.X + (valid ? row : 0) * p.ldx;
            if (xst) {
                ptx::mbar_wait(x_full, xph);
                xph ^= 1;
            }
            for (int t = 1; t <= p.Q; ++t) {
                float xs[SS];
#pragma unroll
                for (int s = 0; s < SS; ++s)
                    xs[s] = (valid && s < p.S) ? (xst ? xrow[(t - 1) * p.S + s] : __ldg(xrow + (int64_t)(t - 1) * p.S + s))
                                               : 0.0f;
                if (xst && t == p.Q) {   // last x(t) of this tile read: the block may be replaced
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(x_empty);
                }
                float a[2][16];
                if (t >= 2) {
                    ptx::mbar_wait(acc_full + ach, aph);
                    ptx::tc_fence_after();
                    tmem_ld16f(lane_base + ach * kFM + 32 * u, a[0]);
                    tmem_ld16f(lane_base + ach * kFM + 32 * u + 16, a[1]);
                    ptx::tmem_wait_ld();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(acc_empty + ach);
                    if (++ach == 2) { ach = 0; aph ^= 1; }
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i) a[0][i] = a[1][i] = 0.0f;
                }
                float hv[32];
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
#pragma unroll
                    for (int e2 = 0; e2 < 2; ++e2) {
                        const int j = 32 * u + i + e2;
                        const float* w = p.wb + j * (SS + 1);
                        float v = a[(i + e2) >> 4][(i + e2) & 15] + w[0];
#pragma unroll
                        for (int s = 0; s < SS; ++s) v = fmaf(xs[s], w[1 + s], v);
                        // accurate activation forms (common.cuh; DESIGN R26)
                        hv[i + e2] = is_tanh ? tanh_e2(kA * v) : sig_e2(kA * v);
                    }
                }
                if (t < p.Q) {
                    // h(t) -> ring slot t % NS as fp16 hi|lo, SW128 K-major (row r, K = neuron)
                    uint8_t* slot = hist + (size_t)(t % p.NS) * kFSlotBytes + (u >> 1) * kFPair;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint4 hi, lo;
                        uint32_t* hp = &hi.x;
                        uint32_t* lp = &lo.x;
#pragma unroll
                        for (int w2 = 0; w2 < 4; ++w2) {
                            const float x0 = hv[8 * c + 2 * w2], x1 = hv[8 * c + 2 * w2 + 1];
                            const __half2 h2 = __floats2half2_rn(x0, x1);
                            const float2 hf = __half22float2(h2);
                            const __half2 l2 = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
                            hp[w2] = *reinterpret_cast<const uint32_t*>(&h2);
                            lp[w2] = *reinterpret_cast<const uint32_t*>(&l2);
                        }
                        const uint32_t off = ptx::sw128_offset((uint32_t)r, (uint32_t)(32 * (u & 1) + 8 * c));
                        *reinterpret_cast<uint4*>(slot + off) = hi;
                        *reinterpret_cast<uint4*>(slot + kFTile + off) = lo;
                    }
                    fence_proxy_async_global();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(hist_ready);
                } else if (valid && p.rbeta) {   // fused readout: this thread's 32 neurons
                    double yacc = 0.0;
#pragma unroll
                    for (int i = 0; i < 32; ++i) yacc = fma((double)hv[i], __ldg(p.rbeta + 32 * u + i), yacc);
                    p.ryp[u * p.N + row] = yacc;
                } else if (valid) {
                    float* dst = p.H + row * p.ldh + 32 * u;
                    if (((p.ldh | (int64_t)(reinterpret_cast<uintptr_t>(p.H) >> 2)) & 3) == 0) {
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            reinterpret_cast<float4*>(dst)[c] =
                                make_float4(hv[4 * c], hv[4 * c + 1], hv[4 * c + 2], hv[4 * c + 3]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i) dst[i] = hv[i];
                    }
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kFProdWarp) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 256);
    }
}

// B images of A_k (scaled by 2^sigma): image[(k*KS + s)*2 + part][sw128(j, kk)] = A_k[64 s + kk][j]
__global__ void k_pack_fc(const float* __restrict__ A, int M, int Leff, float scale, uint8_t* __restrict__ img) {
    const int KS = M / 64;
    const int64_t total = (int64_t)Leff * KS * 128 * 64;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int kk = (int)(e % 64);
        const int j = (int)((e / 64) % 128);
        const int s = (int)((e / (64 * 128)) % KS);
        const int k = (int)(e / ((int64_t)64 * 128 * KS));
        const float v = A[((size_t)k * M + 64 * s + kk) * M + j] * scale;
        const __half hi = __float2half_rn(v);
        const __half lo = __float2half_rn(v - __half2float(hi));
        uint8_t* base = img + (size_t)((k * KS + s) * 2) * kFTile;
        const uint32_t off = ptx::sw128_offset((uint32_t)j, (uint32_t)kk);
        *reinterpret_cast<__half*>(base + off) = hi;
        *reinterpret_cast<__half*>(base + kFTile + off) = lo;
    }
}

int fc_padded_s(int S) { return S <= 1 ? 1 : (S <= 2 ? 2 : 4); }
int fc_leff(const elmrnn* h) { return std::min(h->fc_lags, std::max(h->Q - 1, 0)); }

template <int SS>
cudaError_t launch_fc_ss(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    static FcParams p;   // host staging of the parameter block
    p.X = X; p.ldx = ldx; p.N = N; p.H = H; p.ldh = ldh;
    p.Aimg = static_cast<const uint8_t*>(h->tc_ops);
    p.S = h->S; p.Q = h->Q; p.L = fc_leff(h); p.NS = p.L + 1; p.act = h->act;
    p.two_pass = h->weight_grid == 1;
    p.ntiles = (N + kFRows - 1) / kFRows;
    p.xbytes = ptx::xstage_host(X, ldx, kFSmem);   // a1: stage each full tile's X block when it fits
    p.rbeta = h->ro_beta; p.ryp = h->ro_yp;
    h->ro_slots = 4;
    const int smem = kFSmem + (int)p.xbytes;
    p.k_act = (h->act == 1 ? 2.8853900817779268f : -1.4426950408889634f) * h->tc_inv_scale;
    std::copy(h->tc_wb.begin(), h->tc_wb.end(), p.wb);
    const int grid = (int)std::min<int64_t>(p.ntiles, h->sm_count);
    const size_t need = (size_t)grid * p.NS * kFSlotBytes;
    cudaError_t e;
    if (need > h->scratch_bytes) {
        if (h->scratch) cudaFree(h->scratch);
        h->scratch = nullptr;
        h->scratch_bytes = 0;
        if ((e = cudaMalloc(&h->scratch, need))) return e;
        h->scratch_bytes = need;
    }
    p.hist = reinterpret_cast<uint8_t*>(h->scratch);
    if ((e = cudaFuncSetAttribute(k_fc_tc<SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    k_fc_tc<SS><<<grid, kFThreads, smem, h->stream>>>(p);
    h->launches++;
    return cudaGetLastError();
}

}  // namespace

bool fc_tc_supported(const elmrnn* h) {
    return h->arch == kArchFC && h->M == kFM && h->S <= 4 && (fc_padded_s(h->S) + 1) * kFM <= kFWbMax;
}

cudaError_t fc_tc_prepare(elmrnn* h) {
    const int M = h->M, S = h->S, SP = fc_padded_s(S), Leff = fc_leff(h);
    const size_t bytes = (size_t)std::max(Leff, 1) * kFSlotBytes;
    cudaError_t e;
    if ((e = cudaMalloc(&h->tc_ops, bytes))) return e;
    h->tc_ops_bytes = bytes;
    // sigma: largest power of two keeping |A_k| 2^sigma < 1 (|A_k| <= 1/sqrt(M L))
    const int sigma = h->rec_scale == 1 ? 0 : (int)std::floor(std::log2(std::sqrt((double)M * h->fc_lags)));
    const float scale = std::ldexp(1.0f, sigma);
    h->tc_inv_scale = std::ldexp(1.0f, -sigma);
    std::vector<float> W((size_t)S * M), b(M);
    if ((e = cudaMemcpyAsync(W.data(), h->W, sizeof(float) * S * M, cudaMemcpyDeviceToHost, h->stream))) return e;
    if ((e = cudaMemcpyAsync(b.data(), h->b, sizeof(float) * M, cudaMemcpyDeviceToHost, h->stream))) return e;
    if ((e = cudaStreamSynchronize(h->stream))) return e;
    h->tc_wb.assign((size_t)M * (SP + 1), 0.0f);
    for (int j = 0; j < M; ++j) {
        float* d = h->tc_wb.data() + (size_t)j * (SP + 1);
        d[0] = b[j] * scale;
        for (int s2 = 0; s2 < S; ++s2) d[1 + s2] = W[(size_t)s2 * M + j] * scale;
    }
    if (Leff > 0) {
        const int64_t total = (int64_t)Leff * (M / 64) * 128 * 64;
        const int blocks = (int)std::min<int64_t>((total + 255) / 256, 4096);
        k_pack_fc<<<blocks, 256, 0, h->stream>>>(h->rec, M, Leff, scale, static_cast<uint8_t*>(h->tc_ops));
        h->launches++;
    }
    return cudaGetLastError();
}

cudaError_t launch_fc_tc(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    switch (fc_padded_s(h->S)) {
    case 1: return launch_fc_ss<1>(h, X, ldx, N, H, ldh);
    case 2: return launch_fc_ss<2>(h, X, ldx, N, H, ldh);
    case 4: return launch_fc_ss<4>(h, X, ldx, N, H, ldh);
    }
    return cudaErrorNotSupported;
}

}  // namespace elm
