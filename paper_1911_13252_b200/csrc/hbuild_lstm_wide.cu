// hbuild_lstm_wide.cu -- tcgen05 tensor-core H builder for the LSTM (S2.2.5,
// P:128-142, dense U, reading R10) at WIDE hidden layers, 256 < M <= 1024
// (BASELINE configs[4], C5: M in {512, 1024}):
//   a(t) = h(t-1) [128 x M] . U_cat [M x 4M]   + x(t) W + b,  gates (o, c, lambda, in)
//
// At M = 256 the whole recurrent state of a 128-row tile lives on chip
// (hbuild_dense_tc.cu: A = h(t-1) in TMEM, c(t) in registers).  Beyond that it
// does not fit (h(t-1) as fp16 hi|lo is 256 KB at M = 512, c(t) another
// 256 KB), so this kernel follows the FC builder's design instead:
//   * h(t) is written by the epilogue straight into a per-CTA global image
//     (two slots, t % 2) in the MMA's K-major SW128 fp16 hi|lo layout, and
//     streamed back per (chunk, K-slice) by the bulk-copy producer together
//     with the matching U_cat slice: both operands from shared memory (SS).
//   * c(t) lives in a per-CTA global array laid out so each epilogue warp
//     reads and writes 1 KB contiguous per chunk.
// Precision and gate epilogue are those of the M <= 256 kernel: 3-pass fp16
// hi/lo split (2-pass with fp16-grid weights) into one fp32 TMEM accumulator,
// U pre-scaled by 2^sigma, exp2 constants folded into W|b, shared reciprocals.
//
//   smem: 3 stages x [A = h(t-1) slice hi|lo 32 KB, B = U_cat slice hi|lo 32 KB]
//   TMEM: 2 x 128 accumulator columns (chunk n+1's MMAs overlap chunk n's epilogue)
//   warps 0..15 epilogue (quadrant w % 4, neurons 8 (w / 4) .. +7 of a chunk),
//   16 bulk-copy producer + TMEM allocator, 17 MMA issuer.
//   Per step t >= 2: NCH = M/32 chunks x KS = M/64 K-slices; step 1 has h(0) = 0
//   and needs no MMA.  Step t+1's loads wait for every epilogue warp to have
//   written its part of h(t) (one mbarrier per step).
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace elm {

namespace {

constexpr int kWRows = 128;
constexpr int kWTile = 128 * 64 * 2;          // one 128 x 64 fp16 SW128 tile (16 KB)
constexpr int kWPair = 2 * kWTile;            // hi + lo
constexpr int kWEpiWarps = 16;
constexpr int kWProdWarp = kWEpiWarps, kWMmaWarp = kWEpiWarps + 1;
constexpr int kWThreads = (kWEpiWarps + 2) * 32;
// PAIR: one MMA unit = two 32-neuron chunks (N = 256 accumulator columns, 128 x 256 x 16
// MMAs): h(t-1) is streamed once per chunk PAIR instead of once per chunk, and each
// stage carries 32 KB of A for 64 KB of B (the SS operand bytes per MMA flop drop by a
// quarter); 2 stages of 96 KB.  Else 3 stages of 64 KB, N = 128.
template <bool PAIR>
struct WCfg {
    static constexpr int STAGES = PAIR ? 2 : 3;
    static constexpr int BTILE = PAIR ? 2 * kWTile : kWTile;    // B hi (or lo) bytes per stage
    static constexpr int STAGE = kWPair + 2 * BTILE;              // A hi|lo + B hi|lo
    static constexpr int SMEM = 1024 + STAGES * STAGE + 256;      // + the X block
    static constexpr int ACC = PAIR ? 256 : 128;                  // accumulator columns per unit
    static constexpr int TMEM_COLS = 2 * ACC;
};

struct WideParams {
    const float* X;
    int64_t ldx, N;
    float* H;
    int64_t ldh;
    const uint8_t* Uimg;   // [units][KS][hi|lo][16 KB per chunk of the unit] (hbuild_dense_tc.cu k_pack_u)
    const float* wb;       // [M][4][SS+1]: k_g (b, W_0..W_{S-1})
    uint8_t* hist;         // [grid][2][KS][hi|lo][16 KB]: A images of h(t)
    float* cst;            // [grid][NCH][4][128][8]: c(t)
    int M, S, Q, NCH, KS;
    int two_pass;
    int64_t ntiles;
    uint32_t xbytes;       // a1: bytes of a tile's X block staged by cp.async.bulk (0: x(t) via L1)
    const double* rbeta;   // fused readout (Eq. 4): no H store; ryp[u * N + row] = H[row][u's neurons] . beta
    double* ryp;
    float k_sig, k_tanh;   // -log2(e) 2^-sigma, 2 log2(e) 2^-sigma
};

__device__ __forceinline__ void tmem_ld16w(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void fence_proxy_async_global_w() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int SS, bool PAIR>
__global__ void __launch_bounds__(kWThreads, 1) k_lstm_wide(const __grid_constant__ WideParams p) {
    using CF = WCfg<PAIR>;
    constexpr int kWStages = CF::STAGES, kWStageBytes = CF::STAGE;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stages = smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(stages + kWStages * kWStageBytes);
    uint64_t* full = bars;                        // [kWStages]
    uint64_t* empty = bars + kWStages;            // [kWStages]
    uint64_t* acc_full = bars + 2 * kWStages;     // [2]
    uint64_t* acc_empty = acc_full + 2;           // [2]
    uint64_t* hist_ready = acc_empty + 2;         // all of h(t) is in the image (t < Q)
    uint64_t* x_full = hist_ready + 1;            // the tile's X block has landed
    uint64_t* x_empty = x_full + 1;               // every epilogue warp has read its last x(t)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(x_empty + 1);
    float* xbuf = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);   // the tile's X block

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kWStages; ++i) {
            ptx::mbar_init(full + i, 1);
            ptx::mbar_init(empty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(acc_full + i, 1);
            ptx::mbar_init(acc_empty + i, kWEpiWarps);
        }
        ptx::mbar_init(hist_ready, kWEpiWarps);
        ptx::mbar_init(x_full, 1);
        ptx::mbar_init(x_empty, kWEpiWarps);
        ptx::fence_mbar_init();
    }
    if (warp == kWProdWarp) {
        ptx::tmem_alloc(tmem_slot, CF::TMEM_COLS);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int NCH = p.NCH, KS = p.KS, NU = PAIR ? NCH / 2 : NCH;   // MMA units per step
    const size_t slot_bytes = (size_t)KS * kWPair;
    uint8_t* hist = p.hist + (size_t)blockIdx.x * 2 * slot_bytes;

    if (warp == kWProdWarp) {
        // ---------------- producer: per step t >= 2, (chunk n, K-slice ks) pairs of
        // [h(t-1) slice ks | U_cat chunk n slice ks]; whole warp loops, one lane issues
        uint32_t st = 0, ph = 0, hph = 0, xph = 0;
        const uint32_t bbytes = p.two_pass ? CF::BTILE : 2 * CF::BTILE;   // U hi only when U_lo = 0
        for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            if (ptx::xstage_tile(p.xbytes, tile, p.N))   // the tile's X block (a1)
                ptx::xstage_issue(xbuf, p.X, p.ldx, tile, p.xbytes, x_full, x_empty, xph);
            for (int t = 2; t <= p.Q; ++t) {
                const uint8_t* slot = hist + (size_t)((t - 1) & 1) * slot_bytes;
                ptx::mbar_wait(hist_ready, hph);   // h(t-1) fully written by the epilogue
                hph ^= 1;
                fence_proxy_async_global_w();
                for (int n = 0; n < NU; ++n) {
                    for (int ks = 0; ks < KS; ++ks) {
                        ptx::mbar_wait(empty + st, ph ^ 1);
                        if (ptx::elect_one()) {
                            uint8_t* sb = stages + st * kWStageBytes;
                            ptx::mbar_arrive_expect_tx(full + st, kWPair + bbytes);
                            ptx::bulk_g2s(sb, slot + (size_t)ks * kWPair, kWPair, full + st);
                            ptx::bulk_g2s(sb + kWPair, p.Uimg + (size_t)(n * KS + ks) * 2 * CF::BTILE, bbytes,
                                          full + st);
                        }
                        __syncwarp();
                        if (++st == kWStages) { st = 0; ph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == kWMmaWarp) {
        // ---------------- MMA issuer: 12 SS MMAs (4 K-steps x 3 passes) per stage
        constexpr uint32_t idesc = ptx::idesc_f16(128, CF::ACC);
        const uint64_t dbase = ptx::desc_sw128_kmajor(ptx::smem_u32(stages));
        const bool two = p.two_pass != 0;
        uint32_t st = 0, ph = 0, ach = 0, aph = 0;
        for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            for (int t = 2; t <= p.Q; ++t) {
                for (int n = 0; n < NU; ++n) {
                    ptx::mbar_wait(acc_empty + ach, aph ^ 1);
                    ptx::tc_fence_after();
                    const uint32_t d = tmem + ach * CF::ACC;
                    for (int ks = 0; ks < KS; ++ks) {
                        ptx::mbar_wait(full + st, ph);
                        ptx::tc_fence_after();
                        const uint64_t ah = dbase + (uint64_t)((st * kWStageBytes) >> 4);
                        const uint64_t al = ah + (uint64_t)(kWTile >> 4);
                        const uint64_t bh = ah + (uint64_t)(kWPair >> 4);
                        const uint64_t bl = bh + (uint64_t)(CF::BTILE >> 4);
                        if (ptx::elect_one()) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                ptx::mma_f16_ss(d, ah + 2 * kk, bh + 2 * kk, idesc, (ks == 0 && kk == 0) ? 0u : 1u);
                                ptx::mma_f16_ss(d, al + 2 * kk, bh + 2 * kk, idesc, 1u);
                                if (!two) ptx::mma_f16_ss(d, ah + 2 * kk, bl + 2 * kk, idesc, 1u);
                            }
                            ptx::mma_commit(empty + st);
                            if (ks == KS - 1) ptx::mma_commit(acc_full + ach);
                        }
                        __syncwarp();
                        if (++st == kWStages) { st = 0; ph ^= 1; }
                    }
                    if (++ach == 2) { ach = 0; aph ^= 1; }
                }
            }
        }
    } else {
        // ---------------- epilogue: gates, c/h update, h(t) image, H(Q) store
        const int q = warp & 3, u = warp >> 2;
        const int r = 32 * q + lane;                  // tile row = TMEM lane
        const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
        const float kS = p.k_sig, kT = p.k_tanh;
        float* cbase = p.cst + (size_t)blockIdx.x * NCH * 4 * 128 * 8;
        uint32_t ach = 0, aph = 0, xph = 0;
        for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            const int64_t row = tile * kWRows + r;
            const bool valid = row < p.N;
            const bool xst = ptx::xstage_tile(p.xbytes, tile, p.N);
            const float* xrow = xst ? xbuf + (int64_t)r * p.ldx : p.X + (valid ? row : 0) * p.ldx;
            if (xst) {
                ptx::mbar_wait(x_full, xph);
                xph ^= 1;
            }
            double yacc = 0.0;   // fused readout partial
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
                uint8_t* slot = hist + (size_t)(t & 1) * slot_bytes;
                for (int n = 0; n < NCH; ++n) {
                    float a[2][16];   // 2 groups x 4 neurons x (o, c, lambda, in), scaled domain
                    if (t >= 2) {
                        // PAIR: chunks 2m, 2m+1 are the two 128-column halves of one accumulator
                        const bool first = !PAIR || (n & 1) == 0, last = !PAIR || (n & 1) == 1;
                        if (first) {
                            ptx::mbar_wait(acc_full + ach, aph);
                            ptx::tc_fence_after();
                        }
                        const uint32_t acol = ach * CF::ACC + (PAIR ? (n & 1) * 128 : 0);
                        tmem_ld16w(lane_base + acol + (8 * u) * 4, a[0]);
                        tmem_ld16w(lane_base + acol + (8 * u + 4) * 4, a[1]);
                        ptx::tmem_wait_ld();
                        if (last) {
                            ptx::tc_fence_before();
                            __syncwarp();
                            if (lane == 0) ptx::mbar_arrive(acc_empty + ach);
                            if (++ach == 2) { ach = 0; aph ^= 1; }
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i) a[0][i] = a[1][i] = 0.0f;
                    }
                    float4* cptr = reinterpret_cast<float4*>(cbase + (((size_t)n * 4 + u) * 128 + r) * 8);
                    float c[8];
                    if (t >= 2) {
                        const float4 c0 = cptr[0], c1 = cptr[1];
                        c[0] = c0.x; c[1] = c0.y; c[2] = c0.z; c[3] = c0.w;
                        c[4] = c1.x; c[5] = c1.y; c[6] = c1.z; c[7] = c1.w;
                    } else {
#pragma unroll
                        for (int i = 0; i < 8; ++i) c[i] = 0.0f;
                    }
                    float hv[8];
#pragma unroll
                    for (int g4 = 0; g4 < 2; ++g4) {
#pragma unroll
                        for (int nb = 0; nb < 4; ++nb) {
                            const int j = n * 32 + 8 * u + 4 * g4 + nb;
                            const float* w = p.wb + (size_t)j * (4 * (SS + 1));   // [gate][b, W_0..W_{S-1}]
                            float arg[4];
#pragma unroll
                            for (int g = 0; g < 4; ++g) {
                                float v = fmaf(g == 1 ? kT : kS, a[g4][nb * 4 + g], __ldg(w + g * (SS + 1)));
#pragma unroll
                                for (int s = 0; s < SS; ++s) v = fmaf(xs[s], __ldg(w + g * (SS + 1) + 1 + s), v);
                                arg[g] = v;
                            }
                            // accurate gate forms (common.cuh sig_e2 / tanh_e2; DESIGN R26)
                            const float so = sig_e2(arg[0]), tc = tanh_e2(arg[1]);
                            const float sl = sig_e2(arg[2]), si = sig_e2(arg[3]);
                            const int ci = 4 * g4 + nb;
                            const float cn = fmaf(sl, c[ci], si * tc);
                            c[ci] = cn;
                            hv[4 * g4 + nb] = so * tanh_acc(cn);
                        }
                    }
                    if (t < p.Q) {
                        cptr[0] = make_float4(c[0], c[1], c[2], c[3]);
                        cptr[1] = make_float4(c[4], c[5], c[6], c[7]);
                        // h(t) of neurons K = 32 n + 8 u .. +7 -> slot t % 2, K-slice K / 64
                        uint4 hi, lo;
                        uint32_t* hp = &hi.x;
                        uint32_t* lp = &lo.x;
#pragma unroll
                        for (int w2 = 0; w2 < 4; ++w2) {
                            const __half2 h2 = __floats2half2_rn(hv[2 * w2], hv[2 * w2 + 1]);
                            const float2 hf = __half22float2(h2);
                            const __half2 l2 = __floats2half2_rn(hv[2 * w2] - hf.x, hv[2 * w2 + 1] - hf.y);
                            hp[w2] = *reinterpret_cast<const uint32_t*>(&h2);
                            lp[w2] = *reinterpret_cast<const uint32_t*>(&l2);
                        }
                        const int K = 32 * n + 8 * u;
                        uint8_t* sl = slot + (size_t)(K >> 6) * kWPair;
                        const uint32_t off = ptx::sw128_offset((uint32_t)r, (uint32_t)(K & 63));
                        *reinterpret_cast<uint4*>(sl + off) = hi;
                        *reinterpret_cast<uint4*>(sl + kWTile + off) = lo;
                    } else if (valid && p.rbeta) {
#pragma unroll
                        for (int i = 0; i < 8; ++i) yacc = fma((double)hv[i], __ldg(p.rbeta + n * 32 + 8 * u + i), yacc);
                    } else if (valid) {
                        float* d1 = p.H + row * p.ldh + n * 32 + 8 * u;
                        if (((p.ldh | (int64_t)(reinterpret_cast<uintptr_t>(p.H) >> 2)) & 3) == 0) {
                            float4* dst = reinterpret_cast<float4*>(d1);
                            dst[0] = make_float4(hv[0], hv[1], hv[2], hv[3]);
                            dst[1] = make_float4(hv[4], hv[5], hv[6], hv[7]);
                        } else {
#pragma unroll
                            for (int i = 0; i < 8; ++i) d1[i] = hv[i];
                        }
                    }
                }
                if (t < p.Q) {   // hand h(t) to the producer of step t+1
                    fence_proxy_async_global_w();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(hist_ready);
                }
            }
            if (p.rbeta && valid) p.ryp[u * p.N + row] = yacc;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kWProdWarp) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, CF::TMEM_COLS);
    }
}

template <int SS, bool PAIR>
cudaError_t launch_wide_ss(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    using CF = WCfg<PAIR>;
    constexpr int kWSmem = CF::SMEM;
    WideParams p{};
    p.X = X; p.ldx = ldx; p.N = N; p.H = H; p.ldh = ldh;
    p.M = h->M; p.S = h->S; p.Q = h->Q; p.NCH = h->M / 32; p.KS = h->M / 64;
    p.two_pass = h->weight_grid == 1;
    p.ntiles = (N + kWRows - 1) / kWRows;
    p.xbytes = ptx::xstage_host(X, ldx, kWSmem);   // a1: stage each full tile's X block when it fits
    p.rbeta = h->ro_beta; p.ryp = h->ro_yp;
    h->ro_slots = 4;
    const int smem = kWSmem + (int)p.xbytes;
    p.k_sig = -1.4426950408889634f * h->tc_inv_scale;
    p.k_tanh = 2.8853900817779268f * h->tc_inv_scale;
    const size_t img_bytes = (size_t)p.NCH * p.KS * kWPair;
    p.Uimg = static_cast<const uint8_t*>(h->tc_ops);
    p.wb = reinterpret_cast<const float*>(static_cast<const uint8_t*>(h->tc_ops) + img_bytes);
    const int grid = (int)std::min<int64_t>(p.ntiles, h->sm_count);
    const size_t hist_bytes = (size_t)grid * 2 * p.KS * kWPair;
    const size_t c_bytes = (size_t)grid * p.M * 128 * sizeof(float);
    cudaError_t e;
    if (hist_bytes + c_bytes > h->scratch_bytes) {
        if (h->scratch) cudaFree(h->scratch);
        h->scratch = nullptr;
        h->scratch_bytes = 0;
        if ((e = cudaMalloc(&h->scratch, hist_bytes + c_bytes))) return e;
        h->scratch_bytes = hist_bytes + c_bytes;
    }
    p.hist = reinterpret_cast<uint8_t*>(h->scratch);
    p.cst = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(h->scratch) + hist_bytes);
    if ((e = cudaFuncSetAttribute(k_lstm_wide<SS, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    k_lstm_wide<SS, PAIR><<<grid, kWThreads, smem, h->stream>>>(p);
    h->launches++;
    return cudaGetLastError();
}

}  // namespace

// chunk pairs (N = 256 MMA units): every wide M has an even chunk count (M % 64 == 0)
bool lstm_wide_pair(const elmrnn* h) { return h->tune.wide_pair != 0; }

bool lstm_wide_supported(const elmrnn* h) {
    return h->arch == kArchLSTM && h->M > 256 && h->M <= 1024 && h->M % 64 == 0 && h->S <= 4;
}

size_t lstm_wide_wb_offset(const elmrnn* h) { return (size_t)(h->M / 32) * (h->M / 64) * kWPair; }

cudaError_t launch_lstm_wide(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    switch (h->S <= 1 ? 1 : (h->S <= 2 ? 2 : 4)) {
    case 1: return lstm_wide_pair(h) ? launch_wide_ss<1, true>(h, X, ldx, N, H, ldh) : launch_wide_ss<1, false>(h, X, ldx, N, H, ldh);
    case 2: return lstm_wide_pair(h) ? launch_wide_ss<2, true>(h, X, ldx, N, H, ldh) : launch_wide_ss<2, false>(h, X, ldx, N, H, ldh);
    case 4: return lstm_wide_pair(h) ? launch_wide_ss<4, true>(h, X, ldx, N, H, ldh) : launch_wide_ss<4, false>(h, X, ldx, N, H, ldh);
    }
    return cudaErrorNotSupported;
}

}  // namespace elm
