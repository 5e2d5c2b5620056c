// hbuild_gru_wide.cu -- tcgen05 tensor-core H builder for the GRU (S2.2.6,
// P:144-150, Cho form with dense U, readings R10-R12) at WIDE hidden layers,
// 128 < M <= 1024 (BASELINE configs[4], C5):
//   z = sigma(x W_z + h U_z + b_z),  r = sigma(x W_r + h U_r + b_r)
//   n = tanh(x W_f + (r o h) U_f + b_f),  h <- (1 - z) o h + z o n
// The M = 128 kernel (hbuild_gru_tc.cu) keeps both A operands in TMEM; here
// they do not fit, so the design of the wide LSTM builder (hbuild_lstm_wide.cu)
// is used for both phases of a step:
//   phase 1: NC1 = M/64 chunks of 128 columns (64 neurons x (z, r)),
//            A = h(t-1) from a per-CTA global SW128 image (slot t % 2);
//   phase 2: NC2 = M/128 chunks of 128 columns (128 neurons, gate f),
//            A = r o h(t-1) from a second per-CTA image written by phase 1.
// h(t) and z live in per-CTA global fp32 arrays laid out
// [neuron / 8][row][neuron % 8] (1 KB contiguous per warp access).
// Precision: 3-pass fp16 hi/lo split (2-pass with fp16-grid weights), U_cat
// pre-scaled by 2^sigma, exp2 constants folded into W|b.
//   smem: 3 stages x [A slice hi|lo 32 KB, B slice hi|lo 32 KB]; TMEM 2 x 128 columns
//   warps 0..15 epilogue, 16 bulk-copy producer + TMEM allocator, 17 MMA issuer.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace elm {

namespace {

constexpr int kQRows = 128;
constexpr int kQTile = 128 * 64 * 2;
constexpr int kQPair = 2 * kQTile;
constexpr int kQEpiWarps = 16;
constexpr int kQProdWarp = kQEpiWarps, kQMmaWarp = kQEpiWarps + 1;
constexpr int kQThreads = (kQEpiWarps + 2) * 32;
// PAIR (M % 256 == 0): MMA units of two chunks of the same phase (N = 256), as in
// hbuild_lstm_wide.cu: the A image is streamed once per chunk pair; 2 stages of 96 KB.
template <bool PAIR>
struct QCfg {
    static constexpr int STAGES = PAIR ? 2 : 3;
    static constexpr int BTILE = PAIR ? 2 * kQTile : kQTile;
    static constexpr int STAGE = kQPair + 2 * BTILE;
    static constexpr int SMEM = 1024 + STAGES * STAGE + 256;   // + the X block
    static constexpr int ACC = PAIR ? 256 : 128;
    static constexpr int TMEM_COLS = 2 * ACC;
};

struct GruWideParams {
    const float* X;
    int64_t ldx, N;
    float* H;
    int64_t ldh;
    const uint8_t* Uimg;   // [NC1 + NC2][KS][hi|lo][16 KB]
    const float* wb;       // [M][3][SS+1]: k_g (b, W_0..W_{S-1})
    uint8_t* img;          // [grid][3][KS][hi|lo][16 KB]: h slots 0, 1 and r o h
    float* hst;            // [grid][M/8][128][8] h(t)
    float* zst;            // [grid][M/8][128][8] z
    int M, S, Q, NC1, NC2, KS;
    int two_pass;
    int64_t ntiles;
    uint32_t xbytes;       // a1: bytes of a tile's X block staged by cp.async.bulk (0: x(t) via L1)
    const double* rbeta;   // fused readout (Eq. 4): no H store; ryp[u * N + row] = H[row][u's neurons] . beta
    double* ryp;
    float k_sig, k_tanh;
};

__device__ __forceinline__ void tmem_ld16q(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void fence_proxy_async_global_q() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
// 8 fp32 values -> fp16 hi|lo (two uint4) at K index k (multiple of 8) of row r in an image
__device__ __forceinline__ void put_hilo8(uint8_t* image, int r, int k, const float* v) {
    uint4 hi, lo;
    uint32_t* hp = &hi.x;
    uint32_t* lp = &lo.x;
#pragma unroll
    for (int w2 = 0; w2 < 4; ++w2) {
        const __half2 h2 = __floats2half2_rn(v[2 * w2], v[2 * w2 + 1]);
        const float2 hf = __half22float2(h2);
        const __half2 l2 = __floats2half2_rn(v[2 * w2] - hf.x, v[2 * w2 + 1] - hf.y);
        hp[w2] = *reinterpret_cast<const uint32_t*>(&h2);
        lp[w2] = *reinterpret_cast<const uint32_t*>(&l2);
    }
    uint8_t* sl = image + (size_t)(k >> 6) * kQPair;
    const uint32_t off = ptx::sw128_offset((uint32_t)r, (uint32_t)(k & 63));
    *reinterpret_cast<uint4*>(sl + off) = hi;
    *reinterpret_cast<uint4*>(sl + kQTile + off) = lo;
}
__device__ __forceinline__ void ld8(const float* p, float* v) {
    const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void st8(float* p, const float* v) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

template <int SS, bool PAIR>
__global__ void __launch_bounds__(kQThreads, 1) k_gru_wide(const __grid_constant__ GruWideParams p) {
    using CF = QCfg<PAIR>;
    constexpr int kQStages = CF::STAGES, kQStageBytes = CF::STAGE;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stages = smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(stages + kQStages * kQStageBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + kQStages;
    uint64_t* acc_full = bars + 2 * kQStages;   // [2]
    uint64_t* acc_empty = acc_full + 2;         // [2]
    uint64_t* hist_ready = acc_empty + 2;       // h(t) image complete (t < Q)
    uint64_t* rh_ready = hist_ready + 1;        // r o h(t-1) image complete (t >= 2)
    uint64_t* x_full = rh_ready + 1;            // the tile's X block has landed
    uint64_t* x_empty = x_full + 1;             // every epilogue warp has read its last x(t)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(x_empty + 1);
    float* xbuf = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);   // the tile's X block

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kQStages; ++i) {
            ptx::mbar_init(full + i, 1);
            ptx::mbar_init(empty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(acc_full + i, 1);
            ptx::mbar_init(acc_empty + i, kQEpiWarps);
        }
        ptx::mbar_init(hist_ready, kQEpiWarps);
        ptx::mbar_init(rh_ready, kQEpiWarps);
        ptx::mbar_init(x_full, 1);
        ptx::mbar_init(x_empty, kQEpiWarps);
        ptx::fence_mbar_init();
    }
    if (warp == kQProdWarp) {
        ptx::tmem_alloc(tmem_slot, CF::TMEM_COLS);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int M = p.M, NC1 = p.NC1, NC2 = p.NC2, KS = p.KS;
    const size_t img_bytes = (size_t)KS * kQPair;
    uint8_t* img = p.img + (size_t)blockIdx.x * 3 * img_bytes;
    uint8_t* rh_img = img + 2 * img_bytes;

    if (warp == kQProdWarp) {
        uint32_t st = 0, ph = 0, hph = 0, rph = 0, xph = 0;
        const uint32_t bbytes = p.two_pass ? CF::BTILE : 2 * CF::BTILE;
        auto load = [&](const uint8_t* a_img, int chunk) {   // chunk = MMA unit index
            for (int ks = 0; ks < KS; ++ks) {
                ptx::mbar_wait(empty + st, ph ^ 1);
                if (ptx::elect_one()) {
                    uint8_t* sb = stages + st * kQStageBytes;
                    ptx::mbar_arrive_expect_tx(full + st, kQPair + bbytes);
                    ptx::bulk_g2s(sb, a_img + (size_t)ks * kQPair, kQPair, full + st);
                    ptx::bulk_g2s(sb + kQPair, p.Uimg + (size_t)(chunk * KS + ks) * 2 * CF::BTILE, bbytes, full + st);
                }
                __syncwarp();
                if (++st == kQStages) { st = 0; ph ^= 1; }
            }
        };
        for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            if (ptx::xstage_tile(p.xbytes, tile, p.N))   // the tile's X block (a1)
                ptx::xstage_issue(xbuf, p.X, p.ldx, tile, p.xbytes, x_full, x_empty, xph);
            for (int t = 2; t <= p.Q; ++t) {
                ptx::mbar_wait(hist_ready, hph);
                hph ^= 1;
                fence_proxy_async_global_q();
                const uint8_t* hslot = img + (size_t)((t - 1) & 1) * img_bytes;
                const int U1 = PAIR ? NC1 / 2 : NC1, U2 = PAIR ? NC2 / 2 : NC2;
                for (int c = 0; c < U1; ++c) load(hslot, c);
                ptx::mbar_wait(rh_ready, rph);
                rph ^= 1;
                fence_proxy_async_global_q();
                for (int c = 0; c < U2; ++c) load(rh_img, U1 + c);
            }
        }
    } else if (warp == kQMmaWarp) {
        constexpr uint32_t idesc = ptx::idesc_f16(128, CF::ACC);
        const uint64_t dbase = ptx::desc_sw128_kmajor(ptx::smem_u32(stages));
        const bool two = p.two_pass != 0;
        uint32_t st = 0, ph = 0, ach = 0, aph = 0;
        const int NU = PAIR ? (NC1 + NC2) / 2 : NC1 + NC2;
        for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            for (int t = 2; t <= p.Q; ++t) {
                for (int n = 0; n < NU; ++n) {
                    ptx::mbar_wait(acc_empty + ach, aph ^ 1);
                    ptx::tc_fence_after();
                    const uint32_t d = tmem + ach * CF::ACC;
                    for (int ks = 0; ks < KS; ++ks) {
                        ptx::mbar_wait(full + st, ph);
                        ptx::tc_fence_after();
                        const uint64_t ah = dbase + (uint64_t)((st * kQStageBytes) >> 4);
                        const uint64_t al = ah + (uint64_t)(kQTile >> 4);
                        const uint64_t bh = ah + (uint64_t)(kQPair >> 4);
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
                        if (++st == kQStages) { st = 0; ph ^= 1; }
                    }
                    if (++ach == 2) { ach = 0; aph ^= 1; }
                }
            }
        }
    } else {
        const int q = warp & 3, u = warp >> 2;
        const int r = 32 * q + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
        const float kS = p.k_sig, kT = p.k_tanh;
        float* hst = p.hst + (size_t)blockIdx.x * M * 128;
        float* zst = p.zst + (size_t)blockIdx.x * M * 128;
        auto sidx = [&](int j) { return ((size_t)(j >> 3) * 128 + r) * 8; };   // 8 consecutive neurons j..j+7
        uint32_t ach = 0, aph = 0, xph = 0;
        for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            const int64_t row = tile * kQRows + r;
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
                // ---- phase 1: z, r of neurons 64 c + 16 u + 0..15; r o h(t-1) -> image
                for (int c = 0; c < NC1; ++c) {
                    float a[2][16];   // 16 neurons x (z, r) interleaved
                    if (t >= 2) {
                        const bool first = !PAIR || (c & 1) == 0, last = !PAIR || (c & 1) == 1;
                        if (first) {
                            ptx::mbar_wait(acc_full + ach, aph);
                            ptx::tc_fence_after();
                        }
                        const uint32_t acol = ach * CF::ACC + (PAIR ? (c & 1) * 128 : 0);
                        tmem_ld16q(lane_base + acol + 32 * u, a[0]);
                        tmem_ld16q(lane_base + acol + 32 * u + 16, a[1]);
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
#pragma unroll
                    for (int half = 0; half < 2; ++half) {
                        const int j0 = 64 * c + 16 * u + 8 * half;
                        float hp[8], zv[8], rh[8];
                        if (t >= 2) ld8(hst + sidx(j0), hp);
                        else {
#pragma unroll
                            for (int i = 0; i < 8; ++i) hp[i] = 0.0f;
                        }
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            const int j = j0 + i;
                            const float* w = p.wb + (size_t)j * (3 * (SS + 1));
                            float pz = fmaf(kS, a[half][2 * i], __ldg(w));
                            float pr = fmaf(kS, a[half][2 * i + 1], __ldg(w + SS + 1));
#pragma unroll
                            for (int s = 0; s < SS; ++s) {
                                pz = fmaf(xs[s], __ldg(w + 1 + s), pz);
                                pr = fmaf(xs[s], __ldg(w + SS + 2 + s), pr);
                            }
                            zv[i] = sig_e2(pz);           // z (accurate form, DESIGN R26)
                            rh[i] = sig_e2(pr) * hp[i];   // r o h(t-1)
                        }
                        st8(zst + sidx(j0), zv);
                        if (t >= 2) put_hilo8(rh_img, r, j0, rh);
                    }
                }
                if (t >= 2) {   // r o h(t-1) complete: phase 2 may start
                    fence_proxy_async_global_q();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(rh_ready);
                }
                // ---- phase 2: n = tanh(.), h <- (1 - z) h + z n for neurons 128 c + 32 u + 0..31
                for (int c = 0; c < NC2; ++c) {
                    float a2[2][16];
                    if (t >= 2) {
                        const bool first = !PAIR || (c & 1) == 0, last = !PAIR || (c & 1) == 1;
                        if (first) {
                            ptx::mbar_wait(acc_full + ach, aph);
                            ptx::tc_fence_after();
                        }
                        const uint32_t acol = ach * CF::ACC + (PAIR ? (c & 1) * 128 : 0);
                        tmem_ld16q(lane_base + acol + 32 * u, a2[0]);
                        tmem_ld16q(lane_base + acol + 32 * u + 16, a2[1]);
                        ptx::tmem_wait_ld();
                        if (last) {
                            ptx::tc_fence_before();
                            __syncwarp();
                            if (lane == 0) ptx::mbar_arrive(acc_empty + ach);
                            if (++ach == 2) { ach = 0; aph ^= 1; }
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i) a2[0][i] = a2[1][i] = 0.0f;
                    }
#pragma unroll
                    for (int g8 = 0; g8 < 4; ++g8) {
                        const int j0 = 128 * c + 32 * u + 8 * g8;
                        float hp[8], zv[8];
                        if (t >= 2) ld8(hst + sidx(j0), hp);
                        else {
#pragma unroll
                            for (int i = 0; i < 8; ++i) hp[i] = 0.0f;
                        }
                        ld8(zst + sidx(j0), zv);
#pragma unroll
                        for (int i = 0; i < 8; i += 2) {
                            float dn[2];
#pragma unroll
                            for (int k2 = 0; k2 < 2; ++k2) {
                                const int j = j0 + i + k2;
                                const float* w = p.wb + (size_t)j * (3 * (SS + 1)) + 2 * (SS + 1);
                                float pn = fmaf(kT, a2[g8 >> 1][(g8 & 1) * 8 + i + k2], __ldg(w));
#pragma unroll
                                for (int s = 0; s < SS; ++s) pn = fmaf(xs[s], __ldg(w + 1 + s), pn);
                                dn[k2] = tanh_e2_sig(pn);
                            }
                            const float n0 = dn[0], n1 = dn[1];
                            hp[i] = fmaf(zv[i], n0 - hp[i], hp[i]);        // (1 - z) h + z n
                            hp[i + 1] = fmaf(zv[i + 1], n1 - hp[i + 1], hp[i + 1]);
                        }
                        if (t < p.Q) {
                            st8(hst + sidx(j0), hp);
                            put_hilo8(img + (size_t)(t & 1) * img_bytes, r, j0, hp);
                        } else if (valid && p.rbeta) {
#pragma unroll
                            for (int i = 0; i < 8; ++i) yacc = fma((double)hp[i], __ldg(p.rbeta + j0 + i), yacc);
                        } else if (valid) {
                            float* d1 = p.H + row * p.ldh + j0;
                            if (((p.ldh | (int64_t)(reinterpret_cast<uintptr_t>(p.H) >> 2)) & 3) == 0) st8(d1, hp);
                            else {
#pragma unroll
                                for (int i = 0; i < 8; ++i) d1[i] = hp[i];
                            }
                        }
                    }
                }
                if (t < p.Q) {   // h(t) complete: step t+1's phase 1 may start
                    fence_proxy_async_global_q();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(hist_ready);
                }
            }
            if (p.rbeta && valid) p.ryp[u * p.N + row] = yacc;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kQProdWarp) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, CF::TMEM_COLS);
    }
}

// U images: phase-1 chunk q < NC1 rows nrow = 2 jj + g (neuron 64 q + jj, gate z|r),
// phase-2 chunk q2 rows = neuron 128 q2 + nrow (gate f); K-major SW128, hi | lo, x 2^sigma.
// pair = 1: chunks 2m, 2m+1 adjacent (one 256-row tile per K-slice and part), as k_pack_u
__global__ void k_pack_u_gru_wide(const float* __restrict__ U, int M, float scale, uint8_t* __restrict__ img,
                                  int pair) {
    const int KS = M / 64, NC1 = M / 64, NC = NC1 + M / 128;
    const int64_t total = (int64_t)NC * KS * 128 * 64;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int kk = (int)(e % 64);
        const int nrow = (int)((e / 64) % 128);
        const int ks = (int)((e / (64 * 128)) % KS);
        const int q = (int)(e / ((int64_t)64 * 128 * KS));
        const int col = q < NC1 ? (nrow & 1) * M + 64 * q + (nrow >> 1) : 2 * M + 128 * (q - NC1) + nrow;
        const float v = U[(size_t)(64 * ks + kk) * (3 * M) + col] * scale;
        const __half hi = __float2half_rn(v);
        const __half lo = __float2half_rn(v - __half2float(hi));
        uint8_t* base = pair ? img + (size_t)(((q >> 1) * KS + ks) * 2) * 2 * kQTile + (size_t)(q & 1) * kQTile
                             : img + (size_t)((q * KS + ks) * 2) * kQTile;
        const uint32_t off = ptx::sw128_offset(nrow, kk);
        *reinterpret_cast<__half*>(base + off) = hi;
        *reinterpret_cast<__half*>(base + (pair ? 2 : 1) * kQTile + off) = lo;
    }
}

int gw_padded_s(int S) { return S <= 1 ? 1 : (S <= 2 ? 2 : 4); }
size_t gw_img_bytes(int M) { return (size_t)(M / 64 + M / 128) * (M / 64) * kQPair; }

bool gw_pair(const elmrnn* h) { return h->tune.wide_pair != 0 && h->M % 256 == 0; }

template <int SS, bool PAIR>
cudaError_t launch_gw(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    constexpr int kQSmem = QCfg<PAIR>::SMEM;
    GruWideParams p{};
    p.X = X; p.ldx = ldx; p.N = N; p.H = H; p.ldh = ldh;
    p.M = h->M; p.S = h->S; p.Q = h->Q; p.NC1 = h->M / 64; p.NC2 = h->M / 128; p.KS = h->M / 64;
    p.two_pass = h->weight_grid == 1;
    p.ntiles = (N + kQRows - 1) / kQRows;
    p.xbytes = ptx::xstage_host(X, ldx, kQSmem);   // a1: stage each full tile's X block when it fits
    p.rbeta = h->ro_beta; p.ryp = h->ro_yp;
    h->ro_slots = 4;
    const int smem = kQSmem + (int)p.xbytes;
    p.k_sig = -1.4426950408889634f * h->tc_inv_scale;
    p.k_tanh = 2.8853900817779268f * h->tc_inv_scale;
    p.Uimg = static_cast<const uint8_t*>(h->tc_ops);
    p.wb = reinterpret_cast<const float*>(static_cast<const uint8_t*>(h->tc_ops) + gw_img_bytes(h->M));
    const int grid = (int)std::min<int64_t>(p.ntiles, h->sm_count);
    const size_t img = (size_t)grid * 3 * p.KS * kQPair;
    const size_t st = (size_t)grid * p.M * 128 * sizeof(float);
    cudaError_t e;
    if (img + 2 * st > h->scratch_bytes) {
        if (h->scratch) cudaFree(h->scratch);
        h->scratch = nullptr;
        h->scratch_bytes = 0;
        if ((e = cudaMalloc(&h->scratch, img + 2 * st))) return e;
        h->scratch_bytes = img + 2 * st;
    }
    uint8_t* base = reinterpret_cast<uint8_t*>(h->scratch);
    p.img = base;
    p.hst = reinterpret_cast<float*>(base + img);
    p.zst = reinterpret_cast<float*>(base + img + st);
    if ((e = cudaFuncSetAttribute(k_gru_wide<SS, PAIR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    k_gru_wide<SS, PAIR><<<grid, kQThreads, smem, h->stream>>>(p);
    h->launches++;
    return cudaGetLastError();
}

}  // namespace

bool gru_wide_supported(const elmrnn* h) {
    return h->arch == kArchGRU && h->M > 128 && h->M <= 1024 && h->M % 128 == 0 && h->S <= 4;
}

cudaError_t gru_wide_prepare(elmrnn* h) {
    cudaError_t e;
    const int M = h->M, S = h->S, SP = gw_padded_s(S), GM = 3 * M;
    const size_t ib = gw_img_bytes(M);
    const size_t bytes = ib + sizeof(float) * (size_t)M * 3 * (SP + 1);
    if ((e = cudaMalloc(&h->tc_ops, bytes))) return e;
    h->tc_ops_bytes = bytes;
    const int sigma = h->rec_scale == 1 ? 0 : (int)std::floor(std::log2(std::sqrt((double)M)));
    const float scale = std::ldexp(1.0f, sigma);
    h->tc_inv_scale = std::ldexp(1.0f, -sigma);
    std::vector<float> W((size_t)S * GM), b(GM);
    if ((e = cudaMemcpyAsync(W.data(), h->W, sizeof(float) * S * GM, cudaMemcpyDeviceToHost, h->stream))) return e;
    if ((e = cudaMemcpyAsync(b.data(), h->b, sizeof(float) * GM, cudaMemcpyDeviceToHost, h->stream))) return e;
    if ((e = cudaStreamSynchronize(h->stream))) return e;
    h->tc_wb.assign((size_t)M * 3 * (SP + 1), 0.0f);
    for (int j = 0; j < M; ++j)
        for (int g = 0; g < 3; ++g) {
            const double kg = g == 2 ? 2.8853900817779268 : -1.4426950408889634;
            float* d = h->tc_wb.data() + ((size_t)j * 3 + g) * (SP + 1);
            d[0] = (float)(kg * b[g * M + j]);
            for (int s2 = 0; s2 < S; ++s2) d[1 + s2] = (float)(kg * W[(size_t)s2 * GM + g * M + j]);
        }
    if ((e = cudaMemcpyAsync(static_cast<uint8_t*>(h->tc_ops) + ib, h->tc_wb.data(), sizeof(float) * h->tc_wb.size(),
                             cudaMemcpyHostToDevice, h->stream)))
        return e;
    const int64_t total = (int64_t)(M / 64 + M / 128) * (M / 64) * 128 * 64;
    k_pack_u_gru_wide<<<(int)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, h->stream>>>(
        h->rec, M, scale, static_cast<uint8_t*>(h->tc_ops), gw_pair(h) ? 1 : 0);
    h->launches++;
    return cudaGetLastError();
}

cudaError_t launch_gru_wide(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    switch (gw_padded_s(h->S)) {
    case 1: return gw_pair(h) ? launch_gw<1, true>(h, X, ldx, N, H, ldh) : launch_gw<1, false>(h, X, ldx, N, H, ldh);
    case 2: return gw_pair(h) ? launch_gw<2, true>(h, X, ldx, N, H, ldh) : launch_gw<2, false>(h, X, ldx, N, H, ldh);
    default: return gw_pair(h) ? launch_gw<4, true>(h, X, ldx, N, H, ldh) : launch_gw<4, false>(h, X, ldx, N, H, ldh);
    }
}

}  // namespace elm
