// hbuild_gru_tc.cu -- tcgen05 tensor-core H builder for the GRU (S2.2.6,
// P:144-150, Cho form with dense U, readings R10-R12), M = 128:
//   z = sigma(x W_z + h U_z + b_z),  r = sigma(x W_r + h U_r + b_r)
//   n = tanh(x W_f + (r o h) U_f + b_f),  h <- (1 - z) o h + z o n
// Two dependent contractions per step: phase 1 [z | r] = h(t-1).[U_z | U_r]
// (N = 2M, two 128-column chunks), phase 2 (r o h).U_f (N = M, one chunk).
// Precision, U images, bulk-copy ring and MMA issue as in the LSTM builder
// (hbuild_dense_tc.cu): 3-pass fp16 hi/lo split into one fp32 TMEM
// accumulator, A operands in TMEM.
//
// TMEM (512 columns): accumulators [0,128) and [128,256); A_h = h(t-1) hi|lo
// [256,384); A_rh = r o h(t-1) hi|lo [384,512).  Both A operands are written
// directly by the epilogue (no staging): A_rh after phase 1 (it is only read
// by phase 2), A_h after phase 2 (only read by the next step's phase 1).
// Epilogue thread = (row, u): neurons 16u..16u+15 and 64+16u..64+16u+15; it
// keeps h(t) of its 32 neurons in registers and z in shared memory.
// The input term x W + b is one more K-step of every chunk's MMA chain (XMMA,
// below): A = [x(t), 1] from a shared-memory SW128 image, B = [W; b] streamed
// with the U slices, so the accumulator holds the whole pre-activation.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace elm {

namespace {

constexpr int kGM = 128;                        // hidden size handled by this kernel
constexpr int kGRows = 128;
constexpr int kGStages = 3;
constexpr int kGSliceBytes = 128 * 64 * 2;
constexpr int kGStageBytes = 2 * kGSliceBytes;
constexpr int kGEpiWarps = 16;
constexpr int kGProdWarp = kGEpiWarps, kGMmaWarp = kGEpiWarps + 1;
constexpr int kGThreads = (kGEpiWarps + 2) * 32;
constexpr int kGKS = kGM / 64;                  // K slices of h(t-1) / r o h(t-1)
constexpr int kGChunks = 3;                     // phase-1 chunks 0, 1; phase-2 chunk 2
#ifndef ELM_GRU_XMMA
#define ELM_GRU_XMMA 1
#endif
// XMMA: x(t) W + b joins the MMA as one more K-slice per chunk, A = [x(t), 1, 0..]
// (fp16 hi|lo, an SW128 image in shared memory written by the epilogue), B = [W; b]
// (rows of the chunk's gates, K = 0..S-1: W, K = S: b); only its first 16 K are used
// (one k-step).  The epilogue then needs no W|b loads and no x W FMAs: C3 GRU (S = 4)
// build 19.9 -> 10.5 ms, S = 1 7.38 -> 7.11 ms (tools/gru_ab.sh, same box).
constexpr int kGX = ELM_GRU_XMMA ? 1 : 0;
constexpr int kGSlices = kGKS + kGX;            // streamed B slices per chunk
constexpr int kGStagesPerStep = kGChunks * kGSlices;
constexpr int kGWbMax = 7168;
constexpr uint32_t kAcc = 0, kAH = 256, kARH = 384;   // TMEM column bases (hi at +0, lo at +64)
constexpr int kZBytes = kGEpiWarps * 32 * 32 * 4;     // z of 32 neurons per thread
constexpr int kGXImg = kGX * 2 * kGSliceBytes;        // A = [x, 1] hi | lo SW128 images
constexpr int kGSmem = 1024 + kGStages * kGStageBytes + kZBytes + kGXImg + 256;   // + the X block

struct GruParams {
    const float* X;
    int64_t ldx, N;
    float* H;
    int64_t ldh;
    const uint8_t* Uimg;   // [3 chunks][KS][hi|lo][16 KB]
    int S, Q;
    int two_pass;          // 1: U on the fp16 grid (weight_grid = 1), U_lo = 0 -> hi.hi + lo.hi only
    int64_t ntiles;
    uint32_t xbytes;       // a1: bytes of a tile's X block staged by cp.async.bulk (0: x(t) via L1)
    const double* rbeta;   // fused readout (Eq. 4): no H store; ryp[u * N + row] = H[row][u's neurons] . beta
    double* ryp;
    float k_sig, k_tanh;   // -log2(e) 2^-sigma, 2 log2(e) 2^-sigma
    float wb[kGWbMax];     // per neuron j, gate g in (z, r, f): [b, W_0..W_{S-1}] x 2^sigma
};


__device__ __forceinline__ void tmem_ld16g(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st8u(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]),
                 "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

// 16 fp32 values -> 8 words of fp16 hi pairs and 8 of lo pairs (A operand layout)
__device__ __forceinline__ void split16(const float (&h)[16], uint32_t (&hi)[8], uint32_t (&lo)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const __half2 a = __floats2half2_rn(h[2 * i], h[2 * i + 1]);
        const float2 af = __half22float2(a);
        const __half2 b = __floats2half2_rn(h[2 * i] - af.x, h[2 * i + 1] - af.y);
        hi[i] = *reinterpret_cast<const uint32_t*>(&a);
        lo[i] = *reinterpret_cast<const uint32_t*>(&b);
    }
}

template <int SS>
__global__ void __launch_bounds__(kGThreads, 1) k_gru_tc(const __grid_constant__ GruParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* stages = smem;
    float* zs = reinterpret_cast<float*>(stages + kGStages * kGStageBytes);   // [warp][item 32][lane]
    uint8_t* ximg = reinterpret_cast<uint8_t*>(zs) + kZBytes;                 // XMMA A operand (1 KB aligned)
    uint64_t* bars = reinterpret_cast<uint64_t*>(ximg + kGXImg);
    uint64_t* full = bars;
    uint64_t* empty = bars + kGStages;
    uint64_t* acc_full = bars + 2 * kGStages;
    uint64_t* acc_empty = acc_full + 2;
    uint64_t* a_ready = acc_empty + 2;   // [KS]: K-slice ks of h(t-1) is in TMEM
    uint64_t* rh_ready = a_ready + kGKS; // [KS]: K-slice ks of r o h(t-1) is in TMEM
    uint64_t* x_full = rh_ready + kGKS;  // the tile's X block has landed
    uint64_t* x_empty = x_full + 1;      // every epilogue warp has read its last x(t)
    uint64_t* xa_ready = x_empty + 1;    // XMMA: the A image holds [x(t), 1] of this step
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xa_ready + 1);
    float* xbuf = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);   // the tile's X block

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kGStages; ++i) {
            ptx::mbar_init(full + i, 1);
            ptx::mbar_init(empty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(acc_full + i, 1);
            ptx::mbar_init(acc_empty + i, kGEpiWarps);
        }
        for (int i = 0; i < kGKS; ++i) ptx::mbar_init(a_ready + i, kGEpiWarps);
        for (int i = 0; i < kGKS; ++i) ptx::mbar_init(rh_ready + i, kGEpiWarps);
        ptx::mbar_init(x_full, 1);
        ptx::mbar_init(x_empty, kGEpiWarps);
        ptx::mbar_init(xa_ready, 4);     // the 4 warps of neuron group u = 0 (one per lane quadrant)
        ptx::fence_mbar_init();
    }
    if (warp == kGProdWarp) {
        ptx::tmem_alloc(tmem_slot, 512);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int64_t steps_total = ((p.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x) * p.Q;

    if (warp == kGProdWarp) {
        uint32_t st = 0, ph = 0, xph = 0;
        const uint32_t bytes = p.two_pass ? kGSliceBytes : kGStageBytes;   // hi only when U_lo = 0
        for (int64_t s = 0; s < steps_total; ++s) {
            if (s % p.Q == 0) {   // a new tile: its X block (a1)
                const int64_t tile = blockIdx.x + (s / p.Q) * gridDim.x;
                if (ptx::xstage_tile(p.xbytes, tile, p.N))
                    ptx::xstage_issue(xbuf, p.X, p.ldx, tile, p.xbytes, x_full, x_empty, xph);
            }
            for (int c = 0; c < kGStagesPerStep; ++c) {
                ptx::mbar_wait(empty + st, ph ^ 1);
                if (ptx::elect_one()) {
                    const uint32_t cb = (kGX && c % kGSlices == kGKS) ? kGStageBytes : bytes;   // [W; b]: hi and lo
                    ptx::mbar_arrive_expect_tx(full + st, cb);
                    ptx::bulk_g2s(stages + st * kGStageBytes, p.Uimg + (size_t)c * kGStageBytes, cb, full + st);
                }
                __syncwarp();
                if (++st == kGStages) { st = 0; ph ^= 1; }
            }
        }
    } else if (warp == kGMmaWarp) {
        constexpr uint32_t idesc = ptx::idesc_f16(128, 128);
        const uint64_t dbase = ptx::desc_sw128_kmajor(ptx::smem_u32(stages));
        const bool two = p.two_pass != 0;
        uint32_t st = 0, ph = 0, ach = 0, aph = 0;
        for (int64_t s = 0; s < steps_total; ++s) {
            for (int q = 0; q < kGChunks; ++q) {
                ptx::mbar_wait(acc_empty + ach, aph ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + kAcc + ach * 128;
                const uint32_t abase = tmem + (q < 2 ? kAH : kARH);
                for (int ks = 0; ks < kGSlices; ++ks) {
                    if (q == 0 && ks < kGKS) {   // h(t-1) K-slice ks is in TMEM
                        ptx::mbar_wait(a_ready + ks, (uint32_t)(s & 1));
                        ptx::tc_fence_after();
                    }
                    if (q == 2 && ks < kGKS) {   // K-slice ks of r o h(t-1) is in TMEM
                        ptx::mbar_wait(rh_ready + ks, (uint32_t)(s & 1));
                        ptx::tc_fence_after();
                    }
                    if (kGX && q == 0 && ks == kGKS) {   // [x(t), 1] is in the A image
                        ptx::mbar_wait(xa_ready, (uint32_t)(s & 1));
                        ptx::tc_fence_after();
                    }
                    ptx::mbar_wait(full + st, ph);
                    ptx::tc_fence_after();
                    const uint64_t dbh = dbase + (uint64_t)((st * kGStageBytes) >> 4);
                    const uint64_t dbl = dbh + (uint64_t)(kGSliceBytes >> 4);
                    const uint32_t tah = abase + ks * 32, tal = abase + 64 + ks * 32;
                    if (kGX && ks == kGKS) {   // x(t) W + b: one k-step, A from shared memory, 3 passes
                        if (ptx::elect_one()) {
                            const uint64_t axh = ptx::desc_sw128_kmajor(ptx::smem_u32(ximg));
                            const uint64_t axl = axh + (uint64_t)(kGSliceBytes >> 4);
                            ptx::mma_f16_ss(d, axh, dbh, idesc, 1u);
                            ptx::mma_f16_ss(d, axl, dbh, idesc, 1u);
                            ptx::mma_f16_ss(d, axh, dbl, idesc, 1u);
                            ptx::mma_commit(empty + st);
                            ptx::mma_commit(acc_full + ach);
                        }
                        __syncwarp();
                        if (++st == kGStages) { st = 0; ph ^= 1; }
                        continue;
                    }
                    if (ptx::elect_one()) {
                        ptx::mma_f16_ts(d, tah, dbh, idesc, ks != 0);
                        if (!two) ptx::mma_f16_ts(d, tah, dbl, idesc, 1);
                        ptx::mma_f16_ts(d, tal, dbh, idesc, 1);
#pragma unroll
                        for (int kk = 1; kk < 4; ++kk) {
                            ptx::mma_f16_ts(d, tah + kk * 8, dbh + 2 * kk, idesc, 1);
                            if (!two) ptx::mma_f16_ts(d, tah + kk * 8, dbl + 2 * kk, idesc, 1);
                            ptx::mma_f16_ts(d, tal + kk * 8, dbh + 2 * kk, idesc, 1);
                        }
                        ptx::mma_commit(empty + st);
                        if (ks == kGSlices - 1) ptx::mma_commit(acc_full + ach);
                    }
                    __syncwarp();
                    if (++st == kGStages) { st = 0; ph ^= 1; }
                }
                if (++ach == 2) { ach = 0; aph ^= 1; }
            }
        }
    } else {
        // ---------------- epilogue
        const int q4 = warp & 3, u = warp >> 2;
        const int r = 32 * q4 + lane;
        const uint32_t lb = tmem + ((uint32_t)(32 * q4) << 16);
        const float kS = p.k_sig, kT = p.k_tanh;
        float* my_z = zs + (size_t)warp * 32 * 32 + lane;      // [item][lane]
        float h[32];                                            // h of neurons 16u+i, 64+16u+i
        uint32_t ach = 0, aph = 0, xph = 0;
        // write h (or zero) of this thread's neurons into A_h hi/lo and publish both K-slices
        // K-slice `half` of this thread's h (or zeros) into A_h, then release it
        auto publish_h = [&](int half, bool zero) {
            float v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = zero ? 0.0f : h[half * 16 + i];
            uint32_t hi[8], lo[8];
            split16(v, hi, lo);
            const uint32_t col = (64 * half + 16 * u) / 2;   // two fp16 per column
            tmem_st8u(lb + kAH + col, hi);
            tmem_st8u(lb + kAH + 64 + col, lo);
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(a_ready + half);
        };
#pragma unroll
        for (int i = 0; i < 32; ++i) h[i] = 0.0f;
        publish_h(0, true);
        publish_h(1, true);
        for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            const int64_t row = tile * kGRows + r;
            const bool valid = row < p.N;
            const bool xst = ptx::xstage_tile(p.xbytes, tile, p.N);
            const float* xrow = xst ? xbuf + (int64_t)r * p.ldx : p.X + (valid ? row : 0) * p.ldx;
            if (xst) {
                ptx::mbar_wait(x_full, xph);
                xph ^= 1;
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) h[i] = 0.0f;
            double yacc = 0.0;   // fused readout partial
            // XMMA: write [x(tn), 1, 0..] of this thread's row as fp16 hi|lo into the A image
            // (neuron group u = 0 only) and release it to the MMA warp
            auto put_x = [&](int tn) {
                if (u == 0) {
                    float xv[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k) xv[k] = 0.0f;
#pragma unroll
                    for (int s = 0; s < SS; ++s)
                        xv[s] = (valid && s < p.S)
                                    ? (xst ? xrow[(tn - 1) * p.S + s] : __ldg(xrow + (int64_t)(tn - 1) * p.S + s))
                                    : 0.0f;
                    xv[p.S] = 1.0f;   // the bias column
                    uint32_t hi[8], lo[8];
                    split16(xv, hi, lo);
                    uint8_t* xh = ximg;
                    uint8_t* xl = ximg + kGSliceBytes;
                    *reinterpret_cast<uint4*>(xh + ptx::sw128_offset((uint32_t)r, 0)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                    *reinterpret_cast<uint4*>(xh + ptx::sw128_offset((uint32_t)r, 8)) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
                    *reinterpret_cast<uint4*>(xl + ptx::sw128_offset((uint32_t)r, 0)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
                    *reinterpret_cast<uint4*>(xl + ptx::sw128_offset((uint32_t)r, 8)) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(xa_ready);
                }
                if (xst && tn == p.Q) {   // last x(t) of this tile read: the block may be replaced
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(x_empty);
                }
            };
            if (kGX) put_x(1);
            for (int t = 1; t <= p.Q; ++t) {
                float xs[SS];
#pragma unroll
                for (int s = 0; s < SS; ++s)
                    xs[s] = (!kGX && valid && s < p.S)
                                ? (xst ? xrow[(t - 1) * p.S + s] : __ldg(xrow + (int64_t)(t - 1) * p.S + s))
                                : 0.0f;
                if (!kGX && xst && t == p.Q) {   // last x(t) of this tile read: the block may be replaced
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(x_empty);
                }
                // ---- phase 1: z, r for neurons 64c + 16u + i; r o h -> A_rh
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    ptx::mbar_wait(acc_full + ach, aph);
                    ptx::tc_fence_after();
                    float a[2][16];   // 16 neurons x (z, r) interleaved
                    tmem_ld16g(lb + kAcc + ach * 128 + 32 * u, a[0]);
                    tmem_ld16g(lb + kAcc + ach * 128 + 32 * u + 16, a[1]);
                    ptx::tmem_wait_ld();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(acc_empty + ach);
                    if (++ach == 2) { ach = 0; aph ^= 1; }
                    float rh[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const int j = 64 * c + 16 * u + i;
                        const float* w = p.wb + j * (3 * (SS + 1));
                        // exp2 arguments k_g pre-activation; k_g folded into W|b on the host
                        // (XMMA: x W + b is already in the accumulator)
                        float pz = kGX ? kS * a[i >> 3][(i & 7) * 2] : fmaf(kS, a[i >> 3][(i & 7) * 2], w[0]);
                        float pr = kGX ? kS * a[i >> 3][(i & 7) * 2 + 1] : fmaf(kS, a[i >> 3][(i & 7) * 2 + 1], w[SS + 1]);
                        if (!kGX) {
#pragma unroll
                            for (int s = 0; s < SS; ++s) {
                                pz = fmaf(xs[s], w[1 + s], pz);
                                pr = fmaf(xs[s], w[SS + 2 + s], pr);
                            }
                        }
                        my_z[(c * 16 + i) * 32] = sig_e2(pz);         // z (accurate form, DESIGN R26)
                        rh[i] = sig_e2(pr) * h[c * 16 + i];           // r o h(t-1)
                    }
                    uint32_t hi[8], lo[8];
                    split16(rh, hi, lo);
                    const uint32_t col = (64 * c + 16 * u) / 2;
                    tmem_st8u(lb + kARH + col, hi);
                    tmem_st8u(lb + kARH + 64 + col, lo);
                    ptx::tmem_wait_st();   // K-slice c of r o h is complete: phase 2 may start on it
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(rh_ready + c);
                }
                // ---- phase 2: n = tanh(.), h <- (1 - z) h + z n
                ptx::mbar_wait(acc_full + ach, aph);
                ptx::tc_fence_after();
                float a2[2][16];
                tmem_ld16g(lb + kAcc + ach * 128 + 16 * u, a2[0]);
                tmem_ld16g(lb + kAcc + ach * 128 + 64 + 16 * u, a2[1]);
                ptx::tmem_wait_ld();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(acc_empty + ach);
                if (++ach == 2) { ach = 0; aph ^= 1; }
                // this step's MMAs are complete (phase 2 was the last): the A image may take x(t+1)
                if (kGX && t < p.Q) put_x(t + 1);
#pragma unroll
                for (int c = 0; c < 2; ++c) {   // c = K-slice of the next step's A
#pragma unroll
                    for (int i = 0; i < 16; i += 2) {
                        float dn[2];
#pragma unroll
                        for (int k2 = 0; k2 < 2; ++k2) {
                            const int j = 64 * c + 16 * u + i + k2;
                            const float* w = p.wb + j * (3 * (SS + 1)) + 2 * (SS + 1);
                            float pn = kGX ? kT * a2[c][i + k2] : fmaf(kT, a2[c][i + k2], w[0]);
                            if (!kGX) {
#pragma unroll
                                for (int s = 0; s < SS; ++s) pn = fmaf(xs[s], w[1 + s], pn);
                            }
                            dn[k2] = tanh_e2_sig(pn);
                        }
                        const float n0 = dn[0], n1 = dn[1];
                        const float z0 = my_z[(c * 16 + i) * 32], z1 = my_z[(c * 16 + i + 1) * 32];
                        float& h0 = h[c * 16 + i];
                        float& h1 = h[c * 16 + i + 1];
                        h0 = fmaf(z0, n0 - h0, h0);   // (1 - z) h + z n
                        h1 = fmaf(z1, n1 - h1, h1);
                    }
                    if (t == p.Q && valid && p.rbeta) {
                        const double* bj = p.rbeta + 64 * c + 16 * u;
#pragma unroll
                        for (int i = 0; i < 16; ++i) yacc = fma((double)h[c * 16 + i], __ldg(bj + i), yacc);
                    } else if (t == p.Q && valid) {
                        float* d1 = p.H + row * p.ldh + 64 * c + 16 * u;
                        if (((p.ldh | (int64_t)(reinterpret_cast<uintptr_t>(p.H) >> 2)) & 3) == 0) {
                            float4* dst = reinterpret_cast<float4*>(d1);
#pragma unroll
                            for (int i = 0; i < 4; ++i)
                                dst[i] = make_float4(h[c * 16 + 4 * i], h[c * 16 + 4 * i + 1], h[c * 16 + 4 * i + 2],
                                                     h[c * 16 + 4 * i + 3]);
                        } else {
#pragma unroll
                            for (int i = 0; i < 16; ++i) d1[i] = h[c * 16 + i];
                        }
                    }
                    publish_h(c, t == p.Q);   // next step's A slice c (or h(0) = 0 of the next tile)
                }
            }
            if (p.rbeta && valid) p.ryp[u * p.N + row] = yacc;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kGProdWarp) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

// U images: chunk 0/1 rows nrow = jj*2 + g (neuron 64c + jj, gate z|r), chunk 2
// rows = neuron j (gate f); K-major SW128, hi | lo, scaled by 2^sigma.
__global__ void k_pack_u_gru(const float* __restrict__ U, float scale, uint8_t* __restrict__ img) {
    const int64_t total = (int64_t)kGChunks * kGKS * 128 * 64;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int kk = (int)(e % 64);
        const int nrow = (int)((e / 64) % 128);
        const int ks = (int)((e / (64 * 128)) % kGKS);
        const int q = (int)(e / ((int64_t)64 * 128 * kGKS));
        int col;
        if (q < 2) col = (nrow & 1) * kGM + 64 * q + (nrow >> 1);
        else col = 2 * kGM + nrow;
        const float v = U[(size_t)(64 * ks + kk) * (3 * kGM) + col] * scale;
        const __half hi = __float2half_rn(v);
        const __half lo = __float2half_rn(v - __half2float(hi));
        uint8_t* base = img + (size_t)((q * kGSlices + ks) * 2) * kGSliceBytes;   // kGSlices per chunk (XMMA: + [W; b])
        const uint32_t off = ptx::sw128_offset(nrow, kk);
        *reinterpret_cast<__half*>(base + off) = hi;
        *reinterpret_cast<__half*>(base + kGSliceBytes + off) = lo;
    }
}

int gru_padded_s(int S) { return S <= 1 ? 1 : (S <= 2 ? 2 : 4); }

template <int SS>
cudaError_t launch_gru(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    static GruParams p;
    p.X = X; p.ldx = ldx; p.N = N; p.H = H; p.ldh = ldh;
    p.Uimg = static_cast<const uint8_t*>(h->tc_ops);
    p.S = h->S; p.Q = h->Q;
    p.two_pass = h->weight_grid == 1;
    p.ntiles = (N + kGRows - 1) / kGRows;
    p.xbytes = ptx::xstage_host(X, ldx, kGSmem);   // a1: stage each full tile's X block when it fits
    p.rbeta = h->ro_beta; p.ryp = h->ro_yp;
    h->ro_slots = 4;
    const int smem = kGSmem + (int)p.xbytes;
    p.k_sig = -1.4426950408889634f * h->tc_inv_scale;
    p.k_tanh = 2.8853900817779268f * h->tc_inv_scale;
    std::copy(h->tc_wb.begin(), h->tc_wb.end(), p.wb);
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_gru_tc<SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    const int grid = (int)std::min<int64_t>(p.ntiles, h->sm_count);
    k_gru_tc<SS><<<grid, kGThreads, smem, h->stream>>>(p);
    h->launches++;
    return cudaGetLastError();
}

}  // namespace

bool gru_tc_supported(const elmrnn* h) {
    return h->arch == kArchGRU && h->M == kGM && h->S <= 4 &&
           (size_t)(gru_padded_s(h->S) + 1) * 3 * kGM <= (size_t)kGWbMax;
}

cudaError_t gru_tc_prepare(elmrnn* h) {
    cudaError_t e;
    const size_t bytes = (size_t)kGStagesPerStep * kGStageBytes;
    if ((e = cudaMalloc(&h->tc_ops, bytes))) return e;
    if ((e = cudaMemsetAsync(h->tc_ops, 0, bytes, h->stream))) return e;
    h->tc_ops_bytes = bytes;
    const int sigma = h->rec_scale == 1 ? 0 : (int)std::floor(std::log2(std::sqrt((double)kGM)));
    const float scale = std::ldexp(1.0f, sigma);
    h->tc_inv_scale = std::ldexp(1.0f, -sigma);
    const int GM = 3 * kGM, S = h->S, SP = gru_padded_s(S);
    std::vector<float> W((size_t)S * GM), b(GM);
    if ((e = cudaMemcpyAsync(W.data(), h->W, sizeof(float) * S * GM, cudaMemcpyDeviceToHost, h->stream))) return e;
    if ((e = cudaMemcpyAsync(b.data(), h->b, sizeof(float) * GM, cudaMemcpyDeviceToHost, h->stream))) return e;
    if ((e = cudaStreamSynchronize(h->stream))) return e;
    h->tc_wb.assign((size_t)kGM * 3 * (SP + 1), 0.0f);
    // x k_g: -log2(e) for the sigmoid gates z, r; 2 log2(e) for the tanh candidate f
    for (int j = 0; j < kGM; ++j)
        for (int g = 0; g < 3; ++g) {
            const double kg = g == 2 ? 2.8853900817779268 : -1.4426950408889634;
            float* d = h->tc_wb.data() + ((size_t)j * 3 + g) * (SP + 1);
            d[0] = (float)(kg * b[g * kGM + j]);
            for (int s2 = 0; s2 < S; ++s2) d[1 + s2] = (float)(kg * W[(size_t)s2 * GM + g * kGM + j]);
        }
    const int64_t total = (int64_t)kGChunks * kGKS * 128 * 64;
    k_pack_u_gru<<<(int)std::min<int64_t>((total + 255) / 256, 4096), 256, 0, h->stream>>>(
        h->rec, scale, static_cast<uint8_t*>(h->tc_ops));
    h->launches++;
    if ((e = cudaGetLastError())) return e;
    if (kGX) {   // XMMA B slices: [W; b] x 2^sigma of each chunk's gate rows, K = s (W_s), K = S (b)
        std::vector<uint8_t> xs((size_t)kGChunks * kGStageBytes, 0);
        for (int q = 0; q < kGChunks; ++q)
            for (int nrow = 0; nrow < 128; ++nrow) {
                const int g = q < 2 ? (nrow & 1) : 2, j = q < 2 ? 64 * q + (nrow >> 1) : nrow;
                for (int k = 0; k <= S; ++k) {
                    const float v = (k < S ? W[(size_t)k * GM + g * kGM + j] : b[g * kGM + j]) * scale;
                    const __half hi = __float2half_rn(v);
                    const __half lo = __float2half_rn(v - __half2float(hi));
                    uint8_t* base = xs.data() + (size_t)q * kGStageBytes;
                    const uint32_t off = ptx::sw128_offset((uint32_t)nrow, (uint32_t)k);
                    *reinterpret_cast<__half*>(base + off) = hi;
                    *reinterpret_cast<__half*>(base + kGSliceBytes + off) = lo;
                }
            }
        for (int q = 0; q < kGChunks; ++q)
            if ((e = cudaMemcpyAsync(static_cast<uint8_t*>(h->tc_ops) + ((size_t)q * kGSlices + kGKS) * kGStageBytes,
                                     xs.data() + (size_t)q * kGStageBytes, kGStageBytes, cudaMemcpyHostToDevice,
                                     h->stream)))
                return e;
        if ((e = cudaStreamSynchronize(h->stream))) return e;
    }
    return cudaSuccess;
}

cudaError_t launch_gru_tc(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    switch (gru_padded_s(h->S)) {
    case 1: return launch_gru<1>(h, X, ldx, N, H, ldh);
    case 2: return launch_gru<2>(h, X, ldx, N, H, ldh);
    default: return launch_gru<4>(h, X, ldx, N, H, ldh);
    }
}

}  // namespace elm
