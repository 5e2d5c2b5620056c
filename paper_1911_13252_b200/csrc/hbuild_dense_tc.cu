// hbuild_dense_tc.cu -- tcgen05 tensor-core H builder for the LSTM (S2.2.5,
// P:128-142, dense U, reading R10) at large M: the per-step contraction
//   a(t) = h(t-1) [128 x M] . U_cat [M x 4M]   (gates o, c, lambda, in)
// runs on the 5th-generation tensor cores with fp32-accurate operands, the
// x(t) W + b term and the gate epilogue run on the CUDA cores, and the state
// never leaves the SM for all Q steps.
//
// Precision: a single fp16 (or tf32) pass fails the
// 1e-5 H tolerance.  Every operand is split x = hi + lo with hi = fp16(x),
// lo = fp16(x - hi), and three kind::f16 MMAs accumulate hi.hi + hi.lo + lo.hi
// into ONE fp32 TMEM accumulator (the lo.lo term is below fp32 resolution).
// U is pre-scaled by 2^sigma (exact) so its lo part stays out of fp16
// subnormals; the epilogue multiplies the accumulator by 2^-sigma.
//
// CTA = one persistent tile worker (148 CTAs), 128 sample rows = 128 TMEM lanes.
//   smem: A = h(t-1) hi/lo, K-major SW128 (128 KB at M = 256)
//         B ring: 3 stages x (hi + lo) 128 x 64 fp16 U slices (32 KB each)
//   TMEM: 2 x 128 accumulator columns (double buffered) + M columns of h(t)
//   warps: 0..15 = epilogue (4 per TMEM lane quadrant; a thread owns one row
//          and 8 neurons per chunk and keeps c(t) for its M/4 neurons in
//          registers), 16 = bulk-copy producer (one thread) + TMEM allocator,
//          17 = MMA issuer (one thread; the highest warp id has issue priority).
//   per step: NCH = M/32 chunks of 32 neurons x 4 gates = 128 accumulator
//   columns; chunk n+1's MMAs overlap chunk n's epilogue.  After the last
//   chunk the epilogue converts h(t) (TMEM) to fp16 hi/lo into A and
//   releases the next step's MMAs; after step Q it stores H(Q) rows.
//   W and b (x W + b on FFMA) are kernel parameters: warp-uniform constant
//   bank reads.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace elm {

namespace {

constexpr int kTcRows = 128;
#ifndef ELM_TC256_STAGES
#define ELM_TC256_STAGES 3
#endif
#ifndef ELM_TC_XMMA
#define ELM_TC_XMMA 1
#endif
#ifndef ELM_TC_HOLD
#define ELM_TC_HOLD 1   // hold the last K-slice of h(t) in registers (0: stage it like the others)
#endif
constexpr int kTcSliceBytes = 128 * 64 * 2;      // one 128 x 64 fp16 SW128 tile
constexpr int kTcStageBytes = 2 * kTcSliceBytes;  // hi + lo
constexpr int kTcEpiWarps = 16;                 // 4 per TMEM lane quadrant, 8 neurons per chunk each
constexpr int kTcCtlWarps = 2;                  // 16: bulk-copy producer + TMEM alloc, 17: MMA issuer
constexpr int kTcProdWarp = kTcEpiWarps, kTcMmaWarp = kTcEpiWarps + 1;
constexpr int kTcThreads = (kTcCtlWarps + kTcEpiWarps) * 32;
constexpr int kTcWbMax = 7168;                    // floats of W|b in the parameter block

struct TcParams {
    const float* X;
    int64_t ldx, N;
    float* H;
    int64_t ldh;
    const uint8_t* Uimg;   // [NCH][KS][hi|lo][16 KB] pre-swizzled images
    int S, Q;
    int two_pass;          // 1: U on the fp16 grid (weight_grid = 1), U_lo = 0 -> hi.hi + lo.hi only
    int debug_no_u;        // ELMRNN_DEBUG_NO_U: skip U streaming after step 0 (timing experiment only)
    int64_t ntiles;
    uint32_t xbytes;       // a1: bytes of a tile's X block staged by cp.async.bulk (0: x(t) via L1)
    const double* rbeta;   // fused readout (Eq. 4): no H store; ryp[u * N + row] = H[row][u's neurons] . beta
    double* ryp;
    float k_sig, k_tanh;   // -log2(e) 2^-sigma, 2 log2(e) 2^-sigma
    unsigned long long* trace;   // optional event trace of CTA 0 (ELMRNN_TRACE), else null
    int trace_cap;
    float wb[kTcWbMax];    // per neuron j, gate g: [b, W_0..W_{S-1}] x 2^sigma
};

template <int M>
struct TcCfg {
    static constexpr int STAGES = M == 256 ? ELM_TC256_STAGES : 3;   // U ring depth
    static constexpr int NCH = M / 32;
    static constexpr int KS = M / 64;
    // XM (M = 128): x(t) W + b as one more K-step per chunk (as the GRU builder): A = [x, 1]
    // fp16 hi|lo SW128 image in shared memory, B = [W; b] an extra streamed slice.  At
    // M = 128 the epilogue paces the kernel (MMA per chunk ~1.5k cycles); at M = 256 the
    // MMAs do, and the extra K-step would cost more than the epilogue saves.
    static constexpr int XM = (M == 128 && ELM_TC_XMMA) ? 1 : 0;
    static constexpr int SLICES = KS + XM;                 // streamed B slices per chunk
    static constexpr int XIMG = XM * kTcStageBytes;        // the [x, 1] image, hi | lo
    // staged words per epilogue thread: h(t) hi|lo of chunks 0 .. NCH-3.  The last
    // K-slice bypasses the staging area (chunk NCH-2 waits in 8 registers for the
    // last chunk's MMAs to finish, chunk NCH-1 goes straight into TMEM), which
    // leaves room for the tile's X block next to a 3-stage U ring at M = 256
    static constexpr int HOLD = ELM_TC_HOLD ? 2 : 0;   // chunks held in registers
    static constexpr int ITEMS = (NCH - HOLD) * 8;
    static constexpr int STG_BYTES = kTcEpiWarps * ITEMS * 32 * 4;
    static constexpr int SMEM = 1024 + STAGES * kTcStageBytes + XIMG + STG_BYTES + 256;   // + the X block
    static constexpr int TMEM_COLS = 512;
    static constexpr int A_HI = 256;                       // TMEM columns of A = h(t-1): hi parts
    static constexpr int A_LO = 256 + M / 2;               //   lo parts (2 fp16 per 32-bit column)
};

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// Split 8 fp32 h values into fp16 hi = fp16(h) and lo = fp16(h - hi), packed
// two per 32-bit word (even K index in the low half) as the TMEM A operand wants.
__device__ __forceinline__ void split_h8(const float (&h)[8], uint32_t (&hi)[4], uint32_t (&lo)[4]) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const __half2 a = __floats2half2_rn(h[2 * i], h[2 * i + 1]);   // packed F2FP
        const float2 af = __half22float2(a);
        const __half2 b = __floats2half2_rn(h[2 * i] - af.x, h[2 * i + 1] - af.y);
        hi[i] = *reinterpret_cast<const uint32_t*>(&a);
        lo[i] = *reinterpret_cast<const uint32_t*>(&b);
    }
}

// Event trace (tracing aux subsystem): CTA 0 records (kind, step, chunk, clock)
// for its first trace_cap events when the launcher passes a buffer.
__device__ __forceinline__ void trace_ev(const TcParams& p, uint32_t* cnt, int kind, int step, int chunk) {
    if (p.trace == nullptr || blockIdx.x != 0) return;
    const uint32_t i = atomicAdd(cnt, 1u);
    if ((int)i < p.trace_cap)
        p.trace[i] = ((unsigned long long)kind << 56) | ((unsigned long long)(step & 0xFFFF) << 40) |
                     ((unsigned long long)(chunk & 0xFF) << 32) | (unsigned long long)(clock64() & 0xFFFFFFFFull);
}

template <int M, int SS>
__global__ void __launch_bounds__(kTcThreads, 1) k_lstm_tc(const __grid_constant__ TcParams p) {
    using C = TcCfg<M>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int kTcStages = C::STAGES;
    uint8_t* stages = smem;                                                     // U ring
    uint8_t* ximg = stages + kTcStages * kTcStageBytes;                              // XM: [x, 1] image (1 KB aligned)
    uint32_t* stg = reinterpret_cast<uint32_t*>(ximg + C::XIMG);                     // h(t) hi|lo staging
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stg) + C::STG_BYTES);
    float* xbuf = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bars) + 256);   // the tile's X block
    uint64_t* full = bars;                       // [kTcStages]
    uint64_t* empty = bars + kTcStages;          // [kTcStages]
    uint64_t* acc_full = bars + 2 * kTcStages;   // [2]
    uint64_t* acc_empty = acc_full + 2;          // [2]
    uint64_t* a_ready = acc_empty + 2;           // [KS]: K-slice ks of A = h(t-1) is in TMEM
    uint64_t* a_free = a_ready + C::KS;          // [KS]: the last chunk's MMAs no longer read A slice ks
    uint64_t* x_full = a_free + C::KS;           // the tile's X block has landed
    uint64_t* x_empty = x_full + 1;              // every epilogue warp has read its last x(t)
    uint64_t* xa_ready = x_empty + 1;            // XM: the [x, 1] image holds this step's x(t)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xa_ready + 1);
    uint32_t* trace_cnt = tmem_slot + 1;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kTcStages; ++i) {
            ptx::mbar_init(full + i, 1);
            ptx::mbar_init(empty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            ptx::mbar_init(acc_full + i, 1);
            ptx::mbar_init(acc_empty + i, kTcEpiWarps);
        }
        for (int i = 0; i < C::KS; ++i) ptx::mbar_init(a_ready + i, kTcEpiWarps);
        for (int i = 0; i < C::KS; ++i) ptx::mbar_init(a_free + i, 1);
        ptx::mbar_init(x_full, 1);
        ptx::mbar_init(x_empty, kTcEpiWarps);
        ptx::mbar_init(xa_ready, 4);   // the 4 warps of neuron group u = 0
        *trace_cnt = 0;
        ptx::fence_mbar_init();
    }
    if (warp == kTcProdWarp) {
        ptx::tmem_alloc(tmem_slot, C::TMEM_COLS);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int64_t steps_total = ((p.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x) * p.Q;

    if (warp == kTcProdWarp) {
        // ---------------- producer: stream U slices (chunk, K-slice) from L2.
        // The whole warp runs the loop (warp-uniform state lives in uniform
        // registers); one elected lane issues.
        uint32_t st = 0, ph = 0, xph = 0;
        const uint32_t bytes = p.two_pass ? kTcSliceBytes : kTcStageBytes;   // hi only when U_lo = 0
        for (int64_t s = 0; s < steps_total; ++s) {
            if (s % p.Q == 0) {   // a new tile: its X block (a1)
                const int64_t tile = blockIdx.x + (s / p.Q) * gridDim.x;
                if (ptx::xstage_tile(p.xbytes, tile, p.N))
                    ptx::xstage_issue(xbuf, p.X, p.ldx, tile, p.xbytes, x_full, x_empty, xph);
            }
            for (int c = 0; c < C::NCH * C::SLICES; ++c) {
                ptx::mbar_wait(empty + st, ph ^ 1);
                if (ptx::elect_one()) {
                    // XM's [W; b] slice: hi and lo always (W, b are not on the fp16 grid)
                    const uint32_t cb = (C::XM && c % C::SLICES == C::KS) ? (uint32_t)kTcStageBytes : bytes;
                    if (p.debug_no_u && s > 0) {   // timing experiment only (results invalid)
                        ptx::mbar_arrive(full + st);
                    } else {
                        ptx::mbar_arrive_expect_tx(full + st, cb);
                        ptx::bulk_g2s(stages + st * kTcStageBytes, p.Uimg + (size_t)c * kTcStageBytes, cb,
                                      full + st);
                    }
                }
                __syncwarp();
                if (++st == kTcStages) { st = 0; ph ^= 1; }
            }
        }
    } else if (warp == kTcMmaWarp) {
        // ---------------- MMA issuer (highest warp id = highest issue priority
        // on its SM sub-partition).  Warp-uniform loop, one elected lane issues
        // the 12 MMAs of a K-slice; descriptors and TMEM addresses advance by
        // plain adds (the SW128 start field is in 16-byte units).
        constexpr uint32_t idesc = ptx::idesc_f16(128, 128);
        const uint32_t a_hi = tmem + C::A_HI, a_lo = tmem + C::A_LO;   // A operand in TMEM
        const uint64_t dbase = ptx::desc_sw128_kmajor(ptx::smem_u32(stages));
        const bool two = p.two_pass != 0;
        uint32_t st = 0, ph = 0, ach = 0, aph = 0;
        for (int64_t s = 0; s < steps_total; ++s) {
            if (lane == 0) trace_ev(p, trace_cnt, 1, (int)s, 0);
            for (int n = 0; n < C::NCH; ++n) {
                ptx::mbar_wait(acc_empty + ach, aph ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + ach * 128;
                for (int ks = 0; ks < C::KS; ++ks) {
                    if (n == 0) {   // first chunk of a step: K-slice ks of h(t-1) must be in TMEM
                        ptx::mbar_wait(a_ready + ks, (uint32_t)(s & 1));
                        ptx::tc_fence_after();
                    }
                    ptx::mbar_wait(full + st, ph);
                    ptx::tc_fence_after();
                    const uint64_t dbh = dbase + (uint64_t)((st * kTcStageBytes) >> 4);
                    const uint64_t dbl = dbh + (uint64_t)(kTcSliceBytes >> 4);
                    const uint32_t tah = a_hi + ks * 32, tal = a_lo + ks * 32;
                    if (ptx::elect_one()) {
                        // passes ordered so the two MMAs reading the same B_hi tile are adjacent
                        ptx::mma_f16_ts(d, tah, dbh, idesc, ks != 0);
                        ptx::mma_f16_ts(d, tal, dbh, idesc, 1);
                        if (!two) ptx::mma_f16_ts(d, tah, dbl, idesc, 1);
#pragma unroll
                        for (int kk = 1; kk < 4; ++kk) {
                            ptx::mma_f16_ts(d, tah + kk * 8, dbh + 2 * kk, idesc, 1);
                            ptx::mma_f16_ts(d, tal + kk * 8, dbh + 2 * kk, idesc, 1);
                            if (!two) ptx::mma_f16_ts(d, tah + kk * 8, dbl + 2 * kk, idesc, 1);
                        }
                        ptx::mma_commit(empty + st);                  // frees the U stage
                        // last chunk of the step: A slice ks is free for h(t) once these MMAs retire
                        if (n == C::NCH - 1 && ks < C::KS - 1) ptx::mma_commit(a_free + ks);
                        if (!C::XM && ks == C::KS - 1) ptx::mma_commit(acc_full + ach);   // chunk accumulator ready
                    }
                    __syncwarp();
                    if (++st == kTcStages) { st = 0; ph ^= 1; }
                }
                if constexpr (C::XM != 0) {   // x(t) W + b: one k-step, A = [x, 1] from shared memory
                    if (n == 0) {
                        ptx::mbar_wait(xa_ready, (uint32_t)(s & 1));
                        ptx::tc_fence_after();
                    }
                    ptx::mbar_wait(full + st, ph);
                    ptx::tc_fence_after();
                    const uint64_t dbh = dbase + (uint64_t)((st * kTcStageBytes) >> 4);
                    const uint64_t dbl = dbh + (uint64_t)(kTcSliceBytes >> 4);
                    if (ptx::elect_one()) {
                        const uint64_t axh = ptx::desc_sw128_kmajor(ptx::smem_u32(ximg));
                        const uint64_t axl = axh + (uint64_t)(kTcSliceBytes >> 4);
                        ptx::mma_f16_ss(d, axh, dbh, idesc, 1u);
                        ptx::mma_f16_ss(d, axl, dbh, idesc, 1u);
                        ptx::mma_f16_ss(d, axh, dbl, idesc, 1u);
                        ptx::mma_commit(empty + st);
                        ptx::mma_commit(acc_full + ach);
                    }
                    __syncwarp();
                    if (++st == kTcStages) { st = 0; ph ^= 1; }
                }
                if (lane == 0) trace_ev(p, trace_cnt, 3, (int)s, n);
                if (++ach == 2) { ach = 0; aph ^= 1; }
            }
        }
    } else {
        // ---------------- epilogue: gates, c/h update, A write-back, H(Q) store
        // Pre-activations stay in the 2^sigma-scaled domain: W, b were scaled on
        // the host, and 2^-sigma is folded into the exp2 argument constants.
        // epilogue warp w: TMEM lane quadrant w % 4 (hardware rule), neuron group u
        const int e = warp, q = warp & 3, u = e >> 2;
        const int r = 32 * q + lane;                 // tile row = TMEM lane
        const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
        const float kS = p.k_sig, kT = p.k_tanh;     // -log2e 2^-sigma, 2 log2e 2^-sigma
        float c[C::NCH * 8];                         // c(t) of neurons n*32 + 8u + 0..7
        uint32_t ach = 0, aph = 0, afph = 0, xph = 0;
        uint32_t* my_stg = stg + (size_t)e * C::ITEMS * 32 + lane;   // [item][lane]
        uint32_t hold[8];                                             // h(t) hi|lo of chunk NCH-2
        {   // h(0) = 0 for the first tile
            const uint32_t z[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int n = 0; n < C::NCH; ++n) {
                ptx::tmem_st4(lane_base + C::A_HI + n * 16 + 4 * u, z);
                ptx::tmem_st4(lane_base + C::A_LO + n * 16 + 4 * u, z);
            }
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0)
                for (int ks = 0; ks < C::KS; ++ks) ptx::mbar_arrive(a_ready + ks);
        }
        // Publish K-slices [k0, k1) of h(t) (staged fp16 hi|lo words) into the
        // TMEM A operand -- or zeros, h(0) of the next tile, after the last step.
        auto publish = [&](int k0, int k1, bool zero) {
#pragma unroll
            for (int n = 0; n < C::NCH; ++n) {
                if (n < 2 * k0 || n >= 2 * k1) continue;
                uint32_t hi[4], lo[4];
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    hi[w] = zero ? 0u : my_stg[(n * 8 + w) * 32];
                    lo[w] = zero ? 0u : my_stg[(n * 8 + 4 + w) * 32];
                }
                ptx::tmem_st4(lane_base + C::A_HI + n * 16 + 4 * u, hi);
                ptx::tmem_st4(lane_base + C::A_LO + n * 16 + 4 * u, lo);
            }
            ptx::tmem_wait_st();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0)
                for (int ks = k0; ks < k1; ++ks) ptx::mbar_arrive(a_ready + ks);
        };
        for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            const int64_t row = tile * kTcRows + r;
            const bool valid = row < p.N;
            const bool xst = ptx::xstage_tile(p.xbytes, tile, p.N);
            const float* xrow = xst ? xbuf + (int64_t)r * p.ldx : p.X + (valid ? row : 0) * p.ldx;
            if (xst) {
                ptx::mbar_wait(x_full, xph);
                xph ^= 1;
            }
            // XM: write [x(tn), 1, 0..] of this row (fp16 hi|lo) into the A image (group u = 0)
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
#pragma unroll
                    for (int q8 = 0; q8 < 2; ++q8) {
                        float h8[8];
#pragma unroll
                        for (int i = 0; i < 8; ++i) h8[i] = xv[8 * q8 + i];
                        uint32_t h4[4], l4[4];
                        split_h8(h8, h4, l4);
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            hi[4 * q8 + i] = h4[i];
                            lo[4 * q8 + i] = l4[i];
                        }
                    }
                    *reinterpret_cast<uint4*>(ximg + ptx::sw128_offset((uint32_t)r, 0)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                    *reinterpret_cast<uint4*>(ximg + ptx::sw128_offset((uint32_t)r, 8)) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
                    *reinterpret_cast<uint4*>(ximg + kTcSliceBytes + ptx::sw128_offset((uint32_t)r, 0)) =
                        make_uint4(lo[0], lo[1], lo[2], lo[3]);
                    *reinterpret_cast<uint4*>(ximg + kTcSliceBytes + ptx::sw128_offset((uint32_t)r, 8)) =
                        make_uint4(lo[4], lo[5], lo[6], lo[7]);
                    ptx::fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(xa_ready);
                }
                if (xst && tn == p.Q) {   // last x(t) of this tile read: the block may be replaced
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(x_empty);
                }
            };
            if constexpr (C::XM != 0) put_x(1);
#pragma unroll
            for (int i = 0; i < C::NCH * 8; ++i) c[i] = 0.0f;
            double yacc = 0.0;   // fused readout partial
            for (int t = 1; t <= p.Q; ++t) {
                float xs[SS];
#pragma unroll
                for (int s = 0; s < SS; ++s)
                    xs[s] = (!C::XM && valid && s < p.S)
                                ? (xst ? xrow[(t - 1) * p.S + s] : __ldg(xrow + (int64_t)(t - 1) * p.S + s))
                                : 0.0f;
                if (!C::XM && xst && t == p.Q) {   // last x(t) of this tile read: the block may be replaced
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(x_empty);
                }
#pragma unroll
                for (int n = 0; n < C::NCH; ++n) {
                    if (n == C::NCH - 1) {
                        // h(t) slices 0..KS-2 (chunks 0..NCH-3) are staged: move each into
                        // the TMEM A operand as soon as the last chunk's MMAs have read the
                        // old one, so step t+1's first MMAs overlap this chunk's epilogue
                        for (int ks = 0; ks < C::KS - 1; ++ks) {
                            ptx::mbar_wait(a_free + ks, afph);
                            ptx::tc_fence_after();
                            publish(ks, ks + 1, t == p.Q);
                        }
                        afph ^= 1;
                    }
                    ptx::mbar_wait(acc_full + ach, aph);
                    ptx::tc_fence_after();
                    if (C::HOLD && n == C::NCH - 1) {
                        // the last chunk's MMAs are done with A: chunk NCH-2's h(t), held in
                        // registers since its epilogue, goes into the last K-slice now
                        uint32_t hi[4], lo[4];
#pragma unroll
                        for (int w = 0; w < 4; ++w) {
                            hi[w] = t == p.Q ? 0u : hold[w];
                            lo[w] = t == p.Q ? 0u : hold[4 + w];
                        }
                        ptx::tmem_st4(lane_base + C::A_HI + (C::NCH - 2) * 16 + 4 * u, hi);
                        ptx::tmem_st4(lane_base + C::A_LO + (C::NCH - 2) * 16 + 4 * u, lo);
                    }
                    // XM: every MMA of step t has completed (the last chunk's included): the
                    // A image may take x(t+1) for the next step
                    if (C::XM && n == C::NCH - 1 && t < p.Q) put_x(t + 1);
                    if (e == 0 && lane == 0) trace_ev(p, trace_cnt, 4, t, n);
                    float a[2][16];   // 2 groups x 4 neurons x (o, c, lambda, in), scaled domain
                    tmem_ld16(lane_base + ach * 128 + (8 * u) * 4, a[0]);
                    tmem_ld16(lane_base + ach * 128 + (8 * u + 4) * 4, a[1]);
                    ptx::tmem_wait_ld();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(acc_empty + ach);   // accumulator drained
                    float hv[8];
                    // gates: sig_e2 / tanh_e2 (common.cuh) -- accurate forms, no shared
                    // reciprocal (a shared one biased H; measured, DESIGN R26)
#pragma unroll
                    for (int g4 = 0; g4 < 2; ++g4) {
#pragma unroll
                        for (int nb = 0; nb < 4; ++nb) {
                            const int j = n * 32 + 8 * u + 4 * g4 + nb;
                            const float* w = p.wb + j * (4 * (SS + 1));   // [gate][b, W_0..W_{S-1}]
                            // exp2 argument k_g (acc 2^-sigma + b + x W): k_g is folded into
                            // W|b on the host, so it is FFMA(k 2^-sigma, acc, b') + x W'
                            float arg[4];
#pragma unroll
                            for (int g = 0; g < 4; ++g) {
                                if constexpr (C::XM != 0) {   // x W + b is in the accumulator
                                    arg[g] = (g == 1 ? kT : kS) * a[g4][nb * 4 + g];
                                } else {
                                    float v = fmaf(g == 1 ? kT : kS, a[g4][nb * 4 + g], w[g * (SS + 1)]);
#pragma unroll
                                    for (int s = 0; s < SS; ++s) v = fmaf(xs[s], w[g * (SS + 1) + 1 + s], v);
                                    arg[g] = v;
                                }
                            }
                            const float so = sig_e2(arg[0]);   // o
                            const float tc = tanh_e2(arg[1]);  // c~
                            const float sl = sig_e2(arg[2]);   // lambda
                            const float si = sig_e2(arg[3]);   // in
                            const int ci = n * 8 + 4 * g4 + nb;
                            const float cn = fmaf(sl, c[ci], si * tc);
                            c[ci] = cn;
                            hv[4 * g4 + nb] = so * tanh_acc(cn);
                        }
                    }
                    // stage h(t) of these 8 neurons as fp16 hi|lo pairs (the A operand
                    // format); at the last step also store the fp32 H(Q) row segment
                    {
                        uint32_t hi[4], lo[4];
                        split_h8(hv, hi, lo);
                        if (C::HOLD && n == C::NCH - 1) {   // A is free: straight into TMEM (zeros after step Q)
#pragma unroll
                            for (int w = 0; w < 4; ++w)
                                if (t == p.Q) hi[w] = lo[w] = 0u;
                            ptx::tmem_st4(lane_base + C::A_HI + n * 16 + 4 * u, hi);
                            ptx::tmem_st4(lane_base + C::A_LO + n * 16 + 4 * u, lo);
                        } else if (C::HOLD && n == C::NCH - 2) {
#pragma unroll
                            for (int w = 0; w < 4; ++w) {
                                hold[w] = hi[w];
                                hold[4 + w] = lo[w];
                            }
                        } else {
#pragma unroll
                            for (int w = 0; w < 4; ++w) {
                                my_stg[(n * 8 + w) * 32] = hi[w];
                                my_stg[(n * 8 + 4 + w) * 32] = lo[w];
                            }
                        }
                    }
                    if (t == p.Q && valid && p.rbeta) {
                        const double* bj = p.rbeta + n * 32 + 8 * u;
#pragma unroll
                        for (int i = 0; i < 8; ++i) yacc = fma((double)hv[i], __ldg(bj + i), yacc);
                    } else if (t == p.Q && valid) {
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
                    if (e == 0 && lane == 0) trace_ev(p, trace_cnt, 5, t, n);
                    if (++ach == 2) { ach = 0; aph ^= 1; }
                }
                if (C::HOLD) {   // the last K-slice is in TMEM: release it
                    ptx::tmem_wait_st();
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(a_ready + C::KS - 1);
                } else {
                    publish(C::KS - 1, C::KS, t == p.Q);
                }
                if (e == 0 && lane == 0) trace_ev(p, trace_cnt, 6, t, 0);
            }
            if (p.rbeta && valid) p.ryp[u * p.N + row] = yacc;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kTcProdWarp) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

// Build the pre-swizzled fp16 hi/lo images of U_cat (scaled by 2^sigma):
// image[(n*KS + s)*2 + part][sw128(nrow = jj*4 + g, kk)] for neuron n*32+jj, gate g, K = 64s + kk.
// pair = 1 (wide LSTM with N = 256 MMA units): chunks 2m, 2m+1 of a K-slice are adjacent
// 16 KB tiles, i.e. one 256-row SW128 tile: image[((m*KS + s)*2 + part)][chunk % 2][16 KB]
// slices: streamed slices per chunk in the non-pair layout (KS, or KS + 1 with the XM [W; b] slice)
__global__ void k_pack_u(const float* __restrict__ U, int M, float scale, uint8_t* __restrict__ img, int pair,
                         int slices) {
    const int KS = M / 64, NCH = M / 32;
    const int64_t total = (int64_t)NCH * KS * 128 * 64;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        int kk = (int)(e % 64);
        int nrow = (int)((e / 64) % 128);
        int s = (int)((e / (64 * 128)) % KS);
        int n = (int)(e / ((int64_t)64 * 128 * KS));
        int jj = nrow >> 2, g = nrow & 3;
        float v = U[(size_t)(64 * s + kk) * (4 * M) + g * M + n * 32 + jj] * scale;
        __half hi = __float2half_rn(v);
        __half lo = __float2half_rn(v - __half2float(hi));
        uint8_t* base = pair ? img + (size_t)(((n >> 1) * KS + s) * 2) * 2 * kTcSliceBytes + (size_t)(n & 1) * kTcSliceBytes
                             : img + (size_t)((n * slices + s) * 2) * kTcSliceBytes;
        uint32_t off = ptx::sw128_offset(nrow, kk);
        *reinterpret_cast<__half*>(base + off) = hi;
        *reinterpret_cast<__half*>(base + (pair ? 2 : 1) * kTcSliceBytes + off) = lo;
    }
}

template <int M, int SS>
cudaError_t launch_lstm_tc(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    using C = TcCfg<M>;
    static TcParams p;   // host staging of the (large) parameter block
    p.X = X; p.ldx = ldx; p.N = N; p.H = H; p.ldh = ldh;
    p.Uimg = static_cast<const uint8_t*>(h->tc_ops);
    p.S = h->S; p.Q = h->Q;
    p.two_pass = h->weight_grid == 1;
    p.debug_no_u = std::getenv("ELMRNN_DEBUG_NO_U") != nullptr;
    p.ntiles = (N + kTcRows - 1) / kTcRows;
    // a1: stage each full tile's X block when X is 16-byte aligned and it fits
    p.xbytes = ptx::xstage_host(X, ldx, C::SMEM);   // a1: stage each full tile's X block when it fits
    p.rbeta = h->ro_beta; p.ryp = h->ro_yp;
    h->ro_slots = 4;
    const int smem = C::SMEM + (int)p.xbytes;
    p.k_sig = -1.4426950408889634f * h->tc_inv_scale;
    p.k_tanh = 2.8853900817779268f * h->tc_inv_scale;
    std::copy(h->tc_wb.begin(), h->tc_wb.end(), p.wb);   // W | b captured at init
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_lstm_tc<M, SS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem))) return e;
    int grid = (int)std::min<int64_t>(p.ntiles, h->sm_count);
    const char* tpath = std::getenv("ELMRNN_TRACE");
    unsigned long long* tbuf = nullptr;
    p.trace = nullptr;
    p.trace_cap = 0;
    if (tpath && *tpath) {
        p.trace_cap = 1 << 16;
        if ((e = cudaMalloc(&tbuf, sizeof(unsigned long long) * p.trace_cap))) return e;
        cudaMemsetAsync(tbuf, 0, sizeof(unsigned long long) * p.trace_cap, h->stream);
        p.trace = tbuf;
    }
    k_lstm_tc<M, SS><<<grid, kTcThreads, smem, h->stream>>>(p);
    h->launches++;
    if ((e = cudaGetLastError())) return e;
    if (tbuf) {   // debug path: synchronous dump of CTA 0's event trace
        std::vector<unsigned long long> hbuf(p.trace_cap);
        cudaMemcpyAsync(hbuf.data(), tbuf, sizeof(unsigned long long) * p.trace_cap, cudaMemcpyDeviceToHost,
                        h->stream);
        cudaStreamSynchronize(h->stream);
        cudaFree(tbuf);
        if (FILE* f = std::fopen(tpath, "w")) {
            std::fprintf(f, "kind,step,chunk,clock\n");
            for (auto v : hbuf)
                if (v) std::fprintf(f, "%llu,%llu,%llu,%llu\n", v >> 56, (v >> 40) & 0xFFFF, (v >> 32) & 0xFF,
                                    v & 0xFFFFFFFFull);
            std::fclose(f);
        }
    }
    return cudaSuccess;
}

}  // namespace

// the kernel is specialised on S in {1, 2, 4}; S = 3 rounds up with zero W
static int tc_padded_s(int S) { return S <= 1 ? 1 : (S <= 2 ? 2 : 4); }

bool tc_supported(const elmrnn* h) {
    if (h->arch == kArchGRU) return gru_tc_supported(h) || gru_wide_supported(h);
    if (h->arch == kArchFC) return fc_tc_supported(h);
    if (h->arch != kArchLSTM) return false;
    if (lstm_wide_supported(h)) return true;   // 256 < M <= 1024: hbuild_lstm_wide.cu
    if (h->M != 128 && h->M != 256) return false;
    if (h->S > 4) return false;
    return (tc_padded_s(h->S) + 1) * 4 * h->M <= kTcWbMax;
}

cudaError_t tc_prepare(elmrnn* h) {
    if (h->arch == kArchGRU) return gru_tc_supported(h) ? gru_tc_prepare(h) : gru_wide_prepare(h);
    if (h->arch == kArchFC) return fc_tc_prepare(h);
    const int M = h->M;
    const bool wide = lstm_wide_supported(h);
    const int xm = (!wide && M == 128) ? TcCfg<128>::XM : 0;   // the XM [W; b] slice per chunk
    const int slices = M / 64 + xm;
    size_t bytes = (size_t)(M / 32) * slices * kTcStageBytes;
    if (wide) bytes += sizeof(float) * (size_t)M * 4 * (tc_padded_s(h->S) + 1);   // W | b in global memory
    cudaError_t e;
    if ((e = cudaMalloc(&h->tc_ops, bytes))) return e;
    h->tc_ops_bytes = bytes;
    if ((e = cudaMemsetAsync(h->tc_ops, 0, bytes, h->stream))) return e;
    // sigma: largest power of two keeping |U| * 2^sigma < 1 (exact scaling)
    int sigma = h->rec_scale == 1 ? 0 : (int)std::floor(std::log2(std::sqrt((double)M)));
    float scale = std::ldexp(1.0f, sigma);
    h->tc_inv_scale = std::ldexp(1.0f, -sigma);
    // W | b for the x(t) W + b epilogue term travel in the kernel parameter
    // block, scaled by 2^sigma (exact) and laid out [neuron][gate][b, W_0..W_{S-1}]
    const int GM = 4 * M, S = h->S, SP = tc_padded_s(S);
    std::vector<float> W((size_t)S * GM), b(GM);
    if ((e = cudaMemcpyAsync(W.data(), h->W, sizeof(float) * S * GM, cudaMemcpyDeviceToHost, h->stream))) return e;
    if ((e = cudaMemcpyAsync(b.data(), h->b, sizeof(float) * GM, cudaMemcpyDeviceToHost, h->stream))) return e;
    if ((e = cudaStreamSynchronize(h->stream))) return e;
    // [j][gate][b, W_0..W_{S-1}] x k_g with k_g = -log2(e) (sigmoid gates o, lambda, in)
    // or 2 log2(e) (tanh gate c~): the epilogue's exp2 argument is k_g pre-activation
    h->tc_wb.assign((size_t)M * 4 * (SP + 1), 0.0f);
    for (int j = 0; j < M; ++j)
        for (int g = 0; g < 4; ++g) {
            const double kg = g == 1 ? 2.8853900817779268 : -1.4426950408889634;
            float* d = h->tc_wb.data() + ((size_t)j * 4 + g) * (SP + 1);
            d[0] = (float)(kg * b[g * M + j]);
            for (int s2 = 0; s2 < S; ++s2) d[1 + s2] = (float)(kg * W[(size_t)s2 * GM + g * M + j]);
        }
    if (wide &&
        (e = cudaMemcpyAsync(static_cast<uint8_t*>(h->tc_ops) + lstm_wide_wb_offset(h), h->tc_wb.data(),
                             sizeof(float) * h->tc_wb.size(), cudaMemcpyHostToDevice, h->stream)))
        return e;
    int64_t total = (int64_t)(M / 32) * (M / 64) * 128 * 64;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 4096);
    k_pack_u<<<blocks, 256, 0, h->stream>>>(h->rec, M, scale, static_cast<uint8_t*>(h->tc_ops),
                                            wide && lstm_wide_pair(h) ? 1 : 0, slices);
    h->launches++;
    if ((e = cudaGetLastError())) return e;
    if (xm) {   // XM B slices: [W; b] x 2^sigma of each chunk's gate rows (nrow = jj*4 + g), K = s (W_s), K = S (b)
        const int NCH = M / 32;
        std::vector<uint8_t> xs((size_t)NCH * kTcStageBytes, 0);
        for (int n = 0; n < NCH; ++n)
            for (int nrow = 0; nrow < 128; ++nrow) {
                const int jj = nrow >> 2, g = nrow & 3, j = n * 32 + jj;
                for (int k = 0; k <= S; ++k) {
                    const float v = (k < S ? W[(size_t)k * GM + g * M + j] : b[g * M + j]) * scale;
                    const __half hi = __float2half_rn(v);
                    const __half lo = __float2half_rn(v - __half2float(hi));
                    uint8_t* base = xs.data() + (size_t)n * kTcStageBytes;
                    const uint32_t off = ptx::sw128_offset((uint32_t)nrow, (uint32_t)k);
                    *reinterpret_cast<__half*>(base + off) = hi;
                    *reinterpret_cast<__half*>(base + kTcSliceBytes + off) = lo;
                }
            }
        for (int n = 0; n < NCH; ++n)
            if ((e = cudaMemcpyAsync(static_cast<uint8_t*>(h->tc_ops) + ((size_t)n * slices + M / 64) * kTcStageBytes,
                                     xs.data() + (size_t)n * kTcStageBytes, kTcStageBytes, cudaMemcpyHostToDevice,
                                     h->stream)))
                return e;
        if ((e = cudaStreamSynchronize(h->stream))) return e;
    }
    return cudaSuccess;
}

template <int M>
static cudaError_t launch_m(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    switch (tc_padded_s(h->S)) {
    case 1: return launch_lstm_tc<M, 1>(h, X, ldx, N, H, ldh);
    case 2: return launch_lstm_tc<M, 2>(h, X, ldx, N, H, ldh);
    case 4: return launch_lstm_tc<M, 4>(h, X, ldx, N, H, ldh);
    }
    return cudaErrorNotSupported;
}

cudaError_t launch_dense_tc(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    if (h->arch == kArchGRU)
        return gru_tc_supported(h) ? launch_gru_tc(h, X, ldx, N, H, ldh) : launch_gru_wide(h, X, ldx, N, H, ldh);
    if (h->arch == kArchFC) return launch_fc_tc(h, X, ldx, N, H, ldh);
    if (h->M == 256) return launch_m<256>(h, X, ldx, N, H, ldh);
    if (h->M == 128) return launch_m<128>(h, X, ldx, N, H, ldh);
    if (lstm_wide_supported(h)) return launch_lstm_wide(h, X, ldx, N, H, ldh);
    return cudaErrorNotSupported;
}

}  // namespace elm
