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
//   warps: 0 = bulk-copy producer (U stages from L2), 1 = MMA issuer (one
//          thread), 2 = TMEM allocator, 3 idle, 4..11 = epilogue (2 per TMEM
//          lane quadrant; a thread owns one row and 16 neurons per chunk and
//          keeps c(t) for its 128 neurons in registers).
//   per step: NCH = M/32 chunks of 32 neurons x 4 gates = 128 accumulator
//   columns; chunk n+1's MMAs overlap chunk n's epilogue.  After the last
//   chunk the epilogue converts h(t) (TMEM) to fp16 hi/lo into A and
//   releases the next step's MMAs; after step Q it stores H(Q) rows.
//   W and b (x W + b on FFMA) are kernel parameters: warp-uniform constant
//   bank reads.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace elm {

namespace {

constexpr int kTcRows = 128;
constexpr int kTcStages = 3;
constexpr int kTcSliceBytes = 128 * 64 * 2;      // one 128 x 64 fp16 SW128 tile
constexpr int kTcStageBytes = 2 * kTcSliceBytes;  // hi + lo
constexpr int kTcEpiWarps = 8;
constexpr int kTcThreads = (4 + kTcEpiWarps) * 32;
constexpr int kTcWbMax = 7168;                    // floats of W|b in the parameter block

struct TcParams {
    const float* X;
    int64_t ldx, N;
    float* H;
    int64_t ldh;
    const uint8_t* Uimg;   // [NCH][KS][hi|lo][16 KB] pre-swizzled images
    int S, Q;
    int64_t ntiles;
    float inv_scale;       // 2^-sigma
    float wb[kTcWbMax];    // W [S][4M] then b [4M]
};

template <int M>
struct TcCfg {
    static constexpr int NCH = M / 32;
    static constexpr int KS = M / 64;
    static constexpr int A_BYTES = kTcRows * M * 2;   // one of hi / lo
    static constexpr int SMEM = 1024 + 2 * A_BYTES + kTcStages * kTcStageBytes + 256;
    static constexpr int TMEM_COLS = 512;
    static constexpr int H_COL = 256;                 // first h(t) staging column
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
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            taddr),
        "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
        "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
        "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
        "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
        "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
        "r"(__float_as_uint(v[15]))
        : "memory");
}

// Write 16 consecutive h values (K indices k0..k0+15, k0 % 16 == 0) of row r
// into the A operand as fp16 hi and lo parts (K-major SW128, 64-wide slices).
__device__ __forceinline__ void store_h16(uint8_t* A_hi, uint8_t* A_lo, int r, int k0, const float (&h)[16]) {
    uint32_t hi[8], lo[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        __half a0 = __float2half_rn(h[2 * i]), a1 = __float2half_rn(h[2 * i + 1]);
        __half b0 = __float2half_rn(h[2 * i] - __half2float(a0));
        __half b1 = __float2half_rn(h[2 * i + 1] - __half2float(a1));
        hi[i] = (uint32_t)__half_as_ushort(a0) | ((uint32_t)__half_as_ushort(a1) << 16);
        lo[i] = (uint32_t)__half_as_ushort(b0) | ((uint32_t)__half_as_ushort(b1) << 16);
    }
    const int s = k0 >> 6, kin = k0 & 63;
    const uint32_t o0 = s * kTcSliceBytes + ptx::sw128_offset(r, kin);
    const uint32_t o1 = s * kTcSliceBytes + ptx::sw128_offset(r, kin + 8);
    *reinterpret_cast<uint4*>(A_hi + o0) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(A_hi + o1) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
    *reinterpret_cast<uint4*>(A_lo + o0) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
    *reinterpret_cast<uint4*>(A_lo + o1) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
}

template <int M>
__global__ void __launch_bounds__(kTcThreads, 1) k_lstm_tc(const __grid_constant__ TcParams p) {
    using C = TcCfg<M>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* A_hi = smem;
    uint8_t* A_lo = A_hi + C::A_BYTES;
    uint8_t* stages = A_lo + C::A_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(stages + kTcStages * kTcStageBytes);
    uint64_t* full = bars;                       // [kTcStages]
    uint64_t* empty = bars + kTcStages;          // [kTcStages]
    uint64_t* acc_full = bars + 2 * kTcStages;   // [2]
    uint64_t* acc_empty = acc_full + 2;          // [2]
    uint64_t* a_ready = acc_empty + 2;           // [1]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_ready + 1);

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
        ptx::mbar_init(a_ready, kTcEpiWarps);
        ptx::fence_mbar_init();
    }
    if (warp == 2) {
        ptx::tmem_alloc(tmem_slot, C::TMEM_COLS);
        ptx::tmem_relinquish();
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int64_t steps_total = ((p.ntiles - blockIdx.x + gridDim.x - 1) / gridDim.x) * p.Q;

    if (warp == 0) {
        // ---------------- producer: stream U slices (chunk, K-slice) from L2
        if (lane == 0) {
            uint32_t st = 0, ph = 0;
            for (int64_t s = 0; s < steps_total; ++s) {
                for (int c = 0; c < C::NCH * C::KS; ++c) {
                    ptx::mbar_wait(empty + st, ph ^ 1);
                    ptx::mbar_arrive_expect_tx(full + st, kTcStageBytes);
                    ptx::bulk_g2s(stages + st * kTcStageBytes, p.Uimg + (size_t)c * kTcStageBytes, kTcStageBytes,
                                  full + st);
                    if (++st == kTcStages) { st = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_f16(128, 128);
            const uint32_t a_hi = ptx::smem_u32(A_hi), a_lo = ptx::smem_u32(A_lo);
            const uint32_t b0 = ptx::smem_u32(stages);
            uint32_t st = 0, ph = 0, ach = 0, aph = 0;
            for (int64_t s = 0; s < steps_total; ++s) {
                ptx::mbar_wait(a_ready, (uint32_t)(s & 1));   // h(t-1) hi/lo is in A
                ptx::tc_fence_after();
                for (int n = 0; n < C::NCH; ++n) {
                    ptx::mbar_wait(acc_empty + ach, aph ^ 1);
                    ptx::tc_fence_after();
                    const uint32_t d = tmem + ach * 128;
                    for (int ks = 0; ks < C::KS; ++ks) {
                        ptx::mbar_wait(full + st, ph);
                        ptx::tc_fence_after();
                        const uint32_t bh = b0 + st * kTcStageBytes, bl = bh + kTcSliceBytes;
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            const uint64_t dah = ptx::desc_sw128_kmajor(a_hi + ks * kTcSliceBytes + kk * 32);
                            const uint64_t dal = ptx::desc_sw128_kmajor(a_lo + ks * kTcSliceBytes + kk * 32);
                            const uint64_t dbh = ptx::desc_sw128_kmajor(bh + kk * 32);
                            const uint64_t dbl = ptx::desc_sw128_kmajor(bl + kk * 32);
                            ptx::mma_f16_ss(d, dah, dbh, idesc, (ks | kk) != 0);
                            ptx::mma_f16_ss(d, dah, dbl, idesc, 1);
                            ptx::mma_f16_ss(d, dal, dbh, idesc, 1);
                        }
                        ptx::mma_commit(empty + st);                      // frees the U stage
                        if (++st == kTcStages) { st = 0; ph ^= 1; }
                    }
                    ptx::mma_commit(acc_full + ach);                      // chunk accumulator ready
                    if (++ach == 2) { ach = 0; aph ^= 1; }
                }
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue: gates, c/h update, A write-back, H(Q) store
        const int e = warp - 4, q = e & 3, u = e >> 2;
        const int r = 32 * q + lane;                 // tile row = TMEM lane
        const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
        const int S = p.S, GM = 4 * M;
        const float* Wp = p.wb;
        const float* bp = p.wb + S * GM;
        float c[C::NCH * 16];
        uint32_t ach = 0, aph = 0;
        // h(0) = 0 for the first tile
        {
            float z[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) z[i] = 0.0f;
#pragma unroll
            for (int n = 0; n < C::NCH; ++n) store_h16(A_hi, A_lo, r, n * 32 + 16 * u, z);
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(a_ready);
        }
        for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x) {
            const int64_t row = tile * kTcRows + r;
            const bool valid = row < p.N;
            const float* xrow = p.X + (valid ? row : 0) * p.ldx;
#pragma unroll
            for (int i = 0; i < C::NCH * 16; ++i) c[i] = 0.0f;
            for (int t = 1; t <= p.Q; ++t) {
                float xs[8];
#pragma unroll
                for (int s = 0; s < 8; ++s) xs[s] = (s < S && valid) ? __ldg(xrow + (int64_t)(t - 1) * S + s) : 0.0f;
#pragma unroll
                for (int n = 0; n < C::NCH; ++n) {
                    ptx::mbar_wait(acc_full + ach, aph);
                    ptx::tc_fence_after();
                    float hv[16];
#pragma unroll
                    for (int g4 = 0; g4 < 4; ++g4) {
                        float a[16];   // 4 neurons x (o, c, lambda, in)
                        tmem_ld16(lane_base + ach * 128 + (16 * u + 4 * g4) * 4, a);
                        ptx::tmem_wait_ld();
                        if (g4 == 3) {   // accumulator buffer fully read: release it
                            ptx::tc_fence_before();
                            __syncwarp();
                            if (lane == 0) ptx::mbar_arrive(acc_empty + ach);
                        }
#pragma unroll
                        for (int nb = 0; nb < 4; ++nb) {
                            const int jl = 16 * u + 4 * g4 + nb;   // neuron within chunk
                            const int j = n * 32 + jl;
                            float pre[4];
#pragma unroll
                            for (int g = 0; g < 4; ++g) {
                                float v = fmaf(a[nb * 4 + g], p.inv_scale, bp[g * M + j]);
#pragma unroll
                                for (int s = 0; s < 8; ++s)
                                    if (s < S) v = fmaf(xs[s], Wp[s * GM + g * M + j], v);
                                pre[g] = v;
                            }
                            const int ci = n * 16 + 4 * g4 + nb;
                            const float cn = sigmoidf_(pre[2]) * c[ci] + sigmoidf_(pre[3]) * tanhf_(pre[1]);
                            c[ci] = cn;
                            hv[4 * g4 + nb] = sigmoidf_(pre[0]) * tanhf_(cn);
                        }
                    }
                    tmem_st16(lane_base + C::H_COL + n * 32 + 16 * u, hv);
                    if (++ach == 2) { ach = 0; aph ^= 1; }
                }
                // all MMAs of step t are complete (the last chunk's commit covers them):
                // publish h(t) as the next A operand, or store H(Q) and reset A for the next tile
                ptx::tmem_wait_st();
#pragma unroll
                for (int n = 0; n < C::NCH; ++n) {
                    float hv[16];
                    tmem_ld16(lane_base + C::H_COL + n * 32 + 16 * u, hv);
                    ptx::tmem_wait_ld();
                    if (t == p.Q) {
                        if (valid) {
                            float4* dst = reinterpret_cast<float4*>(p.H + row * p.ldh + n * 32 + 16 * u);
                            if ((p.ldh & 3) == 0) {
#pragma unroll
                                for (int i = 0; i < 4; ++i)
                                    dst[i] = make_float4(hv[4 * i], hv[4 * i + 1], hv[4 * i + 2], hv[4 * i + 3]);
                            } else {
                                float* d1 = p.H + row * p.ldh + n * 32 + 16 * u;
#pragma unroll
                                for (int i = 0; i < 16; ++i) d1[i] = hv[i];
                            }
                        }
#pragma unroll
                        for (int i = 0; i < 16; ++i) hv[i] = 0.0f;   // h(0) of the next tile
                    }
                    store_h16(A_hi, A_lo, r, n * 32 + 16 * u, hv);
                }
                ptx::fence_proxy_async_smem();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(a_ready);
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, C::TMEM_COLS);
    }
}

// Build the pre-swizzled fp16 hi/lo images of U_cat (scaled by 2^sigma):
// image[(n*KS + s)*2 + part][sw128(nrow = jj*4 + g, kk)] for neuron n*32+jj, gate g, K = 64s + kk.
__global__ void k_pack_u(const float* __restrict__ U, int M, float scale, uint8_t* __restrict__ img) {
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
        uint8_t* base = img + (size_t)((n * KS + s) * 2) * kTcSliceBytes;
        uint32_t off = ptx::sw128_offset(nrow, kk);
        *reinterpret_cast<__half*>(base + off) = hi;
        *reinterpret_cast<__half*>(base + kTcSliceBytes + off) = lo;
    }
}

template <int M>
cudaError_t launch_lstm_tc(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    using C = TcCfg<M>;
    static TcParams p;   // host staging of the (large) parameter block
    p.X = X; p.ldx = ldx; p.N = N; p.H = H; p.ldh = ldh;
    p.Uimg = static_cast<const uint8_t*>(h->tc_ops);
    p.S = h->S; p.Q = h->Q;
    p.ntiles = (N + kTcRows - 1) / kTcRows;
    p.inv_scale = h->tc_inv_scale;
    std::copy(h->tc_wb.begin(), h->tc_wb.end(), p.wb);   // W | b captured at init
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_lstm_tc<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM))) return e;
    int grid = (int)std::min<int64_t>(p.ntiles, h->sm_count);
    k_lstm_tc<M><<<grid, kTcThreads, C::SMEM, h->stream>>>(p);
    h->launches++;
    return cudaGetLastError();
}

}  // namespace

bool tc_supported(const elmrnn* h) {
    if (h->arch != kArchLSTM) return false;
    if (h->M != 128 && h->M != 256) return false;
    if (h->S > 8) return false;
    return (h->S + 1) * 4 * h->M <= kTcWbMax;
}

cudaError_t tc_prepare(elmrnn* h) {
    const int M = h->M;
    size_t bytes = (size_t)(M / 32) * (M / 64) * kTcStageBytes;
    cudaError_t e;
    if ((e = cudaMalloc(&h->tc_ops, bytes))) return e;
    h->tc_ops_bytes = bytes;
    // sigma: largest power of two keeping |U| * 2^sigma < 1 (exact scaling)
    int sigma = h->rec_scale == 1 ? 0 : (int)std::floor(std::log2(std::sqrt((double)M)));
    float scale = std::ldexp(1.0f, sigma);
    h->tc_inv_scale = std::ldexp(1.0f, -sigma);
    // W | b for the x(t) W + b epilogue term travel in the kernel parameter block
    const int GM = 4 * M;
    h->tc_wb.assign((size_t)(h->S + 1) * GM, 0.0f);
    if ((e = cudaMemcpyAsync(h->tc_wb.data(), h->W, sizeof(float) * h->S * GM, cudaMemcpyDeviceToHost, h->stream)))
        return e;
    if ((e = cudaMemcpyAsync(h->tc_wb.data() + (size_t)h->S * GM, h->b, sizeof(float) * GM, cudaMemcpyDeviceToHost,
                             h->stream)))
        return e;
    if ((e = cudaStreamSynchronize(h->stream))) return e;
    int64_t total = (int64_t)(M / 32) * (M / 64) * 128 * 64;
    int blocks = (int)std::min<int64_t>((total + 255) / 256, 4096);
    k_pack_u<<<blocks, 256, 0, h->stream>>>(h->rec, M, scale, static_cast<uint8_t*>(h->tc_ops));
    h->launches++;
    return cudaGetLastError();
}

cudaError_t launch_dense_tc(elmrnn* h, const float* X, int64_t ldx, int64_t N, float* H, int64_t ldh) {
    if (h->M == 256) return launch_lstm_tc<256>(h, X, ldx, N, H, ldh);
    if (h->M == 128) return launch_lstm_tc<128>(h, X, ldx, N, H, ldh);
    return cudaErrorNotSupported;
}

}  // namespace elm
