// weights.cu -- Alg. 1 line 1 "Randomly assign W, alpha, b" on the GPU.
//
// Counter-based generator of DESIGN.md "Weights" (readings R1, R2): each
// element of logical block `block_id` is
//   key = mix(seed ^ (0xD1B54A32D192ED03 * (block_id+1))),
//   u   = (mix(key + idx) >> 11) * 2^-53,  w = fp32((2u - 1) * scale)
// with mix = SplitMix64's finaliser, idx the row-major index in the logical
// block.  Order independent, so one thread per element.  Blocks that enter a
// tensor-core contraction (FC A, LSTM/GRU U) may be rounded to the fp16 grid
// (RNE) or the tf32 grid (RNA) (opts.weight_grid).  The kernel writes straight
// into the packed device layouts the builders read.
#include <algorithm>
#include <cmath>

#include <cuda_fp16.h>

#include "common.cuh"

namespace elm {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static uint64_t mix64_host(uint64_t z) {
    z += 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// logical [rows][cols] -> dst[r*ld + off + c] (or transposed dst[c*ld + off + r])
__global__ void k_gen_block(uint64_t key, double scale, int grid, int64_t rows, int64_t cols,
                            float* __restrict__ dst, int64_t ld, int64_t off, int transpose) {
    int64_t n = rows * cols;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n;
         idx += (int64_t)gridDim.x * blockDim.x) {
        uint64_t r = mix64(key + (uint64_t)idx);
        double u = (double)(r >> 11) * 0x1p-53;
        float f = __double2float_rn((2.0 * u - 1.0) * scale);
        if (grid == 1) {
            f = __half2float(__float2half_rn(f));
        } else if (grid == 2) {
            uint32_t t;
            asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(t) : "f"(f));
            f = __uint_as_float(t);
        }
        int64_t rr = idx / cols, cc = idx - rr * cols;
        if (transpose)
            dst[cc * ld + off + rr] = f;
        else
            dst[rr * ld + off + cc] = f;
    }
}

// alphaT[k][j] = sum_l A[k][l][j] for k < min(L, Q), 0 otherwise (A logical [L][M][M])
__global__ void k_colsum_lags(const float* __restrict__ A, int M, int L, int Q, float* __restrict__ alT) {
    const int64_t n = (int64_t)Q * M;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(e / M), j = (int)(e % M);
        double s = 0.0;
        if (k < L)
            for (int l = 0; l < M; ++l) s += (double)A[((int64_t)k * M + l) * M + j];
        alT[e] = (float)s;
    }
}

int num_blocks(int arch) {
    switch (arch) {
    case kArchElman: case kArchJordan: case kArchFC: case kArchFCEq8: return 3;
    case kArchNarmax: return 4;
    case kArchLSTM: case kArchLSTMDiag: return 12;
    case kArchGRU: case kArchGRUDiag: return 9;
    }
    return -1;
}

// Logical shape, scale and MMA flag of a block (DESIGN.md "Weights" table).
static bool block_desc(const elmrnn* h, int id, int64_t* rows, int64_t* cols, double* scale, int* mma) {
    const int S = h->S, M = h->M, Q = h->Q;
    const bool unit = h->rec_scale == 1;
    *scale = 1.0;
    *mma = 0;
    switch (h->arch) {
    case kArchElman: case kArchJordan:
        if (id == 0) { *rows = S; *cols = M; return true; }
        if (id == 1) { *rows = 1; *cols = M; return true; }
        if (id == 2) {
            *rows = M; *cols = Q;
            if (h->arch == kArchElman && !unit) *scale = 1.0 / std::sqrt((double)Q);
            return true;
        }
        return false;
    case kArchNarmax:
        if (id == 0) { *rows = S; *cols = M; return true; }
        if (id == 1) { *rows = 1; *cols = M; return true; }
        if (id == 2) { *rows = M; *cols = h->F; return true; }
        if (id == 3) { *rows = M; *cols = h->R; return true; }
        return false;
    case kArchFC:
        if (id == 0) { *rows = S; *cols = M; return true; }
        if (id == 1) { *rows = 1; *cols = M; return true; }
        if (id == 2) {
            *rows = (int64_t)h->fc_lags * M; *cols = M; *mma = 1;
            if (!unit) *scale = 1.0 / std::sqrt((double)M * (double)h->fc_lags);
            return true;
        }
        return false;
    case kArchFCEq8:   // the FC blocks; per-cell use only (no MMA, no grid rounding)
        if (id == 0) { *rows = S; *cols = M; return true; }
        if (id == 1) { *rows = 1; *cols = M; return true; }
        if (id == 2) {
            *rows = (int64_t)h->fc_lags * M; *cols = M;
            if (!unit) *scale = 1.0 / std::sqrt((double)M * (double)h->fc_lags);
            return true;
        }
        return false;
    case kArchLSTMDiag: case kArchGRUDiag:   // per gate W [S][M], u [M] (fan-in 1), b [M]
        if (id < 0 || id >= 3 * h->G) return false;
        if (id % 3 == 0) { *rows = S; *cols = M; return true; }
        *rows = 1; *cols = M;
        return true;
    case kArchLSTM: case kArchGRU: {
        if (id < 0 || id >= 3 * h->G) return false;
        int kind = id % 3;
        if (kind == 0) { *rows = S; *cols = M; return true; }
        if (kind == 1) {
            *rows = M; *cols = M; *mma = 1;
            if (!unit) *scale = 1.0 / std::sqrt((double)M);
            return true;
        }
        *rows = 1; *cols = M;
        return true;
    }
    }
    return false;
}

int64_t logical_block_len(const elmrnn* h, int block_id) {
    int64_t r, c; double s; int m;
    if (!block_desc(h, block_id, &r, &c, &s, &m)) return -1;
    return r * c;
}

static cudaError_t launch_gen(elmrnn* h, int id, float* dst, int64_t ld, int64_t off, int transpose) {
    int64_t rows, cols; double scale; int mma;
    if (!block_desc(h, id, &rows, &cols, &scale, &mma)) return cudaErrorInvalidValue;
    if (rows * cols == 0) return cudaSuccess;
    uint64_t key = mix64_host(h->seed ^ (0xD1B54A32D192ED03ULL * (uint64_t)(id + 1)));
    int64_t n = rows * cols;
    int threads = 256;
    int64_t blocks = (n + threads - 1) / threads;
    if (blocks > 4096) blocks = 4096;
    k_gen_block<<<(int)blocks, threads, 0, h->stream>>>(key, scale, mma ? h->weight_grid : 0, rows, cols,
                                                       dst, ld, off, transpose);
    h->launches++;
    return cudaGetLastError();
}

// Packed layouts:
//   W   [S][G*M]   (gate g in columns g*M .. g*M+M-1)
//   b   [G*M]
//   rec Elman/Jordan alpha^T [Q][M]; NARMAX W'^T [F][M] then W''^T [R][M]; FC A [L*M][M];
//       LSTM/GRU U_cat [M][G*M]; diagonal LSTM/GRU u [G*M];
//       FC by Eq. 8: alpha^T [Q][M] with alpha[k][j] = sum_l A[k][l][j]
cudaError_t gen_weights(elmrnn* h) {
    cudaError_t e;
    const int M = h->M, GM = h->G * h->M;
    switch (h->arch) {
    case kArchElman: case kArchJordan:
        if ((e = launch_gen(h, 0, h->W, M, 0, 0))) return e;
        if ((e = launch_gen(h, 1, h->b, M, 0, 0))) return e;
        return launch_gen(h, 2, h->rec, M, 0, 1);
    case kArchNarmax:
        if ((e = launch_gen(h, 0, h->W, M, 0, 0))) return e;
        if ((e = launch_gen(h, 1, h->b, M, 0, 0))) return e;
        if ((e = launch_gen(h, 2, h->rec, M, 0, 1))) return e;
        // W''^T [R][M] after W'^T: read only when an error window is given (R30)
        return launch_gen(h, 3, h->rec + (size_t)h->F * M, M, 0, 1);
    case kArchFC:
        if ((e = launch_gen(h, 0, h->W, M, 0, 0))) return e;
        if ((e = launch_gen(h, 1, h->b, M, 0, 0))) return e;
        return launch_gen(h, 2, h->rec, M, 0, 0);
    case kArchFCEq8: {
        // Eq. 8: sum_l alpha[j,l,k] h_j(t-k) = (sum_l A[k-1][l][j]) h_j(t-k): the
        // per-lag column sums are formed once here (init, untimed) into alpha^T [Q][M]
        if ((e = launch_gen(h, 0, h->W, M, 0, 0))) return e;
        if ((e = launch_gen(h, 1, h->b, M, 0, 0))) return e;
        const int L = h->fc_lags;
        float* A = nullptr;
        if ((e = cudaMalloc(&A, sizeof(float) * (size_t)L * M * M))) return e;
        if ((e = launch_gen(h, 2, A, M, 0, 0))) { cudaFree(A); return e; }
        const int64_t n = (int64_t)h->Q * M;
        k_colsum_lags<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, h->stream>>>(A, M, L, h->Q, h->rec);
        h->launches++;
        e = cudaGetLastError();
        cudaStreamSynchronize(h->stream);
        cudaFree(A);
        return e;
    }
    case kArchLSTMDiag: case kArchGRUDiag:   // W [S][G*M], u [G*M] (in rec), b [G*M]
        for (int g = 0; g < h->G; ++g) {
            if ((e = launch_gen(h, 3 * g, h->W, GM, (int64_t)g * M, 0))) return e;
            if ((e = launch_gen(h, 3 * g + 1, h->rec, GM, (int64_t)g * M, 0))) return e;
            if ((e = launch_gen(h, 3 * g + 2, h->b, GM, (int64_t)g * M, 0))) return e;
        }
        return cudaSuccess;
    case kArchLSTM: case kArchGRU:
        for (int g = 0; g < h->G; ++g) {
            if ((e = launch_gen(h, 3 * g, h->W, GM, (int64_t)g * M, 0))) return e;
            if ((e = launch_gen(h, 3 * g + 1, h->rec, GM, (int64_t)g * M, 0))) return e;
            if ((e = launch_gen(h, 3 * g + 2, h->b, GM, (int64_t)g * M, 0))) return e;
        }
        return cudaSuccess;
    }
    return cudaErrorInvalidValue;
}

cudaError_t gen_logical_block(elmrnn* h, int block_id, float* dst_dev, int64_t* count) {
    int64_t rows, cols; double s; int m;
    if (!block_desc(h, block_id, &rows, &cols, &s, &m)) return cudaErrorInvalidValue;
    *count = rows * cols;
    return launch_gen(h, block_id, dst_dev, cols, 0, 0);
}

}  // namespace elm
