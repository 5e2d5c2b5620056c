// Time wy_panel<ROWS> alone (one warp, uncontended): cycles per panel of 16 columns.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1911_13252_b200/csrc/tsqr.cu"
using namespace elm;
template <int ROWS>
__global__ void kp(double* Cg, int LDC, long long* cyc, int reps) {
    extern __shared__ double sm[];
    double* C = sm;
    double* Rd = C + ROWS * LDC;
    double* cg = Rd + 256;
    double* cu = cg + 16;
    double* Gp = cu + 16;
    for (int e = threadIdx.x; e < ROWS * LDC; e += 32) C[e] = Cg[e];
    for (int e = threadIdx.x; e < 256; e += 32) Rd[e] = (e / 16 <= e % 16) ? 1.0 + 0.01 * e : 0.0;
    __syncwarp();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) wy_panel<ROWS>(C, LDC, 0, 16, Rd, cg, cu, Gp);
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = (t1 - t0) / reps;
    Cg[0] = C[5] + cg[3];
}
template <int ROWS> void run() {
    const int LDC = 264;
    std::vector<double> h(ROWS * LDC);
    for (auto& x : h) x = rand() / (double)RAND_MAX - 0.5;
    double* d; long long* c; cudaMalloc(&d, h.size() * 8); cudaMalloc(&c, 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    size_t smem = (ROWS * LDC + 256 + 32 + 256) * 8;
    cudaFuncSetAttribute(kp<ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kp<ROWS><<<1, 32, smem>>>(d, LDC, c, 4);
    kp<ROWS><<<1, 32, smem>>>(d, LDC, c, 16);
    long long hc; cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("wy_panel<%d>: %lld cycles per 16-column panel (%lld per column)  err=%s\n", ROWS, hc, hc / 16,
           cudaGetErrorString(cudaGetLastError()));
}
int main() { run<32>(); run<64>(); run<96>(); return 0; }
