// Per-column phase clocks of the per-column fold (k_tsqr_merge<24, 2>) merging two
// random n x n triangles, CTA 0: slots 0 loop top, 1 after thread k+1's update,
// 2 after its reflector, 3 after the barrier.  Build with -DELM_QR_TRACE.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_1911_13252_b200/csrc/tsqr.cu"
using namespace elm;
int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 65;
    std::vector<double> h(2 * (size_t)n * n, 0.0);
    for (int s = 0; s < 2; ++s)
        for (int i = 0; i < n; ++i)
            for (int j = i; j < n; ++j) h[(size_t)s * n * n + (size_t)i * n + j] = rand() / (double)RAND_MAX - 0.5 + (i == j ? 2 : 0);
    double* d; cudaMalloc(&d, h.size() * 8);
    unsigned long long* tb; cudaMalloc(&tb, 4096 * 8 * 8);
    for (int rep = 0; rep < 3; ++rep) {
        cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
        cudaMemset(tb, 0, 4096 * 8 * 8);
        cudaMemcpyToSymbol(g_qr_trace, &tb, sizeof(tb));
        const int threads = (2 * n + 31) / 32 * 32;
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        k_tsqr_merge<24, 2><<<1, threads>>>(d, 2, 1, n);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        std::vector<unsigned long long> t(4096 * 8);
        cudaMemcpy(t.data(), tb, t.size() * 8, cudaMemcpyDeviceToHost);
        if (rep < 2) continue;
        printf("n=%d merge %.1f us  (%s)\n", n, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
        double s01 = 0, s12 = 0, s23 = 0, s30 = 0; int cnt = 0;
        for (int k = 0; k + 1 < n; ++k) {
            unsigned long long* c = &t[k * 8];
            unsigned long long* nx = &t[(k + 1) * 8];
            if (!c[0] || !c[1] || !c[2] || !c[3] || !nx[0]) continue;
            s01 += (double)(c[1] - c[0]); s12 += (double)(c[2] - c[1]); s23 += (double)(c[3] - c[2]); s30 += (double)(nx[0] - c[3]);
            ++cnt;
        }
        printf("per column (%d cols): top->update(k+1) %.0f  reflector %.0f  ->barrier exit %.0f  ->next top %.0f  total %.0f cycles\n",
               cnt, s01 / cnt, s12 / cnt, s23 / cnt, s30 / cnt, (s01 + s12 + s23 + s30) / cnt);
    }
    return 0;
}
