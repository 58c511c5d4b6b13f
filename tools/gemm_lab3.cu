// GEMM lab 3 (tool): per-CTA phase timestamps (%globaltimer) of the split-K cluster kernel on the
// config-2 K1 shape, to locate the per-launch fixed cost.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2211_15308_b200/csrc/dgemm_tile.cuh"
using namespace dd;
struct StoreEpi {
    double* C; int ldc;
    __device__ void operator()(int, int row, int col, double v) const { C[row + (size_t)col * ldc] = v; }
};
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)
int main() {
    using C = DgemmCfg<64, 64, 16, 2, 2, 4, 2>;
    const int M = 1023, N = 256;
    double *A, *B, *Cm; unsigned long long* ts;
    CK(cudaMalloc(&A, (size_t)1024 * 2048 * 8)); CK(cudaMalloc(&B, (size_t)256 * 2048 * 8)); CK(cudaMalloc(&Cm, (size_t)M * N * 8));
    CK(cudaMemset(A, 0, (size_t)1024 * 2048 * 8)); CK(cudaMemset(B, 0, (size_t)256 * 2048 * 8));
    CK(cudaMalloc(&ts, 4096 * 8 * 8));
    for (int sk : {1, 2, 4}) for (int K : {1024, 2048}) {
        DgemmProblem g{M, N, K, A, 2048, B, 2048};
        for (int w = 0; w < 5; w++) dgemm_launch<C>(g, sk, StoreEpi{Cm, M}, 0);
        CK(cudaMemset(ts, 0, 4096 * 64));
        g.ts = ts;
        unsigned long long* dummy; CK(cudaMalloc(&dummy, 8));
        dgemm_launch<C>(g, sk, StoreEpi{Cm, M}, 0);
        CK(cudaDeviceSynchronize());
        const int nct = 64 * sk;
        std::vector<unsigned long long> h(nct * 8);
        CK(cudaMemcpy(h.data(), ts, h.size() * 8, cudaMemcpyDeviceToHost));
        unsigned long long t0 = ~0ull, tend = 0;
        for (int c = 0; c < nct; c++) { t0 = std::min(t0, h[c * 8]); }
        double mx[8] = {0}, mn[8], av[8] = {0};
        for (int i = 0; i < 8; i++) mn[i] = 1e30;
        for (int c = 0; c < nct; c++)
            for (int i = 0; i < 6; i++) {
                if (!h[c * 8 + i]) continue;
                double v = (h[c * 8 + i] - t0) * 1e-3;
                mx[i] = std::max(mx[i], v); mn[i] = std::min(mn[i], v); av[i] += v / nct;
                if (h[c * 8 + i] > tend) tend = h[c * 8 + i];
            }
        printf("{\"splitk\": %d, \"K\": %d, \"span_us\": %.2f", sk, K, (tend - t0) * 1e-3);
        const char* nm[6] = {"start", "mainloop_end", "barrier", "reduced", "epi_done", "unused"};
        for (int i = 0; i < 6; i++) if (mn[i] < 1e29) printf(", \"%s\": [%.2f, %.2f, %.2f]", nm[i], mn[i], av[i], mx[i]);
        printf("}\n");
    }
    return 0;
}
