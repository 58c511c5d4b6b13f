// GEMM lab 5 (tool, not product): the per-parameter grouped Schur GEMM  Y_p = H_p X_p  as a
// batched DMMA tile GEMM (batch = parameter group), on the config-2/3/5 group shapes.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2211_15308_b200/csrc/dgemm_tile.cuh"

using namespace dd;

struct BEpi {
    double* C; int ldc; int N;
    __device__ void operator()(int b, int row, int col, double v) const { C[row + (size_t)(b * N + col) * ldc] = v; }
};

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

static double* dev_rand(size_t n, unsigned seed) {
    std::vector<double> h(n);
    srand(seed);
    for (auto& v : h) v = (rand() / (double)RAND_MAX) * 2 - 1;
    double* d; CK(cudaMalloc(&d, n * 8)); CK(cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice));
    return d;
}

template <class C>
void run_variant(const char* name, int P, int M, int N, int K, int Mp, const double* A, const double* B, double* Cm,
                 const double* Cref, int sms) {
    int occ = 0;
    cudaFuncSetAttribute(k_dgemm_tile<C, BEpi, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dgemm_tile<C, BEpi, 1>, C::THREADS, C::SMEM);
    DgemmProblem g{M, N, K, A, K, B, K};
    g.sA = (long long)Mp * K; g.sB = (long long)N * K; g.batch = P;
    g.a_static = 1;
    BEpi epi{Cm, M, N};
    for (int sk : {1, 2, 4, 8}) {
        if (K / C::BK / sk < 4) break;
        CK(cudaMemset(Cm, 0, (size_t)M * N * P * 8));
        CK(dgemm_launch<C>(g, sk, epi, 0));
        CK(cudaDeviceSynchronize());
        std::vector<double> h((size_t)M * N * P), r((size_t)M * N * P);
        CK(cudaMemcpy(h.data(), Cm, h.size() * 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(r.data(), Cref, r.size() * 8, cudaMemcpyDeviceToHost));
        double md = 0, mr = 0;
        for (size_t j = 0; j < h.size(); j++) { md = fmax(md, fabs(h[j] - r[j])); mr = fmax(mr, fabs(r[j])); }
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int w = 0; w < 3; w++) dgemm_launch<C>(g, sk, epi, 0);
        const int reps = 20;
        cudaEventRecord(e0);
        for (int w = 0; w < reps; w++) dgemm_launch<C>(g, sk, epi, 0);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / reps;
        printf("{\"variant\": \"%s\", \"P\": %d, \"M\": %d, \"N\": %d, \"K\": %d, \"splitk\": %d, \"occ\": %d, \"ctas\": %d, \"us\": %.2f, \"tflops\": %.2f, \"relerr\": %.2e}\n",
               name, P, M, N, K, sk, occ, dgemm_tiles<C>(M, N) * sk * P, us, 2.0 * M * N * K * P / us / 1e6, md / mr);
    }
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cublasHandle_t hb; cublasCreate(&hb);
    struct Shape { int P, M, N, K; } shapes[] = {{4, 1023, 64, 1024}, {16, 2047, 32, 2048}, {4, 4095, 32, 4096}};
    for (auto s : shapes) {
        const int P = s.P, M = s.M, N = s.N, K = s.K;
        const int Mp = (M + 255) / 256 * 256;
        double* A = dev_rand((size_t)Mp * K * P, 1);
        double* B = dev_rand((size_t)(N + 64) * K * P, 2);
        double *C, *Cr; CK(cudaMalloc(&C, (size_t)M * N * P * 8)); CK(cudaMalloc(&Cr, (size_t)M * N * P * 8));
        const double one = 1.0, zero = 0.0;
        auto ref = [&]() {
            cublasDgemmStridedBatched(hb, CUBLAS_OP_T, CUBLAS_OP_N, M, N, K, &one, A, K, (long long)Mp * K, B, K,
                                      (long long)N * K, &zero, Cr, M, (long long)M * N, P);
        };
        ref(); CK(cudaDeviceSynchronize());
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int w = 0; w < 3; w++) ref();
        cudaEventRecord(e0);
        for (int w = 0; w < 20; w++) ref();
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"variant\": \"cublas_batched\", \"P\": %d, \"M\": %d, \"N\": %d, \"K\": %d, \"us\": %.2f, \"tflops\": %.2f}\n", P,
               M, N, K, ms * 1e3 / 20, 2.0 * M * N * K * P / (ms * 1e3 / 20) / 1e6);
        if (getenv("LAB_SMALL") && s.P != 4) continue;
        run_variant<DgemmCfg<64, 64, 16, 2, 2, 4, 2>>("64x64k16_w2x2_s4", P, M, N, K, Mp, A, B, C, Cr, sms);
        run_variant<DgemmCfg<128, 32, 16, 4, 1, 3, 2>>("128x32k16_w4x1_s3", P, M, N, K, Mp, A, B, C, Cr, sms);
        run_variant<DgemmCfg<128, 32, 32, 4, 1, 3, 2>>("128x32k32_w4x1_s3", P, M, N, K, Mp, A, B, C, Cr, sms);
        run_variant<DgemmCfg<128, 32, 32, 4, 1, 2, 2>>("128x32k32_w4x1_s2", P, M, N, K, Mp, A, B, C, Cr, sms);
        run_variant<DgemmCfg<128, 32, 16, 4, 1, 5, 2>>("128x32k16_w4x1_s5", P, M, N, K, Mp, A, B, C, Cr, sms);
        run_variant<DgemmCfg<128, 32, 16, 2, 1, 3, 2>>("128x32k16_w2x1_s3", P, M, N, K, Mp, A, B, C, Cr, sms);
        run_variant<DgemmCfg<64, 32, 32, 2, 1, 3, 4>>("64x32k32_w2x1_s3", P, M, N, K, Mp, A, B, C, Cr, sms);
        run_variant<DgemmCfg<256, 32, 16, 8, 1, 3, 1>>("256x32k16_w8x1_s3", P, M, N, K, Mp, A, B, C, Cr, sms);
        run_variant<DgemmCfg<128, 64, 16, 4, 2, 3, 1>>("128x64k16_w4x2_s3", P, M, N, K, Mp, A, B, C, Cr, sms);
        run_variant<DgemmCfg<64, 64, 32, 2, 2, 3, 2>>("64x64k32_w2x2_s3", P, M, N, K, Mp, A, B, C, Cr, sms);
        cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(Cr);
    }
    return 0;
}
