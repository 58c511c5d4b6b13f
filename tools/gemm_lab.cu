// GEMM lab (tool, not product): times DMMA tile variants of csrc/dgemm_tile.cuh on the hot-path
// shapes against cuBLAS DGEMM and checks their results.  Prints one JSON object per line.
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <cmath>
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

static double* dev_rand(size_t n, unsigned seed) {
    std::vector<double> h(n);
    srand(seed);
    for (auto& v : h) v = (rand() / (double)RAND_MAX) * 2 - 1;
    double* d; CK(cudaMalloc(&d, n * 8)); CK(cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice));
    return d;
}

template <class C>
void run_variant(const char* name, int M, int N, int K, const double* A, const double* B, double* Cm, const double* Cref,
                 int sms, int splitk_force) {
    int occ = 0;
    cudaFuncSetAttribute(k_dgemm_tile<C, StoreEpi, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dgemm_tile<C, StoreEpi, 1>, C::THREADS, C::SMEM);
    DgemmProblem g{M, N, K, A, K, B, K};
    StoreEpi epi{Cm, M};
    int sks[9] = {0};
    int nsk = 0;
    if (splitk_force > 0) sks[nsk++] = splitk_force;
    else { sks[nsk++] = dgemm_pick_splitk<C>(M, N, K, sms, occ > 0 ? occ : 1); for (int s : {1, 2, 4, 8}) sks[nsk++] = s; }
    for (int i = 0; i < nsk; i++) {
        const int sk = sks[i];
        CK(cudaMemset(Cm, 0, (size_t)M * N * 8));
        CK(dgemm_launch<C>(g, sk, epi, 0));
        CK(cudaDeviceSynchronize());
        // check
        std::vector<double> h((size_t)M * N), r((size_t)M * N);
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
        printf("{\"variant\": \"%s\", \"M\": %d, \"N\": %d, \"K\": %d, \"splitk\": %d, \"picked\": %d, \"occ\": %d, \"us\": %.2f, \"tflops\": %.2f, \"relerr\": %.2e}\n",
               name, M, N, K, sk, i == 0 && splitk_force <= 0, occ, us, 2.0 * M * N * K / us / 1e6, md / mr);
    }
}

template <class C>
void run_streamk(const char* name, int M, int N, int K, const double* A, const double* B, double* Cm, const double* Cref,
                 int sms) {
    int occ = 0;
    cudaFuncSetAttribute(k_dgemm_streamk<C, StoreEpi>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dgemm_streamk<C, StoreEpi>, C::THREADS, C::SMEM);
    DgemmProblem g{M, N, K, A, K, B, K};
    StoreEpi epi{Cm, M};
    for (int o = 1; o <= occ; o++) {
        const int G = dgemm_streamk_grid<C>(M, N, K, sms, o);
        StreamK sk{};
        CK(cudaMalloc(&sk.ws, dgemm_streamk_ws_doubles<C>(M, N, G) * 8));
        const int tiles = dgemm_tiles<C>(M, N);
        CK(cudaMalloc(&sk.counters, (tiles + 1) * 4));
        CK(cudaMemset(sk.counters, 0, (tiles + 1) * 4));
        CK(cudaMemset(Cm, 0, (size_t)M * N * 8));
        CK(dgemm_launch_streamk<C>(g, G, sk, epi, 0));
        CK(cudaDeviceSynchronize());
        std::vector<double> h((size_t)M * N), r((size_t)M * N);
        CK(cudaMemcpy(h.data(), Cm, h.size() * 8, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(r.data(), Cref, r.size() * 8, cudaMemcpyDeviceToHost));
        double md = 0, mr = 0;
        for (size_t j = 0; j < h.size(); j++) { md = fmax(md, fabs(h[j] - r[j])); mr = fmax(mr, fabs(r[j])); }
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int w = 0; w < 3; w++) dgemm_launch_streamk<C>(g, G, sk, epi, 0);
        const int reps = 20;
        cudaEventRecord(e0);
        for (int w = 0; w < reps; w++) dgemm_launch_streamk<C>(g, G, sk, epi, 0);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / reps;
        printf("{\"variant\": \"SK_%s\", \"M\": %d, \"N\": %d, \"K\": %d, \"occ\": %d, \"G\": %d, \"us\": %.2f, \"tflops\": %.2f, \"relerr\": %.2e}\n",
               name, M, N, K, o, G, us, 2.0 * M * N * K / us / 1e6, md / mr);
        cudaFree(sk.ws); cudaFree(sk.counters);
    }
}

int main(int argc, char** argv) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cublasHandle_t hb; cublasCreate(&hb);
    struct Shape { int M, N, K; } all_shapes[] = {{1023, 256, 1024}, {1023, 256, 2048}, {2046, 256, 1024}, {2047, 512, 2048},
                                              {2047, 512, 4096}, {4094, 512, 2048}, {4095, 128, 4096}, {4095, 128, 8192},
                                              {8190, 128, 4096}};
    const int nshapes = argc > 1 ? atoi(argv[1]) : 9;   // first n shapes (3 = config-2 shapes only)
    std::vector<Shape> shapes(all_shapes, all_shapes + nshapes);
    for (auto s : shapes) {
        const int M = s.M, N = s.N, K = s.K;
        const int Mp = (M + 255) / 256 * 256, Np = (N + 255) / 256 * 256;
        double* A = dev_rand((size_t)Mp * K, 1);
        double* B = dev_rand((size_t)Np * K, 2);
        double *C, *Cr; CK(cudaMalloc(&C, (size_t)M * N * 8)); CK(cudaMalloc(&Cr, (size_t)M * N * 8));
        // cuBLAS reference: C (col-major M x N) = A^T(KxM col-major)^T ... A row-major MxK == col-major KxM
        const double one = 1.0, zero = 0.0;
        cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, M, N, K, &one, A, K, B, K, &zero, Cr, M);
        CK(cudaDeviceSynchronize());
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int w = 0; w < 3; w++) cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, M, N, K, &one, A, K, B, K, &zero, Cr, M);
        cudaEventRecord(e0);
        for (int w = 0; w < 20; w++) cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, M, N, K, &one, A, K, B, K, &zero, Cr, M);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"variant\": \"cublas\", \"M\": %d, \"N\": %d, \"K\": %d, \"us\": %.2f, \"tflops\": %.2f}\n", M, N, K,
               ms * 1e3 / 20, 2.0 * M * N * K / (ms * 1e3 / 20) / 1e6);
        const bool big = (M == 4095 && N == 4095);
        const int f = big ? 1 : 0;
        run_streamk<DgemmCfg<64, 64, 16, 2, 2, 4, 2>>("64x64k16_w2x2_s4", M, N, K, A, B, C, Cr, sms);
        run_streamk<DgemmCfg<64, 64, 16, 2, 2, 3, 3>>("64x64k16_w2x2_s3", M, N, K, A, B, C, Cr, sms);

        if (big) { cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(Cr); continue; }
        run_variant<DgemmCfg<64, 64, 16, 2, 2, 4, 2>>("64x64k16_w2x2_s4", M, N, K, A, B, C, Cr, sms, f);
        run_variant<DgemmCfg<64, 64, 16, 2, 2, 3, 3>>("64x64k16_w2x2_s3", M, N, K, A, B, C, Cr, sms, f);
        run_variant<DgemmCfg<64, 64, 32, 2, 2, 3, 2>>("64x64k32_w2x2_s3", M, N, K, A, B, C, Cr, sms, f);
        run_variant<DgemmCfg<128, 64, 16, 4, 2, 3, 2>>("128x64k16_w4x2_s3", M, N, K, A, B, C, Cr, sms, f);
        run_variant<DgemmCfg<64, 128, 16, 2, 4, 3, 2>>("64x128k16_w2x4_s3", M, N, K, A, B, C, Cr, sms, f);
        run_variant<DgemmCfg<128, 64, 16, 2, 2, 3, 2>>("128x64k16_w2x2_s3", M, N, K, A, B, C, Cr, sms, f);
        run_variant<DgemmCfg<64, 64, 16, 2, 2, 6, 2>>("64x64k16_w2x2_s6", M, N, K, A, B, C, Cr, sms, f);
        run_variant<DgemmCfg<32, 64, 16, 1, 2, 4, 4>>("32x64k16_w1x2_s4", M, N, K, A, B, C, Cr, sms, f);
        cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(Cr);
    }
    return 0;
}
