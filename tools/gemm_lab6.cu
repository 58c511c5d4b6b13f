// GEMM lab 6 (tool, not product): the 3D dense fractional term y = F x (F: 16384^2 fp64, 8 columns,
// HBM-bound) as a stream-K DMMA GEMM, over tile / pipeline variants; reports GB/s of F streamed.
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

__global__ void fill(double* p, size_t n, unsigned seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned h = (unsigned)(i * 2654435761u) ^ seed;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        p[i] = (h & 0xffff) / 65536.0 - 0.5;
    }
}

template <class C>
void run(const char* name, int M, int N, int K, const double* A, const double* B, double* Cm, const double* Cref,
         int sms, int occ_req) {
    int occ = 0;
    cudaFuncSetAttribute(k_dgemm_streamk<C, StoreEpi>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_dgemm_streamk<C, StoreEpi>, C::THREADS, C::SMEM);
    if (occ_req > occ) return;
    DgemmProblem g{M, N, K, A, K, B, K};
    StoreEpi epi{Cm, M};
    const int G = dgemm_streamk_grid<C>(M, N, K, sms, occ_req);
    StreamK sk{};
    CK(cudaMalloc(&sk.ws, dgemm_streamk_ws_doubles<C>(M, N, G) * 8));
    const int tiles = dgemm_tiles<C>(M, N);
    CK(cudaMalloc(&sk.counters, (tiles + 1) * 4));
    CK(cudaMemset(sk.counters, 0, (tiles + 1) * 4));
    CK(dgemm_launch_streamk<C>(g, G, sk, epi, 0));
    CK(cudaDeviceSynchronize());
    std::vector<double> h((size_t)M * N), r((size_t)M * N);
    CK(cudaMemcpy(h.data(), Cm, h.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r.data(), Cref, r.size() * 8, cudaMemcpyDeviceToHost));
    double md = 0, mr = 0;
    for (size_t j = 0; j < h.size(); j++) { md = fmax(md, fabs(h[j] - r[j])); mr = fmax(mr, fabs(r[j])); }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w = 0; w < 2; w++) dgemm_launch_streamk<C>(g, G, sk, epi, 0);
    const int reps = 10;
    cudaEventRecord(e0);
    for (int w = 0; w < reps; w++) dgemm_launch_streamk<C>(g, G, sk, epi, 0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / reps;
    printf("{\"variant\": \"%s\", \"occ\": %d, \"G\": %d, \"us\": %.1f, \"GBs\": %.0f, \"relerr\": %.2e}\n", name, occ_req, G,
           us, (double)M * K * 8 / us / 1e3, md / mr);
    cudaFree(sk.ws); cudaFree(sk.counters);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int M = 16384, N = 8, K = 16384;
    double *A, *B, *C, *Cr;
    CK(cudaMalloc(&A, (size_t)M * K * 8)); CK(cudaMalloc(&B, (size_t)(N + 64) * K * 8));
    CK(cudaMalloc(&C, (size_t)M * N * 8)); CK(cudaMalloc(&Cr, (size_t)M * N * 8));
    fill<<<1184, 256>>>(A, (size_t)M * K, 1); fill<<<1184, 256>>>(B, (size_t)(N + 64) * K, 2);
    CK(cudaDeviceSynchronize());
    {   // reference: the library's current configuration
        using C0 = DgemmCfg<128, 8, 16, 4, 1, 4, 2>;
        DgemmProblem g{M, N, K, A, K, B, K};
        StoreEpi epi{Cr, M};
        const int G = dgemm_streamk_grid<C0>(M, N, K, sms, 2);
        StreamK sk{};
        CK(cudaMalloc(&sk.ws, dgemm_streamk_ws_doubles<C0>(M, N, G) * 8));
        CK(cudaMalloc(&sk.counters, (dgemm_tiles<C0>(M, N) + 1) * 4));
        CK(cudaMemset(sk.counters, 0, (dgemm_tiles<C0>(M, N) + 1) * 4));
        cudaFuncSetAttribute(k_dgemm_streamk<C0, StoreEpi>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C0::SMEM);
        CK(dgemm_launch_streamk<C0>(g, G, sk, epi, 0));
        CK(cudaDeviceSynchronize());
    }
    for (int occ : {1, 2, 3, 4}) {
        run<DgemmCfg<128, 8, 16, 4, 1, 4, 2>>("128x8k16_w4_s4", M, N, K, A, B, C, Cr, sms, occ);
        run<DgemmCfg<128, 8, 16, 4, 1, 6, 2>>("128x8k16_w4_s6", M, N, K, A, B, C, Cr, sms, occ);
        run<DgemmCfg<128, 8, 32, 4, 1, 4, 2>>("128x8k32_w4_s4", M, N, K, A, B, C, Cr, sms, occ);
        run<DgemmCfg<128, 8, 32, 4, 1, 6, 1>>("128x8k32_w4_s6", M, N, K, A, B, C, Cr, sms, occ);
        run<DgemmCfg<256, 8, 16, 8, 1, 4, 1>>("256x8k16_w8_s4", M, N, K, A, B, C, Cr, sms, occ);
        run<DgemmCfg<256, 8, 32, 8, 1, 3, 1>>("256x8k32_w8_s3", M, N, K, A, B, C, Cr, sms, occ);
        run<DgemmCfg<64, 8, 32, 2, 1, 4, 4>>("64x8k32_w2_s4", M, N, K, A, B, C, Cr, sms, occ);
        run<DgemmCfg<64, 8, 64, 2, 1, 3, 4>>("64x8k64_w2_s3", M, N, K, A, B, C, Cr, sms, occ);
        run<DgemmCfg<128, 8, 64, 4, 1, 3, 2>>("128x8k64_w4_s3", M, N, K, A, B, C, Cr, sms, occ);
    }
    return 0;
}
