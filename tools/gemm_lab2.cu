// GEMM lab 2 (tool, not product): fixed-overhead decomposition of the config-2 Schur GEMMs.
// Times (a) an empty kernel with the same grid / cluster shape, (b) the split-K tile kernel at
// K = 256 .. 2048 (intercept = per-launch fixed cost), (c) the same inside a CUDA graph.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2211_15308_b200/csrc/dgemm_tile.cuh"
using namespace dd;
struct StoreEpi {
    double* C; int ldc;
    __device__ void operator()(int, int row, int col, double v) const { C[row + (size_t)col * ldc] = v; }
};
struct NullEpi {
    double* C;
    __device__ void operator()(int, int row, int col, double v) const { if (v == 12345.678) C[0] = v; }
};
__global__ void k_empty(int* p) { if (p && threadIdx.x == 9999) p[0] = 1; }
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

template <class F>
static double time_us(F f, int reps = 50) {
    for (int i = 0; i < 5; i++) f();
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; i++) f();
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e3 / reps;
}
template <class F>
static double time_graph_us(F f, int reps = 50) {
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaGraph_t g; cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    for (int i = 0; i < reps; i++) f(s);
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e3 / reps;
}
int main() {
    using C = DgemmCfg<64, 64, 16, 2, 2, 4, 2>;
    const int M = 1023, N = 256, Kmax = 2048;
    std::vector<double> h((size_t)1024 * Kmax);
    for (auto& v : h) v = rand() / (double)RAND_MAX - 0.5;
    double *A, *B, *Cm;
    CK(cudaMalloc(&A, h.size() * 8)); CK(cudaMalloc(&B, (size_t)256 * Kmax * 8)); CK(cudaMalloc(&Cm, (size_t)M * N * 8));
    CK(cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(B, h.data(), (size_t)256 * Kmax * 8, cudaMemcpyHostToDevice));
    for (int sk : {1, 4}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(64, sk, 1); cfg.blockDim = dim3(128, 1, 1); cfg.dynamicSmemBytes = C::SMEM;
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = sk; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = sk > 1 ? 1 : 0;
        CK(cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM));
        double te = time_us([&] { cudaLaunchKernelEx(&cfg, k_empty, (int*)nullptr); });
        double tg = time_graph_us([&](cudaStream_t s) { cudaLaunchConfig_t c2 = cfg; c2.stream = s; cudaLaunchKernelEx(&c2, k_empty, (int*)nullptr); });
        printf("{\"what\": \"empty\", \"splitk\": %d, \"us\": %.2f, \"graph_us\": %.2f}\n", sk, te, tg);
    }
    for (int sk : {1, 2, 4}) {
        for (int K : {64 * sk, 256, 512, 1024, 2048}) {
            DgemmProblem g{M, N, K, A, Kmax, B, Kmax};
            double t = time_us([&] { dgemm_launch<C>(g, sk, StoreEpi{Cm, M}, 0); });
            double tn = time_us([&] { dgemm_launch<C>(g, sk, NullEpi{Cm}, 0); });
            double tg = time_graph_us([&](cudaStream_t s) { dgemm_launch<C>(g, sk, StoreEpi{Cm, M}, s); });
            printf("{\"what\": \"tile\", \"splitk\": %d, \"K\": %d, \"us\": %.2f, \"null_epi_us\": %.2f, \"graph_us\": %.2f, \"tflops\": %.2f}\n",
                   sk, K, t, tn, tg, 2.0 * M * N * K / t / 1e6);
        }
    }
    return 0;
}
