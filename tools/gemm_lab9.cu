// GEMM lab 9 (tool, not product): the config-2 grouped shape (1023 x 1023 per group, 4 groups x 64
// columns) under cluster split-K tile shapes.
// (from lab 8:) the config-5 grouped shape (2047 x 2047 per group, 16 groups x 32
// columns) under the library decompositions vs lab 7's warp-specialised kernel.
// GEMM lab 7 (tool, not product): a warp-specialised DMMA tile GEMM for the grouped Schur shape —
// one producer warp streams the A / B k-stages into the padded shared-memory ring with cp.async and
// signals a per-stage mbarrier (cp.async.mbarrier.arrive.noinc); four consumer warps wait on it,
// run the m16n8k4 DMMA fragments and release the stage on a second mbarrier.  No block barrier in
// the main loop; persistent CTAs walk the output tiles.  Compared with the library's tile kernel
// (k_dgemm_tile<CfgG4, S = 1>, all warps load + compute, __syncthreads per stage) on the same
// grouped problem.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2211_15308_b200/csrc/dgemm_tile.cuh"

using namespace dd;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)

struct StoreEpi {
    double* C; int ldc;
    __device__ void operator()(int, int row, int col, double v) const { C[row + (size_t)col * ldc] = v; }
};

__global__ void fill(double* p, size_t n, unsigned seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned h = (unsigned)(i * 2654435761u) ^ seed;
        h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
        p[i] = (h & 0xffff) / 65536.0 - 0.5;
    }
}

__device__ __forceinline__ void mbar_init(unsigned long long* b, int count) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(b));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(b));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_cp_arrive(unsigned long long* b) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(b));
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
    const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(b));
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra W;\n}" ::"r"(a), "r"(parity) : "memory");
}

template <int BM, int BN, int BK, int ST>
struct WsCfg {
    static constexpr int LDS = BK + 4;
    static constexpr int CW = 4;                             // consumer warps (BM / 32 rows each? -> WM x WN)
    static constexpr int WM = BM / 32, WN = (CW / WM);       // warp grid over the tile
    static constexpr int TM = BM / WM, TN = BN / WN, MI = TM / 16, NI = TN / 8;
    static constexpr int THREADS = (CW + 1) * 32;
    static constexpr size_t SMEM = size_t(ST) * (BM + BN) * LDS * sizeof(double) + 2 * ST * sizeof(unsigned long long);
};

template <class C, int ST>
__global__ void __launch_bounds__(C::THREADS, 1) k_ws(DgemmProblem g, StoreEpi epi, int tiles_m, int ntiles) {
    extern __shared__ __align__(16) double smem[];
    constexpr int BM = C::WM * C::TM, BN = C::WN * C::TN, BK = C::LDS - 4, LDS = C::LDS;
    double* As = smem;
    double* Bs = smem + ST * BM * LDS;
    unsigned long long* full = reinterpret_cast<unsigned long long*>(Bs + ST * BN * LDS);
    unsigned long long* empty = full + ST;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < ST; s++) { mbar_init(&full[s], 32); mbar_init(&empty[s], C::CW); }
    }
    __syncthreads();
    const int ktiles = g.K / BK;
    if (warp == C::CW) {
        // ---------------- producer warp
        int kt_all = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int m0 = (t % tiles_m) * BM, n0 = (t / tiles_m) * BN;
            int grp = g.col_group[n0];
            const double* A = g.A + (size_t)grp * g.sG;
            for (int kt = 0; kt < ktiles; kt++, kt_all++) {
                const int s = kt_all % ST;
                if (kt_all >= ST) mbar_wait(&empty[s], ((kt_all / ST) - 1) & 1);
                double* as = As + s * BM * LDS;
                double* bs = Bs + s * BN * LDS;
                const int k0 = kt * BK;
                for (int c = lane; c < BM * BK / 2; c += 32) {
                    const int row = c / (BK / 2), kc = (c % (BK / 2)) * 2;
                    dg_cp_async16(&as[row * LDS + kc], A + (size_t)(m0 + row) * g.lda + k0 + kc);
                }
                for (int c = lane; c < BN * BK / 2; c += 32) {
                    const int row = c / (BK / 2), kc = (c % (BK / 2)) * 2;
                    dg_cp_async16(&bs[row * LDS + kc], g.B + (size_t)(n0 + row) * g.ldb + k0 + kc);
                }
                mbar_cp_arrive(&full[s]);
            }
        }
        asm volatile("cp.async.wait_all;\n" ::);
        return;
    }
    // ---------------- consumer warps
    const int wm = warp % C::WM, wn = warp / C::WM, gq = lane >> 2, tq = lane & 3;
    int kt_all = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int m0 = (t % tiles_m) * BM, n0 = (t / tiles_m) * BN;
        double acc[C::MI][C::NI][4];
#pragma unroll
        for (int i = 0; i < C::MI; i++)
#pragma unroll
            for (int j = 0; j < C::NI; j++) acc[i][j][0] = acc[i][j][1] = acc[i][j][2] = acc[i][j][3] = 0.0;
        for (int kt = 0; kt < ktiles; kt++, kt_all++) {
            const int s = kt_all % ST;
            mbar_wait(&full[s], (kt_all / ST) & 1);
            const double* as = As + s * BM * LDS + (wm * C::TM + gq) * LDS + tq;
            const double* bs = Bs + s * BN * LDS + (wn * C::TN + gq) * LDS + tq;
#pragma unroll
            for (int kk = 0; kk < BK; kk += 4) {
                double a[C::MI][2], b[C::NI];
#pragma unroll
                for (int mi = 0; mi < C::MI; mi++) { a[mi][0] = as[(mi * 16) * LDS + kk]; a[mi][1] = as[(mi * 16 + 8) * LDS + kk]; }
#pragma unroll
                for (int ni = 0; ni < C::NI; ni++) b[ni] = bs[(ni * 8) * LDS + kk];
#pragma unroll
                for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
                    for (int ni = 0; ni < C::NI; ni++) dg_mma(acc[mi][ni], a[mi][0], a[mi][1], b[ni]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        }
#pragma unroll
        for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
            for (int ni = 0; ni < C::NI; ni++)
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int row = m0 + wm * C::TM + mi * 16 + gq + (q >> 1) * 8;
                    const int col = n0 + wn * C::TN + ni * 8 + tq * 2 + (q & 1);
                    if (row < g.M && col < g.N) epi(0, row, col, acc[mi][ni][q]);
                }
    }
}

template <int BM, int BN, int BK, int ST>
void run_ws(const char* name, const DgemmProblem& g, double* C, const double* Cref, int sms, int occ) {
    using Cf = WsCfg<BM, BN, BK, ST>;
    auto kern = k_ws<Cf, ST>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cf::SMEM));
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, Cf::THREADS, Cf::SMEM);
    if (o < occ) { printf("{\"variant\": \"%s\", \"skip\": \"occupancy %d\"}\n", name, o); return; }
    const int tiles_m = (g.M + BM - 1) / BM, ntiles = tiles_m * (g.N / BN);
    const int G = std::min(ntiles, sms * occ);
    StoreEpi epi{C, g.M};
    kern<<<G, Cf::THREADS, Cf::SMEM>>>(g, epi, tiles_m, ntiles);
    CK(cudaDeviceSynchronize());
    std::vector<double> h((size_t)g.M * g.N), r((size_t)g.M * g.N);
    CK(cudaMemcpy(h.data(), C, h.size() * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(r.data(), Cref, r.size() * 8, cudaMemcpyDeviceToHost));
    double md = 0, mr = 0;
    for (size_t j = 0; j < h.size(); j++) { md = fmax(md, fabs(h[j] - r[j])); mr = fmax(mr, fabs(r[j])); }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int reps = 10;
    cudaEventRecord(e0);
    for (int w = 0; w < reps; w++) kern<<<G, Cf::THREADS, Cf::SMEM>>>(g, epi, tiles_m, ntiles);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / reps;
    printf("{\"variant\": \"%s\", \"occ\": %d, \"G\": %d, \"us\": %.1f, \"TFs\": %.2f, \"relerr\": %.2e}\n", name, occ, G, us,
           2.0 * g.M * g.N * g.K / us / 1e6, md / mr);
}


template <class C0>
void run_lib(const char* name, const DgemmProblem& g, double* C, int splitk, int sms, bool sk_mode) {
    StoreEpi epi{C, g.M};
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int reps = 20;
    float ms = 0;
    if (sk_mode) {
        const int G = dgemm_streamk_grid<C0>(g.M, g.N, g.K, sms, 2);
        StreamK sk{};
        CK(cudaMalloc(&sk.ws, dgemm_streamk_ws_doubles<C0>(g.M, g.N, G) * 8));
        CK(cudaMalloc(&sk.counters, (dgemm_tiles<C0>(g.M, g.N) + 1) * 4));
        CK(cudaMemset(sk.counters, 0, (dgemm_tiles<C0>(g.M, g.N) + 1) * 4));
        cudaFuncSetAttribute(k_dgemm_streamk<C0, StoreEpi>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C0::SMEM);
        CK(dgemm_launch_streamk<C0>(g, G, sk, epi, 0));
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int w = 0; w < reps; w++) dgemm_launch_streamk<C0>(g, G, sk, epi, 0);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
        cudaFree(sk.ws); cudaFree(sk.counters);
    } else {
        CK(dgemm_launch<C0>(g, splitk, epi, 0));
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int w = 0; w < reps; w++) dgemm_launch<C0>(g, splitk, epi, 0);
        cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / reps;
    printf("{\"variant\": \"%s\", \"us\": %.1f, \"TFs\": %.2f}\n", name, us, 2.0 * g.M * g.N * g.K / us / 1e6);
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int M = 1023, NG = 4, N = 64 * NG, K = 1024, lda = 1024;
    double *A, *B, *C, *Cr;
    int* cg;
    CK(cudaMalloc(&A, (size_t)NG * 1024 * lda * 8)); CK(cudaMalloc(&B, (size_t)(N + 64) * K * 8));
    CK(cudaMalloc(&C, (size_t)M * N * 8)); CK(cudaMalloc(&Cr, (size_t)M * N * 8));
    CK(cudaMalloc(&cg, N * 4));
    std::vector<int> h(N);
    for (int c = 0; c < N; c++) h[c] = c / 64;
    CK(cudaMemcpy(cg, h.data(), N * 4, cudaMemcpyHostToDevice));
    fill<<<1184, 256>>>(A, (size_t)NG * 1024 * lda, 1); fill<<<1184, 256>>>(B, (size_t)(N + 64) * K, 2);
    CK(cudaDeviceSynchronize());
    DgemmProblem g{M, N, K, A, lda, B, K};
    g.col_group = cg; g.n_group = NG; g.sG = (long long)1024 * lda;
    // warm L2 like the product (the 4 H_p = 33.5 MB stay L2-resident across PCG iterations)
    run_lib<DgemmCfg<128, 32, 16, 4, 1, 3, 2>>("lib_128x32_s3_S4 (product cfg2)", g, C, 4, sms, false);
    run_lib<DgemmCfg<128, 32, 16, 4, 1, 3, 2>>("lib_128x32_s3_S2", g, C, 2, sms, false);
    run_lib<DgemmCfg<128, 32, 16, 4, 1, 3, 2>>("lib_128x32_s3_S8", g, C, 8, sms, false);
    run_lib<DgemmCfg<128, 32, 16, 4, 1, 4, 2>>("lib_128x32_s4_S4", g, C, 4, sms, false);
    run_lib<DgemmCfg<64, 64, 16, 2, 2, 4, 3>>("lib_64x64_s4_S4", g, C, 4, sms, false);
    run_lib<DgemmCfg<64, 64, 16, 2, 2, 4, 3>>("lib_64x64_s4_S2", g, C, 2, sms, false);
    run_lib<DgemmCfg<64, 64, 16, 2, 2, 3, 3>>("lib_64x64_s3_S4", g, C, 4, sms, false);
    run_lib<DgemmCfg<128, 64, 16, 4, 2, 3, 1>>("lib_128x64_s3_S4_w8", g, C, 4, sms, false);
    run_lib<DgemmCfg<128, 64, 16, 4, 2, 3, 1>>("lib_128x64_s3_S8_w8", g, C, 8, sms, false);
    run_lib<DgemmCfg<64, 64, 16, 2, 2, 4, 3>>("lib_64x64_s4_S8", g, C, 8, sms, false);
    run_lib<DgemmCfg<128, 32, 16, 4, 1, 4, 2>>("lib_streamk_128x32", g, C, 0, sms, true);
    return 0;
}
