// GEMM lab 4 (tool): cluster stream-K (k_dgemm_csk) vs cluster split-K (k_dgemm_tile) on the
// config-2 Schur shapes; correctness against cuBLAS; back-to-back launches inside a CUDA graph.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2211_15308_b200/csrc/dgemm_tile.cuh"
using namespace dd;

// Measured on B200 (round 1): slower than k_dgemm_tile's cluster split-K on the config-2 shapes
// (K1 25.5 vs 22.3 us, K2 45.1 vs 40.8 us at the best NC) — the cross-cluster fix-ups and the
// 71-cluster residency limit cost more than the balance gains; kept here as lab evidence.
namespace dd {
// -------------------------------------------------------------------------- cluster stream-K
// Balanced split-K for problems whose tile count does not fill the GPU evenly (config 2:
// 64 output tiles on 148 SMs x 2 slots).  NC clusters of S CTAs (NC S = resident slots) take
// equal ranges of the (tile, k-tile) units, U/NC each; a cluster range covers a few tile
// segments.  For each segment the S CTAs split its k-tiles evenly, run the DMMA main loop and
// reduce over DSMEM exactly like k_dgemm_tile (push into the owner's buffer, one cluster barrier);
// CTA `rank` then owns accumulator registers r ≡ rank (mod S).  A tile covered by one cluster
// gets its epilogue there; a tile cut by cluster boundaries is assembled from its parts in a
// global workspace: each part's quarter is parked, a per-(tile, quarter) counter elects the
// last arriver, which sums the parts in part order (fixed => bitwise deterministic).
struct ClusterSK {
    double* ws;       // [slots][BM*BN] parts, slot = cfirst(t) + t + part
    int* counters;    // [tiles * S], zero on entry, reset by the reducing CTA
    int NC;           // clusters in the grid (gridDim.x)
};

__device__ __forceinline__ void cl_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <class C, class Epi, int S>
__global__ void __launch_bounds__(C::THREADS, C::MINB) k_dgemm_csk(DgemmProblem g, Epi epi, ClusterSK cs) {
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + C::STAGES * C::BM * C::LDS;
    __shared__ int s_last;
    constexpr int JP = (C::NREG + S - 1) / S;
    double* red = smem + C::SMEM_PIPE / sizeof(double);
    const int tiles_m = (g.M + C::BM - 1) / C::BM;
    const int tiles = tiles_m * ((g.N + C::BN - 1) / C::BN);
    const int KT = g.K / C::BK;
    const long long U = (long long)tiles * KT;
    const int cid = blockIdx.x, rank = blockIdx.y;
    const long long u0 = (long long)cid * U / cs.NC, u1 = (long long)(cid + 1) * U / cs.NC;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = warp % C::WM, wn = warp / C::WM;
    const int gq = lane >> 2, tq = lane & 3;
    const unsigned lred = static_cast<unsigned>(__cvta_generic_to_shared(red));
    unsigned rbase[S];
#pragma unroll
    for (int o = 0; o < S; o++) asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbase[o]) : "r"(lred), "r"(o));

    pdl_wait();
    pdl_launch_dependents();
    long long u = u0;
    bool first = true;
    while (u < u1) {
        const int t = (int)(u / KT);
        const int ks = (int)(u % KT);
        const int ke = (int)min((long long)KT, (long long)ks + (u1 - u));
        const int m0 = (t % tiles_m) * C::BM;
        const int n0 = (t / tiles_m) * C::BN;
        const int len = ke - ks;
        const int kt0 = ks + (rank * len) / S;
        const int nkt = ks + ((rank + 1) * len) / S - kt0;

        double acc[C::MI][C::NI][4];
#pragma unroll
        for (int i = 0; i < C::MI; i++)
#pragma unroll
            for (int j = 0; j < C::NI; j++)
#pragma unroll
                for (int r = 0; r < 4; r++) acc[i][j][r] = 0.0;
        __syncthreads();   // previous segment's pipeline reads are finished
#pragma unroll
        for (int s = 0; s < C::STAGES - 1; s++) {
            if (s < nkt) dg_load_stage<C>(As + s * C::BM * C::LDS, Bs + s * C::BN * C::LDS, g.A, g.lda, g.B, g.ldb, m0, n0,
                                          (kt0 + s) * C::BK, tid);
            dg_cp_commit();
        }
        for (int it = 0; it < nkt; it++) {
            dg_cp_wait<C::STAGES - 2>();
            __syncthreads();
            const int nk = it + C::STAGES - 1;
            if (nk < nkt)
                dg_load_stage<C>(As + (nk % C::STAGES) * C::BM * C::LDS, Bs + (nk % C::STAGES) * C::BN * C::LDS, g.A,
                                 g.lda, g.B, g.ldb, m0, n0, (kt0 + nk) * C::BK, tid);
            dg_cp_commit();
            const double* as = As + (it % C::STAGES) * C::BM * C::LDS + (wm * C::TM + gq) * C::LDS + tq;
            const double* bs = Bs + (it % C::STAGES) * C::BN * C::LDS + (wn * C::TN + gq) * C::LDS + tq;
#pragma unroll
            for (int kk = 0; kk < C::BK; kk += 4) {
                double a[C::MI][2], b[C::NI];
#pragma unroll
                for (int mi = 0; mi < C::MI; mi++) {
                    a[mi][0] = as[(mi * 16) * C::LDS + kk];
                    a[mi][1] = as[(mi * 16 + 8) * C::LDS + kk];
                }
#pragma unroll
                for (int ni = 0; ni < C::NI; ni++) b[ni] = bs[(ni * 8) * C::LDS + kk];
#pragma unroll
                for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
                    for (int ni = 0; ni < C::NI; ni++) dg_mma(acc[mi][ni], a[mi][0], a[mi][1], b[ni]);
            }
        }
        dg_cp_wait<0>();
        // the previous segment's reduction buffer must be read out everywhere before new pushes
        if (!first) cl_barrier();
        first = false;
#pragma unroll
        for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
            for (int ni = 0; ni < C::NI; ni++)
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int r = (mi * C::NI + ni) * 4 + q;
                    const unsigned dst = rbase[r % S] + (unsigned)(((rank * JP + r / S) * C::THREADS + tid) * sizeof(double));
                    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(dst), "d"(acc[mi][ni][q]) : "memory");
                }
        cl_barrier();
        double v[JP];
#pragma unroll
        for (int j = 0; j < JP; j++) v[j] = 0.0;
#pragma unroll
        for (int q = 0; q < S; q++)
#pragma unroll
            for (int j = 0; j < JP; j++)
                if (rank + j * S < C::NREG) v[j] += red[(q * JP + j) * C::THREADS + tid];

        bool emit = true;
        if (!(ks == 0 && ke == KT)) {
            // tile cut by cluster boundaries: park this part's quarter, last arriver assembles
            const long long tu0 = (long long)t * KT;
            auto cl_of = [&](long long uu) {
                int c = (int)((uu * cs.NC) / U);
                while (c + 1 < cs.NC && (long long)(c + 1) * U / cs.NC <= uu) c++;
                while (c > 0 && (long long)c * U / cs.NC > uu) c--;
                return c;
            };
            const int cfirst = cl_of(tu0), clast = cl_of(tu0 + KT - 1);
            const int nparts = clast - cfirst + 1;
            const int part = cid - cfirst;
            double* base = cs.ws + ((size_t)(cfirst + t)) * (C::BM * C::BN);
            double* mine = base + (size_t)part * (C::BM * C::BN);
#pragma unroll
            for (int j = 0; j < JP; j++)
                if (rank + j * S < C::NREG) __stcg(&mine[(rank + j * S) * C::THREADS + tid], v[j]);
            __threadfence();
            __syncthreads();
            if (tid == 0) s_last = (atomicAdd(&cs.counters[t * S + rank], 1) == nparts - 1);
            __syncthreads();
            emit = s_last;
            if (emit) {
                __threadfence();
                double sum[JP];
#pragma unroll
                for (int j = 0; j < JP; j++) sum[j] = 0.0;
                for (int pp = 0; pp < nparts; pp++) {
                    if (pp == part) {
#pragma unroll
                        for (int j = 0; j < JP; j++) sum[j] += v[j];
                    } else {
                        const double* src = base + (size_t)pp * (C::BM * C::BN);
#pragma unroll
                        for (int j = 0; j < JP; j++)
                            if (rank + j * S < C::NREG) sum[j] += __ldcg(&src[(rank + j * S) * C::THREADS + tid]);
                    }
                }
#pragma unroll
                for (int j = 0; j < JP; j++) v[j] = sum[j];
                if (tid == 0) cs.counters[t * S + rank] = 0;
            }
        }
        if (emit) {
#pragma unroll
            for (int j = 0; j < JP; j++) {
                const int r = rank + j * S;
                if (r < C::NREG) {
                    int row, col;
                    dg_coord<C>(r, tid, row, col);
                    row += m0; col += n0;
                    if (row < g.M && col < g.N) epi(0, row, col, v[j]);
                }
            }
        }
        u += len;
    }
    cl_barrier();   // no CTA leaves while a cluster peer may still push into its buffer
}

template <class C, int S>
inline size_t dgemm_csk_ws_doubles(int M, int N, int NC) {
    const size_t tiles = size_t((M + C::BM - 1) / C::BM) * size_t((N + C::BN - 1) / C::BN);
    return (size_t(NC) + 2 * tiles + 2) * C::BM * C::BN;
}

template <class C, class Epi, int S>
inline cudaError_t dgemm_launch_csk(const DgemmProblem& g, int NC, const ClusterSK& cs, const Epi& epi, cudaStream_t st,
                                    bool pdl) {
    constexpr size_t smem = dg_tile_smem<C, S>();
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_dgemm_csk<C, Epi, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        if (smem > 100 * 1024) cudaFuncSetAttribute(k_dgemm_csk<C, Epi, S>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr = true;
    }
    if (g.M <= 0 || g.N <= 0) return cudaSuccess;
    ClusterSK c2 = cs;
    c2.NC = NC;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(NC, S, 1);
    cfg.blockDim = dim3(C::THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = S;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    dg_set_pdl(cfg, at, pdl);
    return cudaLaunchKernelEx(&cfg, k_dgemm_csk<C, Epi, S>, g, epi, c2);
}

}  // namespace dd
struct StoreEpi {
    double* C; int ldc;
    __device__ void operator()(int, int row, int col, double v) const { C[row + (size_t)col * ldc] = v; }
};
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1); } } while (0)
template <class F>
static double time_graph_us(F f, int reps = 40) {
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (int i = 0; i < 3; i++) f(s);
    cudaStreamSynchronize(s);
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
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cublasHandle_t hb; cublasCreate(&hb);
    struct Sh { int M, N, K; } shapes[] = {{1023, 256, 1024}, {1023, 256, 2048}, {2047, 512, 2048}, {1023, 200, 1024}, {300, 37, 512}};
    for (auto sh : shapes) {
        const int M = sh.M, N = sh.N, K = sh.K;
        const int Mp = (M + 255) / 256 * 256, Np = (N + 255) / 256 * 256;
        std::vector<double> h((size_t)std::max(Mp, Np) * K);
        for (auto& v : h) v = rand() / (double)RAND_MAX - 0.5;
        double *A, *B, *Cm, *Cr;
        CK(cudaMalloc(&A, (size_t)Mp * K * 8)); CK(cudaMalloc(&B, (size_t)Np * K * 8));
        CK(cudaMalloc(&Cm, (size_t)M * N * 8)); CK(cudaMalloc(&Cr, (size_t)M * N * 8));
        CK(cudaMemcpy(A, h.data(), (size_t)Mp * K * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(B, h.data(), (size_t)Np * K * 8, cudaMemcpyHostToDevice));
        const double one = 1.0, zero = 0.0;
        cublasDgemm(hb, CUBLAS_OP_T, CUBLAS_OP_N, M, N, K, &one, A, K, B, K, &zero, Cr, M);
        DgemmProblem g{M, N, K, A, K, B, K};
        StoreEpi epi{Cm, M};
        std::vector<double> hc((size_t)M * N), hr((size_t)M * N);
        CK(cudaMemcpy(hr.data(), Cr, hr.size() * 8, cudaMemcpyDeviceToHost));
        auto relerr = [&]() {
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(hc.data(), Cm, hc.size() * 8, cudaMemcpyDeviceToHost));
            double md = 0, mr = 0;
            for (size_t j = 0; j < hc.size(); j++) { md = fmax(md, fabs(hc[j] - hr[j])); mr = fmax(mr, fabs(hr[j])); }
            return md / mr;
        };
        for (int sk : {2, 4}) {
            CK(cudaMemset(Cm, 0, (size_t)M * N * 8));
            CK(dgemm_launch<C>(g, sk, epi, 0));
            double e = relerr();
            double t = time_graph_us([&](cudaStream_t s) { dgemm_launch<C>(g, sk, epi, s); });
            printf("{\"kernel\": \"tile\", \"M\": %d, \"N\": %d, \"K\": %d, \"S\": %d, \"us\": %.2f, \"tflops\": %.2f, \"relerr\": %.1e}\n",
                   M, N, K, sk, t, 2.0 * M * N * K / t / 1e6, e);
        }
        int maxc = 0;
        {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(74, 4, 1); cfg.blockDim = dim3(C::THREADS, 1, 1);
            cfg.dynamicSmemBytes = dg_tile_smem<C, 4>();
            cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 1; at[0].val.clusterDim.y = 4; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            cudaFuncSetAttribute(k_dgemm_csk<C, StoreEpi, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cfg.dynamicSmemBytes);
            CK(cudaOccupancyMaxActiveClusters(&maxc, k_dgemm_csk<C, StoreEpi, 4>, &cfg));
            printf("{\"max_active_clusters\": %d}\n", maxc);
        }
        for (int NC : {maxc, maxc - 1, 64, 56}) {
            ClusterSK cs{};
            CK(cudaMalloc(&cs.ws, dgemm_csk_ws_doubles<C, 4>(M, N, NC) * 8));
            const int tiles = dgemm_tiles<C>(M, N);
            CK(cudaMalloc(&cs.counters, tiles * 4 * 4));
            CK(cudaMemset(cs.counters, 0, tiles * 4 * 4));
            CK(cudaMemset(Cm, 0, (size_t)M * N * 8));
            CK((dgemm_launch_csk<C, StoreEpi, 4>(g, NC, cs, epi, 0, false)));
            double e = relerr();
            // determinism: a second run is bitwise equal
            std::vector<double> first = hc;
            CK((dgemm_launch_csk<C, StoreEpi, 4>(g, NC, cs, epi, 0, false)));
            relerr();
            bool same = first == hc;
            double t = time_graph_us([&](cudaStream_t s) { dgemm_launch_csk<C, StoreEpi, 4>(g, NC, cs, epi, s, false); });
            printf("{\"kernel\": \"csk\", \"M\": %d, \"N\": %d, \"K\": %d, \"NC\": %d, \"us\": %.2f, \"tflops\": %.2f, \"relerr\": %.1e, \"bitwise_repeat\": %d}\n",
                   M, N, K, NC, t, 2.0 * M * N * K / t / 1e6, e, same ? 1 : 0);
            cudaFree(cs.ws); cudaFree(cs.counters);
        }
        cudaFree(A); cudaFree(B); cudaFree(Cm); cudaFree(Cr);
    }
    return 0;
}
