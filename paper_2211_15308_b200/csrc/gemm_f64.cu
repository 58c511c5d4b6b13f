// FP64 tensor-core GEMM for sm_100a: the fast-diagonalisation transforms and the dense
// fractional term of the Schur apply.
//
// tcgen05 has no f64 kind, so FP64 tensor math on B200 is the warp-level DMMA
// (mma.sync.aligned.m16n8k4 .f64, SASS DMMA.8x8x4); measured 37.2 TFLOP/s issue-bound on this
// pool (MEASURED_FP64.json).  Tiles: 64x64x16 per CTA, 4 warps each owning 32x32 (2x4 m16n8k4
// fragments, 32 fp64 accumulators per thread), 4-stage cp.async pipeline, padded smem rows
// (20 doubles) so fragment loads hit 16 distinct bank pairs.  Split-K partials are reduced by
// the last-arriving CTA in fixed split order (bitwise deterministic).
#include "dd_internal.h"

namespace dd {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], const double (&a)[2], double b) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a[0]), "d"(a[1]), "d"(b));
}

__global__ void __launch_bounds__(GEMM_THREADS, 2) k_dgemm(GemmArgs g) {
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + GEMM_STAGES * GEMM_BM * GEMM_LDS;

    const int tiles_m = (g.M + GEMM_BM - 1) / GEMM_BM;
    const int tile = blockIdx.x;
    const int split = blockIdx.y;
    const int m0 = (tile % tiles_m) * GEMM_BM;   // m fastest: co-resident CTAs share B columns in L2
    const int n0 = (tile / tiles_m) * GEMM_BN;
    const int ktiles = g.K / GEMM_BK;
    const int per = (ktiles + g.splitk - 1) / g.splitk;
    const int kt0 = split * per;
    const int nkt = max(0, min(per, ktiles - kt0));

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = warp & 1, wn = warp >> 1;
    const int gq = lane >> 2, tq = lane & 3;

    double acc[2][4][4];
#pragma unroll
    for (int i = 0; i < 2; i++)
#pragma unroll
        for (int j = 0; j < 4; j++)
#pragma unroll
            for (int r = 0; r < 4; r++) acc[i][j][r] = 0.0;

    auto load_stage = [&](int stage, int kt) {
        const int k0 = kt * GEMM_BK;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int c = tid + GEMM_THREADS * j;
            const int row = c >> 3, kc = (c & 7) * 2;
            cp_async16(&As[(stage * GEMM_BM + row) * GEMM_LDS + kc], g.A + (size_t)(m0 + row) * g.lda + k0 + kc);
            cp_async16(&Bs[(stage * GEMM_BN + row) * GEMM_LDS + kc], g.B + (size_t)(n0 + row) * g.ldb + k0 + kc);
        }
    };

#pragma unroll
    for (int s = 0; s < GEMM_STAGES - 1; s++) {
        if (s < nkt) load_stage(s, kt0 + s);
        cp_async_commit();
    }
    for (int it = 0; it < nkt; it++) {
        cp_async_wait<GEMM_STAGES - 2>();
        __syncthreads();
        const int nk = it + GEMM_STAGES - 1;
        if (nk < nkt) load_stage(nk % GEMM_STAGES, kt0 + nk);
        cp_async_commit();
        const double* as = As + (it % GEMM_STAGES) * GEMM_BM * GEMM_LDS;
        const double* bs = Bs + (it % GEMM_STAGES) * GEMM_BN * GEMM_LDS;
#pragma unroll
        for (int kk = 0; kk < GEMM_BK; kk += 4) {
            double a[2][2], b[4];
#pragma unroll
            for (int mi = 0; mi < 2; mi++) {
                const int r = wm * 32 + mi * 16 + gq;
                a[mi][0] = as[r * GEMM_LDS + kk + tq];
                a[mi][1] = as[(r + 8) * GEMM_LDS + kk + tq];
            }
#pragma unroll
            for (int ni = 0; ni < 4; ni++) b[ni] = bs[(wn * 32 + ni * 8 + gq) * GEMM_LDS + kk + tq];
#pragma unroll
            for (int mi = 0; mi < 2; mi++)
#pragma unroll
                for (int ni = 0; ni < 4; ni++) dmma_16x8x4(acc[mi][ni], a[mi], b[ni]);
        }
    }
    cp_async_wait<0>();

    // ---- split-K: deterministic reduction by the last CTA of the tile
    if (g.splitk > 1) {
        __shared__ int s_last;
        double* mine = g.ws + ((size_t)tile * g.splitk + split) * (GEMM_BM * GEMM_BN);
#pragma unroll
        for (int mi = 0; mi < 2; mi++)
#pragma unroll
            for (int ni = 0; ni < 4; ni++)
#pragma unroll
                for (int r = 0; r < 4; r++) __stcg(&mine[((mi * 4 + ni) * 4 + r) * GEMM_THREADS + tid], acc[mi][ni][r]);
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            const int prev = atomicAdd(&g.counters[tile], 1);
            s_last = (prev == g.splitk - 1);
        }
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        const double* base = g.ws + (size_t)tile * g.splitk * (GEMM_BM * GEMM_BN);
#pragma unroll
        for (int mi = 0; mi < 2; mi++)
#pragma unroll
            for (int ni = 0; ni < 4; ni++)
#pragma unroll
                for (int r = 0; r < 4; r++) {
                    const int idx = ((mi * 4 + ni) * 4 + r) * GEMM_THREADS + tid;
                    double v = 0.0;
                    for (int s = 0; s < g.splitk; s++)
                        v += (s == split) ? acc[mi][ni][r] : __ldcg(&base[(size_t)s * (GEMM_BM * GEMM_BN) + idx]);
                    acc[mi][ni][r] = v;
                }
        if (tid == 0) g.counters[tile] = 0;
    }

    // ---- epilogue
#pragma unroll
    for (int mi = 0; mi < 2; mi++)
#pragma unroll
        for (int ni = 0; ni < 4; ni++)
#pragma unroll
            for (int r = 0; r < 4; r++) {
                const int row = m0 + wm * 32 + mi * 16 + gq + (r >> 1) * 8;
                const int col = n0 + wn * 32 + ni * 8 + tq * 2 + (r & 1);
                if (row >= g.M || col >= g.N) continue;
                const double v = acc[mi][ni][r];
                if (g.epi == EPI_STORE) {
                    g.C[row + (size_t)col * g.ldc] = v;
                } else {  // EPI_SCHUR_DST
                    int p = g.col_param[col];
                    p = p < 0 ? 0 : (p >= g.n_param ? g.n_param - 1 : p);
                    g.C[row + (size_t)col * g.ldc] = g.Kp[p] * g.s[row] * v;
                    g.Zlow[row + (size_t)col * g.ldc] = g.gp[p] * g.X[row + (size_t)col * g.ldx];
                }
            }
}

int gemm_tiles(int M, int N) {
    return ((M + GEMM_BM - 1) / GEMM_BM) * ((N + GEMM_BN - 1) / GEMM_BN);
}

int gemm_pick_splitk(int M, int N, int K, int num_sms) {
    // Aim at ~2 resident CTAs per SM while keeping >= 16 k-tiles per split.
    const int tiles = gemm_tiles(M, N);
    const int ktiles = K / GEMM_BK;
    const int target = 2 * num_sms;
    int best = 1;
    double best_eff = 0.0;
    for (int s = 1; s <= 16; s++) {
        if (ktiles / s < 16 && s > 1) break;
        const int ctas = tiles * s;
        const int slots = 2 * num_sms;
        const int waves = (ctas + slots - 1) / slots;
        double eff = double(ctas) / double(waves * slots);
        eff *= 1.0 - 0.02 * (s - 1);   // partial-sum traffic
        if (ctas < target / 2) eff *= 0.5 + 0.5 * double(ctas) / double(target / 2);
        if (eff > best_eff + 1e-9) { best_eff = eff; best = s; }
    }
    return best;
}

size_t gemm_ws_doubles(int M, int N, int splitk) {
    return splitk > 1 ? size_t(gemm_tiles(M, N)) * splitk * GEMM_BM * GEMM_BN : 0;
}

cudaError_t launch_dgemm(const GemmArgs& a, cudaStream_t st) {
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(k_dgemm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GEMM_SMEM);
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    if (a.M <= 0 || a.N <= 0) return cudaSuccess;
    dim3 grid(gemm_tiles(a.M, a.N), a.splitk);
    k_dgemm<<<grid, GEMM_THREADS, GEMM_SMEM, st>>>(a);
    return cudaGetLastError();
}

}  // namespace dd
