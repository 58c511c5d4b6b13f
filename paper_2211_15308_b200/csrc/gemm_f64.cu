// FP64 tensor-core GEMMs of the Schur apply:
//   K1  T' = (K_c s) ∘ (S_dst X)  and  Zlow = γ_c X     (EPI_SCHUR_DST)
//   K2  Y  = [S_dst | F] [T' ; γX]                        (EPI_STORE)
// on the DMMA tile template of dgemm_tile.cuh.  Two work decompositions, picked per launch from
// the work per CTA (tools/gemm_lab.cu measurements, profiles/):
//   * stream-K over 2 CTAs/SM when every CTA gets >= 64 (tile, k-tile) units — balanced to
//     within one unit on any shape (large configs: 30-32 TFLOP/s, cuBLAS-level);
//   * cluster split-K (DSMEM reduction) for small problems (config 2), where stream-K's
//     segment fix-ups cost more than the imbalance they remove.
// Both reduce partial sums in a fixed order: results are bitwise reproducible.
#include "dd_internal.h"
#include "dgemm_tile.cuh"

namespace dd {

using CfgC = DgemmCfg<64, 64, 16, 2, 2, 4, 2>;   // cluster split-K: 4-stage ring, 2 CTAs/SM
using CfgS = DgemmCfg<64, 64, 16, 2, 2, 3, 3>;   // stream-K: 3-stage ring, run at 2 CTAs/SM
constexpr int OCC_C = 2, OCC_S = 2;
constexpr int SK_MIN_UNITS = 64;   // below this the segment fix-ups outweigh the balance gain

struct EpiStore {
    double* C; int ldc;
    __device__ __forceinline__ void operator()(int, int row, int col, double v) const { C[row + (size_t)col * ldc] = v; }
};

struct EpiAdd {                         // C = v + D   (D column-major, ldd)
    double* C; int ldc; const double* D; int ldd;
    __device__ __forceinline__ void operator()(int, int row, int col, double v) const {
        C[row + (size_t)col * ldc] = v + D[row + (size_t)col * ldd];
    }
};

struct EpiSchurDst {
    double* C; int ldc;                 // Z top half (T')
    double* Zlow;                       // Z bottom half (γ X), same ldc
    const double* X; int ldx;
    const int* col_param; int n_param;
    const double *Kp, *gp, *s;
    __device__ __forceinline__ void operator()(int, int row, int col, double v) const {
        int p = col_param[col];
        p = p < 0 ? 0 : (p >= n_param ? n_param - 1 : p);
        C[row + (size_t)col * ldc] = Kp[p] * s[row] * v;
        Zlow[row + (size_t)col * ldc] = gp[p] * X[row + (size_t)col * ldx];
    }
};

int gemm_tiles(int M, int N) { return dgemm_tiles<CfgC>(M, N); }

static bool use_streamk(int M, int N, int K, int num_sms) {
    const long long U = (long long)dgemm_tiles<CfgS>(M, N) * (K / CfgS::BK);
    return U / ((long long)num_sms * OCC_S) >= SK_MIN_UNITS;
}

int gemm_pick_splitk(int M, int N, int K, int num_sms) {
    if (use_streamk(M, N, K, num_sms)) return 0;    // 0 = stream-K
    return dgemm_pick_splitk<CfgC>(M, N, K, num_sms, OCC_C);
}

size_t gemm_ws_doubles(int M, int N, int num_sms) {
    return dgemm_streamk_ws_doubles<CfgS>(M, N, num_sms * OCC_S);
}

template <class Epi>
static cudaError_t launch(const GemmArgs& a, const Epi& e, cudaStream_t st) {
    DgemmProblem g{a.M, a.N, a.K, a.A, a.lda, a.B, a.ldb};
    g.a_static = a.a_static;
    g.ntl = a.ntl;
    if (a.splitk == 0) {
        StreamK sk{a.ws, a.counters, 0};
        // no PDL here: early-resident CTAs of a stream-K grid land unevenly on the SMs (a third
        // CTA beside the predecessor's two), which breaks the equal-work-per-SM premise (cfg3: -25%)
        return dgemm_launch_streamk<CfgS>(g, dgemm_streamk_grid<CfgS>(a.M, a.N, a.K, a.num_sms, OCC_S), sk, e, st,
                                          false);
    }
    return dgemm_launch<CfgC>(g, a.splitk, e, st, a.pdl != 0);
}

cudaError_t launch_dgemm(const GemmArgs& a, cudaStream_t st) {
    if (a.M <= 0 || a.N <= 0) return cudaSuccess;
    if (a.epi == EPI_STORE) return launch(a, EpiStore{a.C, a.ldc}, st);
    if (a.epi == EPI_ADD) return launch(a, EpiAdd{a.C, a.ldc, a.X, a.ldx}, st);
    return launch(a, EpiSchurDst{a.C, a.ldc, a.Zlow, a.X, a.ldx, a.col_param, a.n_param, a.Kp, a.gp, a.s}, st);
}

}  // namespace dd
