// FP64 tensor-core GEMMs of the Schur apply,
// in the three 2D modes of dd_set_schur_mode:
//   grouped    Y[:, c] = H_{p(c)} X[:, c],  H_p = K_p G + γ_p F      (CfgG, A block per 32-column tile)
//   assembled  Y = [F | G] [γX ; KX]                                 (EPI_STORE; RA mode: G (KX) + U, EPI_ADD)
//   factored   K1  T' = (K_c s) ∘ (S_dst X), Zlow = γ_c X  (EPI_SCHUR_DST);  K2  Y = [S_dst | F] [T' ; γX]
// on the DMMA tile template of dgemm_tile.cuh.  Two work decompositions, picked per launch from
// the work per CTA (tools/gemm_lab*.cu measurements, profiles/):
//   * stream-K over 2 CTAs/SM when every CTA gets >= 64 (tile, k-tile) units — balanced to
//     within one unit on any shape (large configs: 30-32 TFLOP/s, cuBLAS-level);
//   * cluster split-K (DSMEM reduction) for small problems (config 2), where stream-K's
//     segment fix-ups cost more than the imbalance they remove.
// Both reduce partial sums in a fixed order: results are bitwise reproducible.
#include <cstdlib>

#include "dd_internal.h"
#include "dgemm_tile.cuh"

namespace dd {

using CfgC = DgemmCfg<64, 64, 16, 2, 2, 4, 2>;   // cluster split-K: 4-stage ring, 2 CTAs/SM
using CfgS = DgemmCfg<64, 64, 16, 2, 2, 3, 3>;   // stream-K: 3-stage ring, run at 2 CTAs/SM
using CfgG = DgemmCfg<128, 32, 16, 4, 1, 3, 2>; // grouped per-parameter GEMM: 32-column tiles (tools/gemm_lab5.cu)
using CfgG4 = DgemmCfg<128, 32, 16, 4, 1, 4, 2>; // grouped stream-K default: 4-stage ring (DD_GROUPED_STAGES=3|4)
constexpr int OCC_C = 2, OCC_S = 2, OCC_G = 2;
static_assert(CfgG::BN == GEMM_BN_GROUPED, "grouped tile width");
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

int gemm_tiles(int M, int N) {
    // grouped: live-tile lists address 64-column tiles, i.e. up to round_up(N, 64) / 32 tiles
    const int a = dgemm_tiles<CfgC>(M, N), b = dgemm_tiles<CfgG>(M, (N + 63) / 64 * 64);
    return a > b ? a : b;
}

static bool use_streamk(int M, int N, int K, int num_sms) {
    const long long U = (long long)dgemm_tiles<CfgS>(M, N) * (K / CfgS::BK);
    return U / ((long long)num_sms * OCC_S) >= SK_MIN_UNITS;
}

int gemm_pick_splitk(int M, int N, int K, int num_sms) {
    if (use_streamk(M, N, K, num_sms)) return 0;    // 0 = stream-K
    return dgemm_pick_splitk<CfgC>(M, N, K, num_sms, OCC_C);
}

int gemm_pick_splitk_grouped(int M, int N, int K, int num_sms) {
    static const bool no_sk = std::getenv("DD_GROUPED_NO_SK") && std::getenv("DD_GROUPED_NO_SK")[0] == '1';
    if (!no_sk) {
        const long long U = (long long)dgemm_tiles<CfgG>(M, N) * (K / CfgG::BK);
        if (U / ((long long)num_sms * OCC_G) >= SK_MIN_UNITS) return 0;   // stream-K
    }
    return dgemm_pick_splitk<CfgG>(M, N, K, num_sms, OCC_G);
}

size_t gemm_ws_doubles(int M, int N, int num_sms) {
    const size_t a = dgemm_streamk_ws_doubles<CfgS>(M, N, num_sms * OCC_S);
    const size_t b = dgemm_streamk_ws_doubles<CfgG>(M, (N + 63) / 64 * 64, num_sms * OCC_G);
    return a > b ? a : b;
}

template <class Epi>
static cudaError_t launch(const GemmArgs& a, const Epi& e, cudaStream_t st) {
    DgemmProblem g{a.M, a.N, a.K, a.A, a.lda, a.B, a.ldb};
    g.a_static = a.a_static;
    g.ntl = a.ntl;
    g.ntl_bn = a.ntl_bn > 0 ? a.ntl_bn : 64;
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
    if (a.grouped) {
        DgemmProblem g{a.M, a.N, a.K, a.A, a.lda, a.B, a.ldb};
        g.ntl = a.ntl;
        g.ntl_bn = a.ntl_bn > 0 ? a.ntl_bn : 64;
        g.a_static = a.a_static;
        g.col_group = a.col_param; g.n_group = a.n_param; g.sG = a.sG; g.mixed = a.mixed;
        g.alt_A = a.alt_A; g.alt_lda = a.alt_lda; g.alt_B = a.alt_B; g.alt_ldb = a.alt_ldb; g.alt_K = a.alt_K;
        if (a.splitk == 0) {
            // stream-K over the live 32-column tiles; the unit count follows the fallback's K too
            StreamK sk{a.ws, a.counters, 0};
            const int G = dgemm_streamk_grid<CfgG>(a.M, a.N, a.K, a.num_sms, OCC_G);
            // 4-stage ring (cfg5 136 -> 130 us, cfg3 165 -> 156 us against 3 stages; 5 stages or 3 CTAs/SM lose)
            static const int stages = std::getenv("DD_GROUPED_STAGES") ? std::atoi(std::getenv("DD_GROUPED_STAGES")) : 4;
            if (stages == 4) return dgemm_launch_streamk<CfgG4>(g, G, sk, EpiStore{a.C, a.ldc}, st, false);
            return dgemm_launch_streamk<CfgG>(g, G, sk, EpiStore{a.C, a.ldc}, st, false);
        }
        return dgemm_launch<CfgG>(g, a.splitk, EpiStore{a.C, a.ldc}, st, a.pdl != 0);
    }
    if (a.epi == EPI_STORE) return launch(a, EpiStore{a.C, a.ldc}, st);
    if (a.epi == EPI_ADD) return launch(a, EpiAdd{a.C, a.ldc, a.X, a.ldx}, st);
    return launch(a, EpiSchurDst{a.C, a.ldc, a.Zlow, a.X, a.ldx, a.col_param, a.n_param, a.Kp, a.gp, a.s}, st);
}

}  // namespace dd
