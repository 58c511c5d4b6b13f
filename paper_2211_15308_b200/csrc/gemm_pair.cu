// Grouped Schur apply from the shared pair (G, F) (sm_100a, FP64 DMMA) — SURVEY §8(a) rows a-2,
// a-3; PAPER.md:44 (S = K S_unit + γ F), 146-148, 178-180 (Eq.(7)):
//
//     Y[:, c] = (K_p G + γ_p F) X[:, c],   p = col_param[c],   G = S_unit = S_dst diag(s) S_dst,
//
// one GEMM with 2 n^2 flops per column, like the grouped mode's per-parameter matrices H_p, but
// without materialising them: every CTA stages the G and F tiles of its rows once and each warp
// forms its own group's A fragments a = g + ρ_p f, ρ_p = γ_p / K_p, in registers (one DFMA per
// fragment element) before the DMMAs; K_p scales the epilogue.  A CTA tile spans NGRP 32-column groups (one warp column
// per group), so each G / F tile feeds NGRP parameter sets; HBM traffic per apply is the pair
// (2 n^2 doubles, L2-resident between the n-tiles that reuse it) instead of n_param H_p blocks.
//
// Work: stream-K over (output tile, k-tile) units (as k_dgemm_streamk: fixed partition, partials
// of cut tiles summed in segment order by the last arriver — bitwise reproducible).  Live-tile
// lists (s.ntl, 32-column tiles) restrict the n-tiles to unconverged groups.  Mixed batches (a
// 32-column tile holding two parameter sets; device flag) compute the assembled product
// Y = F (γ X) + G (K X) from the PCG kernels' operand Z = [γ X ; K X] instead, as a K-range of
// 2 Kpad (first F against the γ half, then G against the K half) — same result, no host check.
#include <cstdlib>

#include "dd_internal.h"
#include "dgemm_tile.cuh"

namespace dd {

template <int BM_, int NGRP_, int WM_, int STAGES_>
struct PairCfg {
    static constexpr int BM = BM_, NGRP = NGRP_, WM = WM_, WN = NGRP_, STAGES = STAGES_;
    static constexpr int BN = 32 * NGRP, BK = 16, LDS = BK + 4;
    static constexpr int THREADS = WM * WN * 32;
    static constexpr int TM = BM / WM, TN = 32, MI = TM / 16, NI = TN / 8, NREG = MI * NI * 4;
    static constexpr int CPR = BK / 2, ACH = BM * CPR, BCH = BN * CPR;
    static constexpr size_t SMEM = size_t(STAGES) * (2 * BM + BN) * LDS * sizeof(double);
    static_assert(TM % 16 == 0, "warp tile");
};
using CfgP = PairCfg<64, 4, 2, 4>;      // 8 warps, 64 x 128 tiles, 4-stage ring (164 KB): 1 CTA / SM
using CfgP2 = PairCfg<64, 2, 2, 3>;     // 4 warps, 64 x 64 tiles, 3-stage ring (92 KB): 2 CTAs / SM

struct PairProblem {
    int M, N, Kpad;                        // N: columns of this call; Kpad: K-dim of G, F (multiple of 16)
    const double *G, *F; int lda;          // row-major, rows readable up to round_up(M, BM)
    const double* X; int ldx;              // column-major Kpad x N (columns readable up to round_up(N, 64))
    const double* Z; int ldz, zhalf;       // mixed fallback: [γ X ; K X] (K half at row zhalf)
    const int* mixed;                      // device flag (nullptr: never mixed)
    const int* col_param; int n_param;
    const double *Kp, *gp;
    const int* ntl;                        // live 32-column tiles [count, ids...] or nullptr
    double* Y; int ldy;
};

template <class C>
__device__ __forceinline__ void pr_load_rows(double* dst, const double* src, int ld, int row0, int k0, int rows, int tid) {
    // rows x BK doubles from a row-major matrix (row0.., k0..) into padded smem rows
    const int nch = rows * C::CPR;
    for (int c = tid; c < nch; c += C::THREADS) {
        const int row = c / C::CPR, kc = (c % C::CPR) * 2;
        dg_cp_async16(&dst[row * C::LDS + kc], src + (size_t)(row0 + row) * ld + k0 + kc);
    }
}

// B tile: NGRP blocks of 32 columns, block w starting at column col0[w] (< 0: absent)
template <class C>
__device__ __forceinline__ void pr_load_b(double* dst, const double* X, int ldx, const int* col0, int k0, int tid) {
#pragma unroll
    for (int j = 0; j < (C::BCH + C::THREADS - 1) / C::THREADS; j++) {
        const int c = tid + C::THREADS * j;
        if (C::BCH % C::THREADS == 0 || c < C::BCH) {
            const int row = c / C::CPR, kc = (c % C::CPR) * 2;
            int cb = col0[0];
#pragma unroll
            for (int w = 1; w < C::NGRP; w++) if ((row >> 5) == w) cb = col0[w];
            if (cb >= 0) dg_cp_async16(&dst[row * C::LDS + kc], X + (size_t)(cb + (row & 31)) * ldx + k0 + kc);
        }
    }
}

template <class C, bool MIX>
__device__ __forceinline__ void pair_tile_loop(const PairProblem& g, double* smem, int m0, const int* col0, int ks, int ke,
                                               int KT, double Kc, double gc, double (&acc)[C::MI][C::NI][4]) {
    constexpr int ST = (2 * C::BM + C::BN) * C::LDS;       // doubles per stage
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = warp % C::WM, wn = warp / C::WM;
    const int gq = lane >> 2, tq = lane & 3;
    const int nkt = ke - ks;
    auto load_stage = [&](int stage, int kt) {
        double* base = smem + stage * ST;
        if constexpr (MIX) {
            // K-range 2 Kpad: F against the γ half of Z, then G against the K half
            const bool second = kt >= KT;
            const int k0 = (second ? kt - KT : kt) * C::BK;
            pr_load_rows<C>(base, second ? g.G : g.F, g.lda, m0, k0, C::BM, tid);
            pr_load_b<C>(base + 2 * C::BM * C::LDS, g.Z + (second ? g.zhalf : 0), g.ldz, col0, k0, tid);
        } else {
            const int k0 = kt * C::BK;
            pr_load_rows<C>(base, g.G, g.lda, m0, k0, C::BM, tid);
            pr_load_rows<C>(base + C::BM * C::LDS, g.F, g.lda, m0, k0, C::BM, tid);
            pr_load_b<C>(base + 2 * C::BM * C::LDS, g.X, g.ldx, col0, k0, tid);
        }
    };
    __syncthreads();   // the previous segment's smem reads are finished
#pragma unroll
    for (int s = 0; s < C::STAGES - 1; s++) {
        if (s < nkt) load_stage(s, ks + s);
        dg_cp_commit();
    }
    bool live = col0[0] >= 0;
#pragma unroll
    for (int w = 1; w < C::NGRP; w++) if (wn == w) live = col0[w] >= 0;
    for (int it = 0; it < nkt; it++) {
        dg_cp_wait<C::STAGES - 2>();
        __syncthreads();
        const int nk = it + C::STAGES - 1;
        if (nk < nkt) load_stage(nk % C::STAGES, ks + nk);
        dg_cp_commit();
        if (!live) continue;                     // absent group column: nothing to multiply (warp-uniform)
        const double* st = smem + (it % C::STAGES) * ST;
        const double* gs = st + (wm * C::TM + gq) * C::LDS + tq;
        const double* fs = gs + C::BM * C::LDS;
        const double* bs = st + 2 * C::BM * C::LDS + (wn * C::TN + gq) * C::LDS + tq;
#pragma unroll
        for (int kk = 0; kk < C::BK; kk += 4) {
            double a[C::MI][2], b[C::NI];
#pragma unroll
            for (int mi = 0; mi < C::MI; mi++) {
                if constexpr (MIX) {
                    a[mi][0] = gs[(mi * 16) * C::LDS + kk];
                    a[mi][1] = gs[(mi * 16 + 8) * C::LDS + kk];
                } else {
                    // (K G + γ F) = K (G + ρ F), ρ = γ / K: one DFMA per element, K applied in the epilogue
                    a[mi][0] = fma(gc, fs[(mi * 16) * C::LDS + kk], gs[(mi * 16) * C::LDS + kk]);
                    a[mi][1] = fma(gc, fs[(mi * 16 + 8) * C::LDS + kk], gs[(mi * 16 + 8) * C::LDS + kk]);
                }
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
}

template <class C>
__device__ __forceinline__ void pair_coord(int r, int tid, int& row, int& col) {
    const int warp = tid >> 5, lane = tid & 31;
    const int wm = warp % C::WM, wn = warp / C::WM;
    const int f = r >> 2, q = r & 3;
    const int mi = f / C::NI, ni = f % C::NI;
    row = wm * C::TM + mi * 16 + (lane >> 2) + (q >> 1) * 8;
    col = wn * C::TN + ni * 8 + (lane & 3) * 2 + (q & 1);    // within the CTA's BN columns
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, C::THREADS <= 128 ? 2 : 1) k_dgemm_pair(PairProblem g, StreamK sk) {
    extern __shared__ __align__(16) double smem[];
    __shared__ int s_last;
    pdl_launch_dependents();
    pdl_wait();
    const bool mix = g.mixed && *g.mixed;
    const int tiles_m = (g.M + C::BM - 1) / C::BM;
    const int nlive = g.ntl ? g.ntl[0] : (g.N + 31) / 32;
    const int tiles_n = (nlive + C::NGRP - 1) / C::NGRP;
    const int tiles = tiles_m * tiles_n;
    const int KT = g.Kpad / C::BK;
    const int KU = mix ? 2 * KT : KT;               // k-tiles per output tile
    const long long U = (long long)tiles * KU;
    const int b = blockIdx.x;
    const long long u0 = sk_unit_begin(b, U, sk.G), u1 = sk_unit_begin(b + 1, U, sk.G);
    const int tid = threadIdx.x;
    const int wn = (tid >> 5) / C::WM;

    long long u = u0;
    while (u < u1) {
        const int t = (int)(u / KU);
        const int ks = (int)(u % KU);
        const int ke = (int)min((long long)KU, (long long)ks + (u1 - u));
        const int m0 = (t % tiles_m) * C::BM;
        const int tn = t / tiles_m;
        int col0[C::NGRP];
#pragma unroll
        for (int w = 0; w < C::NGRP; w++) {
            const int li = tn * C::NGRP + w;
            int c0 = -1;
            if (li < nlive) c0 = (g.ntl ? g.ntl[1 + li] : li) * 32;
            col0[w] = (c0 >= 0 && c0 < g.N) ? c0 : -1;
        }
        int mycol = col0[0];
#pragma unroll
        for (int w = 1; w < C::NGRP; w++) if (wn == w) mycol = col0[w];
        double Kc = 0.0, gc = 0.0;
        if (mycol >= 0) {
            int p = g.col_param[mycol];
            p = p < 0 ? 0 : (p >= g.n_param ? g.n_param - 1 : p);
            Kc = g.Kp[p]; gc = g.gp[p] / Kc;       // K > 0 (dd_setup validates)
            if (mix) Kc = 1.0;                     // mixed: the operand Z carries K and γ
        }
        double acc[C::MI][C::NI][4];
#pragma unroll
        for (int i = 0; i < C::MI; i++)
#pragma unroll
            for (int j = 0; j < C::NI; j++)
#pragma unroll
                for (int r = 0; r < 4; r++) acc[i][j][r] = 0.0;
        if (mix) pair_tile_loop<C, true>(g, smem, m0, col0, ks, ke, KT, Kc, gc, acc);
        else pair_tile_loop<C, false>(g, smem, m0, col0, ks, ke, KT, Kc, gc, acc);

        bool emit = true;
        if (!(ks == 0 && ke == KU)) {
            // segmented tile: park the partial, count arrivals, the last arriver reduces in segment order
            const long long tu0 = (long long)t * KU;
            const int bfirst = sk_cta_of(tu0, U, sk.G);
            const int blast = sk_cta_of(tu0 + KU - 1, U, sk.G);
            const int nseg = blast - bfirst + 1;
            const int seg = b - bfirst;
            double* slot = sk.ws + ((size_t)(bfirst + t) + seg) * (C::BM * C::BN);
#pragma unroll
            for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
                for (int ni = 0; ni < C::NI; ni++)
#pragma unroll
                    for (int q = 0; q < 4; q++) __stcg(&slot[((mi * C::NI + ni) * 4 + q) * C::THREADS + tid], acc[mi][ni][q]);
            __threadfence();
            __syncthreads();
            if (tid == 0) s_last = (atomicAdd(&sk.counters[t], 1) == nseg - 1);
            __syncthreads();
            emit = s_last;
            if (emit) {
                __threadfence();
                const double* base = sk.ws + (size_t)(bfirst + t) * (C::BM * C::BN);
                // every segment, this CTA's own included (parked above), is read back from the
                // workspace and summed into acc in segment order 0, 1, ... (no second register array:
                // the fix-up needs no more registers than the main loop)
#pragma unroll 1
                for (int s2 = 0; s2 < nseg; s2++) {
                    const double* src = base + (size_t)s2 * (C::BM * C::BN) + tid;
#pragma unroll
                    for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
                        for (int ni = 0; ni < C::NI; ni++)
#pragma unroll
                            for (int q = 0; q < 4; q++) {
                                const double v = __ldcg(&src[((mi * C::NI + ni) * 4 + q) * C::THREADS]);
                                acc[mi][ni][q] = s2 == 0 ? v : acc[mi][ni][q] + v;
                            }
                }
                if (tid == 0) sk.counters[t] = 0;
            }
        }
        if (emit && mycol >= 0) {
#pragma unroll
            for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
                for (int ni = 0; ni < C::NI; ni++)
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        int row, col;
                        pair_coord<C>((mi * C::NI + ni) * 4 + q, tid, row, col);
                        row += m0;
                        col = mycol + (col & 31);
                        if (row < g.M && col < g.N) g.Y[row + (size_t)col * g.ldy] = Kc * acc[mi][ni][q];
                    }
        }
        u += ke - ks;
    }
}

// ------------------------------------------------------------------------------------------- host
template <class C>
static int pair_grid(int M, int N, int Kpad, int num_sms, int occ) {
    const long long tiles = (long long)((M + C::BM - 1) / C::BM) * (((N + 31) / 32 + C::NGRP - 1) / C::NGRP);
    // capped by the unit count of a group-aligned call (a mixed call has twice as many): every CTA
    // must own at least one unit, since a cut tile's segment count is a range of consecutive CTAs
    const long long U = tiles * (Kpad / C::BK);
    long long G = (long long)num_sms * occ;
    if (G > U) G = U;
    return (int)(G < 1 ? 1 : G);
}

template <class C>
static size_t pair_ws(int M, int N, int G) {
    const size_t tiles = size_t((M + C::BM - 1) / C::BM) * size_t(((N + 31) / 32 + C::NGRP - 1) / C::NGRP);
    return (size_t(G) + 2 * tiles + 2) * C::BM * C::BN;
}
size_t gemm_pair_ws_doubles(int M, int N, int num_sms) {
    const size_t a = pair_ws<CfgP>(M, N, num_sms), b = pair_ws<CfgP2>(M, N, 2 * num_sms);
    return a > b ? a : b;
}
int gemm_pair_tiles(int M, int N) {
    const int a = ((M + CfgP::BM - 1) / CfgP::BM) * (((N + 31) / 32 + CfgP::NGRP - 1) / CfgP::NGRP);
    const int b = ((M + CfgP2::BM - 1) / CfgP2::BM) * (((N + 31) / 32 + CfgP2::NGRP - 1) / CfgP2::NGRP);
    return a > b ? a : b;
}

template <class C>
static cudaError_t launch_pair_cfg(const PairArgs& a, int occ, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_dgemm_pair<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    PairProblem g{a.M, a.N, a.Kpad, a.G, a.F, a.lda, a.X, a.ldx, a.Z, a.ldz, a.zhalf, a.mixed,
                  a.col_param, a.n_param, a.Kp, a.gp, a.ntl, a.Y, a.ldy};
    StreamK sk{a.ws, a.counters, pair_grid<C>(a.M, a.N, a.Kpad, a.num_sms, occ)};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sk.G, 1, 1);
    cfg.blockDim = dim3(C::THREADS, 1, 1);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    cfg.attrs = at;
    cfg.numAttrs = 0;
    return cudaLaunchKernelEx(&cfg, k_dgemm_pair<C>, g, sk);
}

cudaError_t launch_gemm_pair(const PairArgs& a, cudaStream_t st) {
    if (a.M <= 0 || a.N <= 0) return cudaSuccess;
    // 4-warp CTAs at 2 per SM (cfg5 149 us) beat 8-warp CTAs at 1 per SM (198 us); DD_PAIR_CFG=1 for the latter
    static const int variant = std::getenv("DD_PAIR_CFG") ? std::atoi(std::getenv("DD_PAIR_CFG")) : 2;
    if (variant == 1) return launch_pair_cfg<CfgP>(a, 1, st);
    return launch_pair_cfg<CfgP2>(a, 2, st);
}

}  // namespace dd
