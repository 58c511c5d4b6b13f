// Host-only definition of the libdd handle and shared host helpers (dd_api.cpp, dd3d.cpp).
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "dd_internal.h"

namespace dd {

dd_status set_error(dd_status s, const std::string& msg);

#define DD_CK(expr)                                                                               \
    do {                                                                                          \
        cudaError_t _e = (expr);                                                                  \
        if (_e != cudaSuccess)                                                                    \
            return ::dd::set_error(_e == cudaErrorMemoryAllocation ? DD_ENOMEM : DD_ECUDA,       \
                                   std::string(#expr) + ": " + cudaGetErrorString(_e));          \
    } while (0)

inline int round_up(int a, int b) { return (a + b - 1) / b * b; }

struct EvPair {
    cudaEvent_t a, b;
    int cls;
};

struct GraphKey {
    int ncols;
    const int* colp;
    const double* x;
    double rtol;
    int maxit, norm_kind;
    const double* xh;                  // PcgState::xh (baked into the graph's kernel parameters)
    bool operator<(const GraphKey& o) const {
        return std::tie(ncols, colp, x, rtol, maxit, norm_kind, xh) <
               std::tie(o.ncols, o.colp, o.x, o.rtol, o.maxit, o.norm_kind, o.xh);
    }
};

// 3D (face interface) state
// RA-evaluated fractional term in 3D (dd_frac DD_FRAC_RA): the r_F systems' sine-domain tables,
// inner-CG state and scratch (V1 = M p, V2 = r_F(L) V1, W1/W2 transform scratch, gcol = γ per column)
struct FSet {
    int nsys = 0;
    double *sys_a = nullptr, *sys_b = nullptr, *sys_w = nullptr, *cs = nullptr, *dg = nullptr, *idg = nullptr;
    double *ix = nullptr, *ir = nullptr, *ip = nullptr, *iq = nullptr, *iz = nullptr, *T1 = nullptr;
    double *irho = nullptr, *irho0 = nullptr;
    int* iactive = nullptr;
    double *V1 = nullptr, *V2 = nullptr, *W1 = nullptr, *W2 = nullptr, *gcol = nullptr;
    cudaGraphExec_t exec = nullptr;
    int key = -1;
    bool on_dev = false;
    int last_iters = 0;
    double *cc1 = nullptr, *cc2 = nullptr;   // Chebyshev tables (see Face3)
    int* kmax = nullptr;
    int kmax_all = 0;
};

struct Face3 {
    int n = 0, n2 = 0, ldf = 0;
    long long NP = 0;                 // padded face size ldf^2
    double* S = nullptr;              // sine matrix, round_up(n,64) x ldf row-major, zero padded
    double* sw = nullptr;             // Schur weights s_ab, NP (padded layout)
    // 3D bulk solve (dd_bulk_solve, allocated on first use): fields [col][layer][face] (+ slack),
    // the layer-major copy [col][face][layer], face buffers [col][face], user-layout Γ vectors, σ
    double *b3X = nullptr, *b3T = nullptr, *b3L = nullptr, *b3Y = nullptr;
    double *b3G = nullptr, *b3W = nullptr, *b3W2 = nullptr, *b3g = nullptr, *b3xg = nullptr, *b3sig = nullptr;
    double *b3Z = nullptr, *b3F = nullptr, *b3P = nullptr;   // bulk PCG: zero faces, γ F x_Γ, padded x_Γ
    double* F = nullptr;              // dense fractional term, rows round_up(NP,256) x NP row-major (DD_FX_FULL=1)
    double* Fp = nullptr;             // packed-symmetric F: upper 128 x 128 blocks as two 64-row halves (default)
    // packed-symmetric H = γ F + K S_unit (one parameter set per 3D handle): the Schur apply is one
    // packed stream, no per-apply slab transforms (DD_FX_FOLD=0 keeps transforms + F); Fp stays for
    // the bulk operator, which needs γ F alone
    double* Hp = nullptr;
    double* Hrows = nullptr;
    // single rank: Hp holds H̃ = T H T^T in the parity-ordered sine domain (T = Sp ⊗ Sp) and the PCG
    // runs there (no transforms around the preconditioner; dd_apply_schur transforms in and out)
    bool hat = false;
    bool hat_cs = false;              // Hp packed class-sparse (one 64 x 64 quadrant per half block)
    double* sw_hat = nullptr;         // the Schur weights s in the parity order (the diagonal of T S_unit T^T)          // the same fold for this rank's rows under a row-sharded pole split (F stays for bulk)
    int* fblk = nullptr;              // (I, J) of each packed block
    double *fxD = nullptr, *fxT = nullptr;   // direct / transposed block partials of the packed stream
    double* Kcol = nullptr;           // per-column K (gathered from col_param)
    // outer vectors [cols_pad][NP]
    double *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr, *z = nullptr, *U1 = nullptr, *U2 = nullptr;
    // pole systems of this rank: coefficients of A and M, weight, sine-diagonal preconditioner
    int nsys = 0;                     // systems handled by this rank
    int nsys_total = 0;
    std::vector<int> sys_ids;         // global system ids of this rank
    double *sys_a = nullptr, *sys_b = nullptr, *sys_w = nullptr;
    double *dg = nullptr, *idg = nullptr, *cs = nullptr;   // sine-domain diagonal / inverse [nsys][NP], D̂ coefficient [nsys]
    double* Dh = nullptr;             // D̂ = S D S (central difference in the sine basis) in the parity order, like S
    // The shifted systems live in the PARITY-ORDERED sine domain: index i <-> mode perm[i], odd
    // modes first (kpar of them), then even ones.  D̂ couples modes of opposite parity only, so in
    // this order it is [[0, E], [E', 0]] and its slab GEMMs skip the zero half of K (kpar != 0
    // when the block edge is 64-aligned).  Sp = P S (forward), SpT = S P^T (backward transform).
    double* Sp = nullptr;
    double* SpT = nullptr;
    int kpar = 0;
    bool cheb_fused = false;          // n_e = 64: one fused kernel per Chebyshev step (k_cheb_step)
    // inner PCG pairs [nsys * max_cols][NP]
    double *ix = nullptr, *ir = nullptr, *ip = nullptr, *iq = nullptr, *iz = nullptr, *T1 = nullptr, *T2 = nullptr;
    double *irho = nullptr, *irho0 = nullptr;
    int* iactive = nullptr;
    double inner_rtol = 1e-13;        // reading A12
    bool inner_cheb = true;           // reading A12': Chebyshev semi-iteration (DD_INNER_CG=1: the CG of round 1)
    double *cc1 = nullptr, *cc2 = nullptr;   // Chebyshev coefficients [nsys][CHEB_KMAX]
    int* kmax = nullptr;                     // a-priori step count per system
    int kmax_all = 0;                        // max over this rank's systems
    int inner_maxit = 400;
    int last_inner_iters = 0;
    cudaGraphExec_t inner_exec = nullptr;   // WHILE graph of the inner CG loop (key: inner_key = columns)
    int inner_key = -1;
    bool inner_iters_on_device = false;
    double* fx_ws = nullptr;
    int* fx_cnt = nullptr;
    // row-sharded F under the pole split: this rank holds rows [fx_r0, fx_r1) of F
    // (F points at row fx_r0); the other rows of γ F p arrive by ncclAllGather (fx_r1 - fx_r0 = NP:
    // unsharded)
    int fx_r0 = 0, fx_r1 = 0, fx_rows_max = 0;
    int* fx_r0s = nullptr;            // device [world + 1]: every rank's first row, then NP
    double *fx_send = nullptr, *fx_recv = nullptr;
    double lam_min = 0.0, lam_max = 0.0;   // spectrum of the face pair (from the setup gevp)
    void* nccl = nullptr;             // ncclComm_t when the poles are split across ranks
    FSet fs;                          // RA-evaluated fractional term (Remark 1), RA mode only
    int rank = 0, world = 1;
};

}  // namespace dd

struct dd_ctx {
    int dim = 2, N = 0, n = 0, ng = 0, Kpad = 0, ldv = 0, lda = 0, Mpad = 0;
    int n_param = 0, n_poles = 0, max_cols = 0, cols_pad = 0, device = 0, num_sms = 148;
    cudaStream_t stream = nullptr;
    std::vector<void*> allocs;
    // fractional perturbation (dd_frac): γ L^t, L = A_Γ + σ M_Γ; mode DENSE or RA (Remark 1)
    double frac_t = -0.5, frac_sigma = 0.0;
    int frac_mode = 0;
    double fra_c0 = 0.0;
    std::vector<double> fra_poles, fra_res;
    // full DD bulk solve (2D, dd_bulk_solve; allocated on first use)
    double *bulk_a = nullptr, *bulk_b = nullptr, *bulk_sinv = nullptr, *bulk_g = nullptr, *bulk_w = nullptr;
    double *bulk_gv = nullptr, *bulk_xg = nullptr;
    double *bpcg_r = nullptr, *bpcg_p = nullptr, *bpcg_q = nullptr, *bpcg_z = nullptr;   // bulk PCG vectors
    // operator data (2D)
    double* W = nullptr;      // 2D: Mpad x lda row-major: [S_dst | F | G] (RA mode: [S_dst | G]), blocks Kpad wide
    int g_off = 0;            // 2D: column offset of G = S_dst diag(s) S_dst (the unit Schur complement) in W
    double* ones = nullptr;   // [n_param] 1.0 (RA-mode bulk PCG: the fractional pole sum without γ)
    int schur_mode = 1;       // 2D Schur apply: 0 factored (K1 + K2), 1 assembled (one GEMM with [F | G]),
                              // 2 grouped (one GEMM with H_p = K_p G + γ_p F per parameter set)
    double* H = nullptr;      // grouped: n_param blocks of Mpad x Kpad (row-major, row stride Kpad)
    double* sw = nullptr;     // Schur weights s_b
    double* Kp = nullptr;     // [n_param]
    double* gp = nullptr;     // [n_param]
    dd::PoleGeom geom{};
    dd::PoleTabs tabs{};
    dd::PoleTabs ftabs{};     // RA of L^t (dd_frac DD_FRAC_RA): one set
    double* q_f = nullptr;    // fractional-term output U (RA mode), ldv x cols_pad
    // workspaces
    double *xw = nullptr, *Z = nullptr, *r = nullptr, *p = nullptr, *q = nullptr;
    double *bst = nullptr, *xst = nullptr;   // host-API staging (ld = n_Γ)
    int* colp_st = nullptr;
    double* gws = nullptr;
    int* gcnt = nullptr;
    // PCG scalars
    double *rho = nullptr, *eta0 = nullptr, *relres = nullptr, *hist = nullptr;
    int *active = nullptr, *iters = nullptr, *ints = nullptr;   // ints: kiter, n_active, n_active_next, done, status, flag
    int hist_cap = 0;
    bool hist_on = false;
    bool pair = false;                  // grouped mode through the shared-pair kernel (no H_p blocks)               // this solve records column 0's history (hist != NULL)
    // pinned host mirrors
    int* h_ints = nullptr;
    int* h_iters = nullptr;       // pinned staging of the per-column results [max_cols]
    double* h_rel = nullptr;
    // profiling
    bool prof = false;
    std::vector<dd::EvPair> ev_pending, ev_free;
    double prof_ms[DD_NKCLASS] = {0, 0, 0, 0};
    long long prof_n[DD_NKCLASS] = {0, 0, 0, 0};
    long long launches = 0;
    // graphs
    bool graph_ok = true;
    std::map<dd::GraphKey, cudaGraphExec_t> graphs;
    int last_split1 = 0, last_split2 = 0, last_ps_warps = 0, last_graph = 0, last_small = 0;
    long long graph_iter_launches = 3;   // kernels per PCG iteration in the captured body
    long long inner_iter_launches = 4;   // kernels per inner-CG iteration (3D WHILE graph)
    long long f_inner_iter_launches = 4; // same for the RA-evaluated fractional term's inner CG
    bool compact = true;      // GEMMs work over live (unconverged) column tiles only (DD_NO_COMPACT=1 disables)
    int* ntl = nullptr;       // live column tiles [count, ids...], written by the PCG kernels
    bool pdl = true;          // programmatic dependent launch between the iteration's kernels (DD_NO_PDL=1 disables)
    bool small_ok = true;     // persistent single-launch PCG for n <= 63 (DD_NO_SMALL=1 disables)
    cudaEvent_t solve_ev[2] = {nullptr, nullptr};
    // RA mode (2D): the fractional pole sum runs beside the Schur GEMM on a second stream
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    long long* dbg = nullptr;   // DD_PHASE_TIMING=1: CTA-0 phase timestamps of the last PCG iteration kernel
    // 3D
    dd::Face3 f3;
};

namespace dd {

template <typename T>
inline cudaError_t dalloc(dd_ctx* c, T** p, size_t count) {
    void* v = nullptr;
    cudaError_t e = cudaMalloc(&v, count * sizeof(T) + 256);
    if (e != cudaSuccess) return e;
    c->allocs.push_back(v);
    e = cudaMemsetAsync(v, 0, count * sizeof(T) + 256, c->stream);
    *p = reinterpret_cast<T*>(v);
    return e;
}

dd_status prof_begin(dd_ctx* c, EvPair& ev, int cls);
dd_status prof_end(dd_ctx* c, EvPair& ev);

#define DD_TIMED(cls, call)                                      \
    do {                                                         \
        ::dd::EvPair _ev{};                                      \
        dd_status _s = ::dd::prof_begin(c, _ev, cls);            \
        if (_s != DD_OK) return _s;                              \
        DD_CK(call);                                             \
        c->launches++;                                           \
        _s = ::dd::prof_end(c, _ev);                             \
        if (_s != DD_OK) return _s;                              \
    } while (0)

// 3D entry points (dd3d.cpp)
dd_status setup_3d(dd_ctx* c, const double* K, const double* mu_inv, const double* poles, const double* residues,
                   const double* c0, const dd_dist* dist);
dd_status schur_3d(dd_ctx* c, int ncols, const int* colp, const double* xin, double* yout, bool user_layout);
dd_status precond_3d(dd_ctx* c, int ncols, const int* colp, const double* rin, double* zout, bool user_layout);
dd_status bulk_solve_3d(dd_ctx* c, int ncols, const int* colp, const double* b, double* x, double rtol, int maxit,
                        int norm_kind, int* iters, double* rel_res);
dd_status bulk_pcg_3d(dd_ctx* c, int ncols, const int* colp, const double* b, double* x, double rtol, int maxit,
                      int* iters, double* rel_res);
dd_status pcg_3d(dd_ctx* c, int ncols, const int* colp, const double* b, double* x, double rtol, int maxit,
                 int norm_kind);
void destroy_3d(dd_ctx* c);

}  // namespace dd
