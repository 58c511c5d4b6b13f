// Internal declarations shared by the libdd translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <vector>

#include "../../include/dd_api.h"

namespace dd {

// ----------------------------------------------------------------------------- GEMM
// FP64 tensor-core GEMM  C = A·B  (A row-major, B column-major, C column-major), DMMA
// (mma.sync .f64) with a cp.async multi-stage pipeline and optional split-K.
constexpr int GEMM_BM = 64, GEMM_BN = 64, GEMM_BK = 16, GEMM_STAGES = 4, GEMM_THREADS = 128;
constexpr int GEMM_LDS = GEMM_BK + 4;   // padded smem row (doubles): conflict-free fragment loads
constexpr size_t GEMM_SMEM = size_t(GEMM_STAGES) * (GEMM_BM + GEMM_BN) * GEMM_LDS * sizeof(double);

enum EpiKind : int {
    EPI_STORE = 0,      // C[i,c] = acc
    EPI_SCHUR_DST = 1,  // C[i,c] = K_c s_i acc   and   Zlow[i,c] = γ_c X[i,c]   (Schur step a-2/a-3)
    EPI_ADD = 2,        // C[i,c] = acc + X[i,c]  (X with ldx)
};

struct GemmArgs {
    int M, N, K;                 // K multiple of GEMM_BK
    const double* A; int lda;    // row-major, rows readable up to round_up(M, BM)
    const double* B; int ldb;    // column-major, columns readable up to round_up(N, BN)
    double* C; int ldc;          // column-major
    int splitk;                  // 0: stream-K; 1..8: cluster split-K
    int num_sms;
    double* ws;                  // stream-K partials (gemm_ws_doubles)
    int* counters;               // [tiles], zero on entry, left zero on exit
    int epi;
    int pdl;                     // launch with programmatic stream serialisation (follows a kernel)
    int a_static;                // A is constant (prefetched before griddepcontrol.wait)
    const int* ntl;              // live column tiles [count, ids...] of width ntl_bn: work over these only (or null)
    int ntl_bn;                  // 64 (default when 0) or 32 (grouped)
    int n_param;
    // EPI_SCHUR_DST
    const int* col_param; const double* Kp; const double* gp; const double* s;
    const double* X; int ldx; double* Zlow;
    // grouped A (EPI_STORE, 32-column tiles): tile [n0, n0+32) multiplies A + col_param[n0] * sG,
    // unless *mixed (some tile spans two groups): then alt_A (M x alt_K) x alt_B for every tile
    int grouped; long long sG; const int* mixed;
    const double* alt_A; int alt_lda; const double* alt_B; int alt_ldb; int alt_K;
};
constexpr int GEMM_BN_GROUPED = 32;

// Grouped Schur apply from the shared pair (gemm_pair.cu): Y[:, c] = (K_p G + γ_p F) X[:, c]
struct PairArgs {
    int M, N, Kpad;
    const double *G, *F; int lda;      // row-major, rows readable up to round_up(M, 64)
    const double* X; int ldx;          // column-major, columns readable up to round_up(N, 64)
    const double* Z; int ldz, zhalf;   // mixed-tile fallback operand [γ X ; K X]
    const int* mixed;                  // device flag
    const int* col_param; int n_param;
    const double *Kp, *gp;
    const int* ntl;                    // live 32-column tiles or null
    double* Y; int ldy;
    double* ws; int* counters; int num_sms;
};
cudaError_t launch_gemm_pair(const PairArgs& a, cudaStream_t st);
size_t gemm_pair_ws_doubles(int M, int N, int num_sms);
int gemm_pair_tiles(int M, int N);
int gemm_pick_splitk_grouped(int M, int N, int K, int num_sms);

int gemm_tiles(int M, int N);
int gemm_pick_splitk(int M, int N, int K, int num_sms);   // 0 = stream-K
size_t gemm_ws_doubles(int M, int N, int num_sms);
cudaError_t launch_dgemm(const GemmArgs& a, cudaStream_t st);

// ----------------------------------------------------------------------------- pole sum
// 1D Γ: each shifted system (A_Γ - p M_Γ) (and M_Γ) is symmetric Toeplitz tridiagonal
// (diag d, off-diagonal e).  The n rows (padded to T LL) are split in T = 32 G chunks of LL <= 32
// rows, one per thread of a G-warp group: rows 0..LL-2 of a chunk are its interior, row LL-1 its
// separator.  Interiors: Thomas with precomputed factors in registers; separators: PCR over the
// group (shuffles for G = 1, shared memory for G > 1).
struct PoleGeom {
    int n;          // rows (n_Γ)
    int LL;         // chunk length (rows per thread), T LL >= n + 1
    int G;          // warps per system group (1, 2, 4, 8)
    int T;          // separators = 32 G
    int J;          // PCR steps = log2 T
    int part;       // first thread whose separator row is >= n (padding): floor(n / LL)
    int Lr_part;    // real interior rows of that thread: n - part * LL   (0..LL-1)
};

struct PoleTabs {
    int max_sys;                // systems per parameter set (mass term + poles), padded
    int n_param;                // parameter sets (col_param is clamped to [0, n_param))
    const int* nsys;            // [n_param]
    const double* w;            // [n_param][max_sys]  weight (c0 or c_k)
    const double* d;            // [n_param][max_sys]  diagonal
    const double* e;            // [n_param][max_sys]  off-diagonal
    const double* invb;         // [n_param][max_sys][LL]  1 / Thomas pivot
    const double* cpr;          // [n_param][max_sys][LL]  e / Thomas pivot
    const double* ufull;        // [n_param][max_sys][LL]  T_{LL-1}^-1 e_1
    const double* upart;        // [n_param][max_sys][LL]  T_{Lr_part}^-1 e_1
    const double* pa;           // [n_param][max_sys][J][T] PCR multipliers (left)
    const double* pb;           // [n_param][max_sys][J][T] PCR multipliers (right)
    const double* pinvb;        // [n_param][max_sys][T]    final 1/b
    // merged-interior pole sum (block_polesum_v2; NULL when the geometry does not qualify):
    // per parameter set a block of v2_stride doubles = W (16 x 16) + max_sys records of V2_REC
    const double* v2;
    int v2_stride;
    int v2_skip;                // diagnostics only (DD_V2_SKIP bitmask: 1 phase A, 2 phase B, 4 phase C)
    int pcr_smem;               // 1: phase B's PCR through the shared-memory rows (DD_PCR_SMEM=1), 0: in registers
};
// v2 pole-sum table layout (dd_api.cpp build_v2_record; pcg_polesum.cu block_polesum_v2)
constexpr int V2_L = 16;        // rows per chunk: 15 interior + 1 separator
constexpr int V2_WSZ = 256;     // merged interior operator W = Σ_k w_k T_int,k^-1, 16 x 16 (row/col 15 zero)
constexpr int V2_REC = 64;      // per system: [0,16) tf, [16,32) w e tf, e, w, 1/D, -, [36,48) PCR α_j,
                                //             [48,64) w e tf reversed (w e tf[14 - i])
constexpr int V2_E = 32, V2_WK = 33, V2_DINV = 34, V2_AL = 36, V2_WREV = 48;

// PCG state for a batch of columns (device).
struct PcgState {
    int n, ldv, ncols;
    const int* col_param;
    double* x; int ldx;                // solution (caller's buffer), column stride ldx
    double *r, *p, *q;                 // n x ncols, column stride ldv
    double *rho, *eta0, *relres;       // [ncols]
    int *active, *iters;               // [ncols]
    double* hist;                      // [maxit+1] column 0
    int* kiter;                        // iteration counter (device)
    int* n_active;                     // active columns after the last iteration
    int* n_active_next;                // scratch counter
    int* done_ctas;                    // scratch counter
    int* status;                       // 0 ok, DD_ENOTSPD
    double rtol; int maxit; int norm_kind;
    unsigned long long cond_handle;    // cudaGraphConditionalHandle (0 = none)
    long long* dbg;                    // optional phase timestamps of CTA 0 (DD_PHASE_TIMING=1)
    int* ntl;                          // live 64-column tiles [count, ids...] for the GEMMs (or null)
    int* ntl_cnt;                      // active columns per live-list tile (zeroed before pcg_init)
    int ntl_bn;                        // live-list tile width: 64, or 32 for the grouped Schur GEMM
    // assembled 2D Schur apply: every new p is also written as the GEMM operand [γ_c p ; K_c p]
    double* zs; int ldz, zhalf;        // Z (column stride ldz), K-half at row zhalf (or zs = null)
    const double *Kp, *gp;             // per-parameter K, γ
    const int* zmixed;                 // grouped apply: write zs only if *zmixed (fallback operand)
    const double* qadd;                // RA mode: q = q + qadd (the fractional term, computed concurrently)
    // dd_pcg_solve_host with a page-locked x: the device alias of the caller's host buffer (n x ncols,
    // column stride n).  The kernel that freezes a column writes its final x there over PCIe, so the
    // device-to-host transfer overlaps the iterations of the columns still running (or null).
    double* xh;
};

PoleGeom make_pole_geom(int n);
bool pole_geom_supported(const PoleGeom& g);
int polesum_groups(const PoleGeom& g);
int polesum_warps(const PoleGeom& g);
bool polesum_compact(const PoleGeom& g, int max_sys);
size_t polesum_smem_v(const PoleGeom& g, int max_sys, int v);
size_t polesum_smem(const PoleGeom& g, int max_sys);
bool polesum_v2_supported(const PoleGeom& g, int max_sys);
cudaError_t launch_pcg_init(const PcgState& s, const PoleGeom& g, const PoleTabs& t, const double* b,
                            int ldb, cudaStream_t st);
cudaError_t launch_pcg_iter(const PcgState& s, const PoleGeom& g, const PoleTabs& t, cudaStream_t st, bool pdl = false);
cudaError_t launch_precond(int ncols, const int* col_param, const PoleGeom& g, const PoleTabs& t,
                           const double* r, int ldr, double* z, int ldz, cudaStream_t st, bool pdl = false);
// RA-evaluated fractional term u = γ M r_F M x (dd_frac DD_FRAC_RA; t: one-parameter-set F tables)
cudaError_t launch_frac_ra(int ncols, const int* col_param, int n_param, const double* gp, const PoleGeom& g,
                           const PoleTabs& t, const double* x, int ldx, double* u, int ldu, double h6, cudaStream_t st,
                           bool pdl = false);
// whole PCG in one launch for n <= 63 (one CTA per column, operators in shared memory)
bool pcg_small_supported(int n);
cudaError_t launch_pcg_small(const PcgState& s, const PoleGeom& g, const PoleTabs& t, const double* b, int ldb,
                             const double* W, int lda, int Kpad, const double* sw, const double* Kp, const double* gp,
                             cudaStream_t st);
cudaError_t launch_copy_cols(int n, int ncols, const double* src, int lds, double* dst, int ldd,
                             cudaStream_t st);
// solve prologue: zero ints[0..nzero) and ntl[0..ntl_len), flag bad parameter ids (ints[5]) and,
// with check_tiles, 32-column tiles holding two parameter sets (ints[6])
cudaError_t launch_solve_prep(int ncols, const int* col_param, int n_param, int* ints, int nzero, int* ntl,
                              int ntl_len, bool check_tiles, cudaStream_t st);
// grouped Schur apply: *mixed = 1 if a 32-column tile holds two parameter sets
cudaError_t launch_check_tiles(int ncols, const int* col_param, int* mixed, cudaStream_t st);
// H_p = K_p G + γ_p F (W blocks at f_off, g_off) for all p: n rows, row stride ldh, H + p sH
cudaError_t launch_group_operators(int n, int n_param, const double* W, int lda, int f_off, int g_off, const double* Kp,
                                   const double* gp, double* H, int ldh, long long sH, cudaStream_t st);
// Z[:, c] = [γ_c x_c ; K_c x_c] (rows 0.. and zhalf..): operand of the assembled Schur GEMM
cudaError_t launch_schur_operand(int n, int ncols, const int* col_param, int n_param, const double* Kp,
                                 const double* gp, const double* x, int ldx, double* Z, int ldz, int zhalf,
                                 cudaStream_t st);
cudaError_t launch_check_params(int ncols, const int* col_param, int n_param, int* flag, cudaStream_t st);

// ----------------------------------------------------------------------------- 2D bulk solve (bulk2d.cu)
cudaError_t bulk_slab_pass(const double* in, double* out, int nslab, int n, int ldf, const double* S, int lds,
                           const double* w, cudaStream_t st);
cudaError_t bulk_in(int n, int ldf, int ncols, const double* b, long long ldb, double* slab, double* gout, int ldg,
                    cudaStream_t st);
cudaError_t bulk_row1(int n, int ldf, int ncols, const double* Yh, const double* s1, double* w, int ldw,
                      cudaStream_t st);
cudaError_t bulk_update(int n, int ldf, int ncols, double* Yh, const double* s1, const double* u, int ldu,
                        const double* sinv, const int* col_param, int n_param, const double* Kp, cudaStream_t st);
cudaError_t bulk_out(int n, int ldf, int ncols, const double* slab, const double* xg, int ldg, double* x, long long ldx,
                     cudaStream_t st);

cudaError_t bulk_apply(int n, int ncols, const double* x, long long nb, const double* fx, int ldfx, const int* col_param,
                       int n_param, const double* Kp, const double* gp, double* y, cudaStream_t st);
cudaError_t bpcg_a(int ncols, long long nb, double* x, double* r, const double* p, const double* q, const double* rho,
                   int* active, int* status, cudaStream_t st);
cudaError_t bpcg_b(int ncols, long long nb, const double* r, const double* z, double* p, double* rho, double* eta0,
                   double* relres, int* active, int* iters, int k, double rtol, int maxit, int init, int* n_active,
                   int* status, cudaStream_t st);

// ----------------------------------------------------------------------------- 3D face (face3d.cu)
struct InnerArgs {
    int n, ldf; long long NP;
    int npair, C;                 // pairs (= systems x columns), columns
    double hh12;                  // h^2 / 12
    const double* sys_a;          // [systems] coefficient of A_Γ (1 for poles, 0 for the mass term)
    const double* sys_b;          // [systems] coefficient of the mass stencil (-p for poles, 1 for M)
    double *x, *r, *p, *q, *z;    // [npair][NP]
    double *rho, *rho0;           // [npair]
    int* active;                  // [npair]
    double rtol;
    const double* dg;             // [systems][NP] sine-diagonal part a α + b μ̃ (0 on padding)
    const double* idg;            // [systems][NP] its inverse (0 on padding)
    const double* cs;             // [systems] coefficient of D̂ v D̂^T: b h^2/24
    // Chebyshev inner solver (reading A12'): per system the step count and the recurrence
    // coefficients d <- c1[k] d + c2[k] P^-1 r of step k (kstride entries per system)
    const double *cc1 = nullptr, *cc2 = nullptr;
    const int* kmax = nullptr;
    int kstride = 0;
    const int* kiter = nullptr;   // device: the current step k (the loop's counter)
    double* x1 = nullptr;         // fused Chebyshev step: second x̂ buffer (x̂ ping-pongs x <-> x1 by step parity)
};
constexpr int CHEB_KMAX = 40;     // upper bound on the a-priori Chebyshev step counts
struct Pcg3 {
    long long NP; int ncols;
    double *x, *r, *p, *q, *z;    // padded face vectors [ncols][NP]
    double *rho, *eta0, *relres;
    int *active, *iters;
    double* hist;
    double rtol; int norm_kind;
    int* status;
};
cudaError_t face_slab_pass(const double* in, double* out, int nslab, int n, int ldf, const double* S, cudaStream_t st);
// 3D bulk solve (bulk3d.cu): full-field fast diagonalisation of the interior block
cudaError_t bulk3_forward(int n, int ldf, int lk, long long NP, int ncols, const double* S, const double* sig,
                          const double* X, double* T, double* Lk, double* Y, cudaStream_t st);
cudaError_t bulk3_inverse(int n, int ldf, int lk, long long NP, int ncols, const double* S, const double* Y, double* T,
                          double* Lk, double* X, cudaStream_t st);
cudaError_t bulk3_in(int n, int ldf, long long NP, int ncols, const double* b, long long ldb, double* X, double* G,
                     cudaStream_t st);
cudaError_t bulk3_layer1(int n, long long NP, int ncols, const double* Y, const double* s1, double* w, cudaStream_t st);
cudaError_t bulk3_g(int n, int ldf, long long NP, int ncols, const double* G, const double* W, double* g, cudaStream_t st);
cudaError_t bulk3_pad(int n, int ldf, long long NP, int ncols, const double* xg, long long lds, double* P,
                      cudaStream_t st);
cudaError_t bulk3_combine(int n, int ldf, long long NP, int ncols, double* Y, const double* XG, const double* s1,
                          const double* sig, const int* col_param, int n_param, const double* Kp, double h,
                          cudaStream_t st);
cudaError_t bulk3_out(int n, int ldf, long long NP, int ncols, const double* X, const double* xg, double* x, long long ldx,
                      cudaStream_t st);
cudaError_t bulk3_apply(int n, int ldf, long long NP, int ncols, const double* x, long long ldx, const double* fx,
                        const int* col_param, int n_param, const double* Kp, double h, double* out, cudaStream_t st);
cudaError_t face_slab_pass_scaled(const double* in, double* out, int nslab, int n, int ldf, const double* S,
                                  const double* w, long long sW, int group, const double* colscale, cudaStream_t st);
// packed-symmetric F stream (fx_sym.cu): upper 128 x 128 blocks, one read per block, two products
int fx_sym_blocks(long long NP);
size_t fx_sym_packed_doubles(long long NP, bool class_sparse = false);
size_t fx_sym_partial_doubles(long long NP, int max_cols);
bool fx_sym_supported(long long NP);
void fx_sym_block_table(long long NP, std::vector<int>& ij);          // (I, J) per packed block
// class_sparse: keep per half only its nonzero 64-column quadrant (the sine-domain H̃ at ldf = 128,
// block-diagonal in the face-index parity classes)
cudaError_t fx_sym_pack(const double* F, long long NP, const int* blk, double* Fp, cudaStream_t st,
                        bool class_sparse = false);
// S_unit folded into F at setup (dd3d.cpp): identity columns of the real face nodes j0.. j0+nb-1,
// and rows pad(j) of the dense F replaced by γ F + Y (Y = K S_unit e_j from the slab passes)
cudaError_t face_identity_cols(int n, int ldf, long long NP, int j0, int nb, double* X, cudaStream_t st);
cudaError_t face_fold_rows(double* F, long long NP, int n, int ldf, int j0, int nb, double gamma, const double* Y,
                           cudaStream_t st);
// B (row-major rows x ldb, row = face node j-major) column block j0..j0+nb-1 <-> padded face vectors
cudaError_t face_gather_cols(const double* B, int rows, int ldb, int j0, int nb, int n, int ldf, long long NP, double* X,
                             cudaStream_t st);
cudaError_t face_scatter_cols(const double* X, int rows, int ldb, int j0, int nb, int n, int ldf, long long NP, double* B,
                              cudaStream_t st);
// F <- γ F + K diag(w) on the padded NP x NP row-major F (w: padded face table)
cudaError_t face_hat_diag(double* F, long long NP, int n, int ldf, double gamma, double K, const double* w,
                          cudaStream_t st);
// D = NULL: q = γ_c F p;  gp = NULL: γ_c = 1
cudaError_t fx_sym_apply(const double* Fp, const int* blk, long long NP, const double* p, double* q, const double* D,
                         int ncols, const int* col_param, int n_param, const double* gp, double* Dpart, double* Tpart,
                         int num_sms, cudaStream_t st, bool class_sparse = false);
size_t face_fx_ws_doubles(long long NP, int ncols, int num_sms);
int face_fx_tiles(long long NP, int ncols);
cudaError_t face_fx(const double* F, long long NP, const double* p, double* q, const double* D, int ncols,
                    const int* col_param, int n_param, const double* gp, double* ws, int* counters, int num_sms,
                    cudaStream_t st,
                    int row0 = 0, int rows = -1);
cudaError_t fx_pack(const double* q, long long NP, int ncols, int r0, int rows, int rows_max, double* buf,
                    cudaStream_t st);
cudaError_t fx_unpack(const double* buf, long long NP, int ncols, int world, int rows_max, const int* r0s, double* q,
                      cudaStream_t st);
cudaError_t fx_zero_outside(long long NP, int ncols, int r0, int r1, double* q, cudaStream_t st);
cudaError_t face_gram_scatter(const double* B, int n2, int kp, double* F, int n, int ldf, long long NP, int num_sms,
                              cudaStream_t st);
cudaError_t face_copy_in(int n, int ldf, long long NP, int ncols, const double* src, int lds, double* dst, cudaStream_t st);
cudaError_t face_copy_out(int n, int ldf, long long NP, int ncols, const double* src, double* dst, int ldd,
                          cudaStream_t st);
cudaError_t face_dense_pair(int n, double hh12, double* A, double* M, cudaStream_t st);
cudaError_t face_mass_cols(int n, double hh12, const double* V, double* out, int ncol, int ldo, cudaStream_t st);
cudaError_t face_mass_axpy(int n, int ldf, long long NP, int ncols, double hh12, const double* v, const double* scale,
                           const double* add, double* out, cudaStream_t st);
cudaError_t scale_transpose(const double* V, const double* w, int n2, double* out, int kp, cudaStream_t st);
cudaError_t face_slab_pass_active(const double* in, double* out, int nslab, int n, int ldf, const double* B,
                                  const int* active, int kpar, cudaStream_t st);
cudaError_t face_inner_op_pass(const double* in, double* q, const double* p, int nslab, int C, int n, int ldf,
                               const double* B, const double* dg, const double* cs, const int* active, int kpar,
                               cudaStream_t st);
cudaError_t face_inner_cheb_pass(const double* in, const InnerArgs& a, const double* bh, const double* B, int kpar,
                                 cudaStream_t st);
cudaError_t inner_init_hat(const InnerArgs& a, const double* bh, cudaStream_t st);
cudaError_t inner_init_cheb(const InnerArgs& a, const double* bh, cudaStream_t st);
// fused Chebyshev step (one persistent kernel per step; n_e = 64, ldf = 128 only — cheb_fused_ok):
// V = D̂ X̂ D̂^T per (pair, 64x64 parity block), the step's epilogue, and the loop condition
bool cheb_fused_ok(int n, int ldf);
cudaError_t cheb_step_fused(const InnerArgs& a, const double* bh, const double* Dh, int* n_active, int* counter,
                            int* done, int maxit, unsigned long long handle, int num_sms, cudaStream_t st,
                            int nsteps = 0);
cudaError_t inner_cond_cheb(const InnerArgs& a, int* n_active, int* counter, int maxit, unsigned long long handle,
                            cudaStream_t st);
cudaError_t inner_update_hat(const InnerArgs& a, int* n_active, cudaStream_t st);
cudaError_t inner_init(const InnerArgs& a, const double* b, cudaStream_t st);
cudaError_t inner_cond(int* n_active, int* counter, int maxit, unsigned long long handle, cudaStream_t st);
cudaError_t inner_start(const InnerArgs& a, cudaStream_t st);
cudaError_t inner_step1(const InnerArgs& a, cudaStream_t st);
cudaError_t inner_step2(const InnerArgs& a, int* n_active, cudaStream_t st);
cudaError_t inner_combine(const InnerArgs& a, const double* w, int nsys, double* zout, cudaStream_t st);
cudaError_t pcg3_start(const Pcg3& s, cudaStream_t st);
cudaError_t pcg3_alpha(const Pcg3& s, cudaStream_t st);
cudaError_t pcg3_beta(const Pcg3& s, int k, int maxit, int* n_active, cudaStream_t st);
cudaError_t gather_param(int ncols, const int* col_param, int n_param, const double* src, double* dst, cudaStream_t st);

}  // namespace dd
