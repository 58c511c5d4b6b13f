/*
 * dd_api.h — C ABI of libdd: B200-native (sm_100a) Schur-complement PCG for operators
 * with fractional interface perturbations (M. Kuchta, arXiv 2211.15308).
 *
 * The system (Eq.(2)):   -K Δ_Ω x + μ^-1 (-Δ_Γ)^{-1/2} x = b,
 * discretised by P1 elements on Ω = (0,1)^d with Γ = {x = 0},
 * homogeneous Dirichlet on ∂Ω\Γ and ∂Γ.  After the split V = V0 ⊕ VΓ (PAPER.md:104-122,
 * Eq.(4)) the library solves the interface (Steklov–Poincaré / Schur) system
 *
 *     S x = b,   S = K (A^ii - A^i0 (A^00)^-1 A^0i) + γ F,   γ = μ^-1,
 *     F = L_h^{-1/2} = (M U) Λ^{-1/2} (M U)^T          (Eq.(7))
 *
 * by PCG from x0 = 0 preconditioned with the rational approximation
 *
 *     P = c0 M_Γ^-1 + Σ_k c_k (A_Γ - p_k M_Γ)^-1       (Eq.(8))
 *
 * of S_Γ^-1 = (K L^{1/2} + γ L^{-1/2})^-1 (Eq.(6)).
 * Pole sign convention (reading A7): `poles` are the scalar poles p_k < 0 of
 * r(λ) = c0 + Σ c_k/(λ - p_k); the library forms A_Γ - p_k M_Γ = A_Γ + |p_k| M_Γ.
 *
 * Layout: every vector argument is n_Γ x ncols, column-major (each column = one right-hand
 * side, contiguous, leading dimension n_Γ), fp64.  Interface ordering is lexicographic:
 * 2D node (0, j h) -> j-1;  3D node (0, j h, k h) -> (j-1)(N-1) + (k-1).
 * All vector pointers of the dd_apply_* / dd_pcg_solve calls are DEVICE pointers on the
 * handle's device; dd_pcg_solve_host takes HOST pointers and stages them itself.
 *
 * Ownership: the caller owns every vector buffer; the handle owns the operator data
 * (sine matrix, F, Schur weights, pole tables), all workspaces (sized by max_cols at
 * setup; apply/solve never allocate) and, when distributed, the NCCL communicator.
 * Streams: apply calls are asynchronous on the handle's stream; dd_pcg_solve synchronises
 * that stream once at the end to fill its host outputs.
 * Thread safety: a handle is not thread-safe; distinct handles are independent.
 * Errors: return codes only; nothing crosses the ABI as an exception.  On DD_EINVAL found
 * by the host-side argument checks no output is written.  Two checks run on the device
 * instead (no host synchronisation in the asynchronous calls): an out-of-range col_param
 * entry is CLAMPED to [0, n_param) by the kernels — dd_apply_schur / dd_apply_precond then
 * return DD_OK with the clamped-parameter outputs (they cannot see the device flag), while
 * dd_pcg_solve / dd_pcg_solve_host / dd_bulk_* read the flag back and return DD_EINVAL
 * AFTER x has been written (its contents are then undefined).  dd_last_error() returns a
 * thread-local description of the last failure.
 */
#ifndef DD_API_H
#define DD_API_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DD_OK = 0,
    DD_EINVAL = 1,      /* invalid argument (nothing written)                              */
    DD_ECUDA = 2,       /* CUDA runtime error                                              */
    DD_ENOMEM = 3,      /* device allocation failed                                        */
    DD_ENOTSPD = 4,     /* p.Sp <= 0 or r.Pr < 0 met in PCG ("indefiniteness") */
    DD_ENOCONV = 5,     /* non-fatal: some column hit maxit; outputs are the last iterate  */
    DD_ENCCL = 6,       /* NCCL error (distributed handles)                                */
    DD_EUNSUPPORTED = 7 /* valid request this build does not implement                     */
} dd_status;

typedef struct {
    int dim;            /* 2: unit square, Γ = edge {x=0};  3: unit cube, Γ = face {x=0}     */
    int cells_per_side; /* N >= 2; mesh size h = 1/N; n = N-1 interior nodes per axis      */
    int gamma_face;     /* 0: {x = 0} (only value supported)                               */
} dd_mesh;

typedef struct {
    int rank, world;              /* this process's rank / number of ranks                 */
    const void* nccl_unique_id;   /* 128-byte ncclUniqueId (broadcast by the caller); NULL with
                                     DD_SHARD_POLES: no communicator — dd_apply_precond returns
                                     this rank's partial pole sum (emulating ranks in one process
                                     for tests; dd_pcg_solve then is NOT the global solve)     */
    int mode;                     /* DD_SHARD_COLUMNS or DD_SHARD_POLES                      */
} dd_dist;
#define DD_SHARD_COLUMNS 0        /* each rank passes its own columns; no collective        */
#define DD_SHARD_POLES 1          /* RA poles split across ranks + allreduce of the sum     */

typedef struct dd_ctx dd_ctx;

/*
 * dd_frac — the fractional perturbation, generalising Eq.(2)'s γ(-Δ_Γ)^{-1/2} to Eq.(9)'s
 * γ L^t:
 *   t         exponent, -1 < t < 1 (Eq.(2): t = -1/2)
 *   shifted   0: L = -Δ_Γ, the pair (A_Γ, M_Γ) (Eq.(2));  1: L = -Δ_Γ + I_Γ, i.e. (A_Γ + M_Γ, M_Γ)
 *             (Eq.(9))
 *   mode      DD_FRAC_DENSE: F = (M U)(Λ_L)^t (M U)^T formed once at setup (Eq.(7));
 *             DD_FRAC_RA: F x ≈ M r_F(L) M x through a second rational approximation
 *             r_F(λ) = fc0 + Σ fc_k/(λ - fp_k) ≈ λ^t applied as a pole sum (Remark 1,
 *             PAPER.md:274-288): linear memory and work, no dense n_Γ² block
 *   fc0, n_fpoles, fpoles, fresidues   r_F for DD_FRAC_RA (host; ignored for DENSE); fp_k < 0
 *             are poles of the unshifted pair (A_Γ, M_Γ), like dd_setup's `poles`
 * The preconditioner's RA (dd_setup's poles/residues) must then approximate
 * (K λ_L^{1/2} + γ λ_L^t)^-1 in λ of the pair (A_Γ, M_Γ) — the library only applies it.
 */
typedef struct {
    double t;
    int shifted;
    int mode;
    double fc0;
    int n_fpoles;
    const double* fpoles;
    const double* fresidues;
} dd_frac;
#define DD_FRAC_DENSE 0
#define DD_FRAC_RA 1

/*
 * dd_setup — build a handle for one mesh and n_param parameter sets.
 *   K[n_param], mu_inv[n_param]   host; K > 0, mu_inv >= 0   (γ = mu_inv)
 *   poles, residues               host [n_param * n_poles]; parameter set j uses entries
 *                                 j*n_poles .. j*n_poles+n_poles-1; every pole < 0 and finite;
 *                                 a zero residue disables that pole (no solve is issued)
 *   c0                            host [n_param]: coefficient of M_Γ^-1 in Eq.(8)
 *   max_cols                      largest ncols any later call may pass (workspace size)
 *   device, cuda_stream           CUDA device ordinal and cudaStream_t (NULL = legacy)
 *   dist                          NULL for a single GPU
 * The RA fit itself is not part of the library (PAPER.md:196-198 defers it to the
 * references); the Python package provides one (rafit.py).
 * 3D (n_param must be 1) with the dense F: setup runs the generalised eigensolve of the face pair
 * (cuSOLVER, n_Γ = (N-1)^2) and keeps two packed-symmetric operators, F (for the bulk operator) and
 * the Schur operator in the parity-ordered sine domain, T (γ F + K S_unit) T^T with T = Sp ⊗ Sp
 * (the PCG runs in that orthogonal basis; dd_apply_schur / dd_pcg_solve take and return
 * physical-domain vectors) — at N = 128 1.08 GB for F; the sine-domain operator is block-diagonal
 * in the face parity classes c(a,b) = par(a) xor par(b) and is stored class-sparse (one 64 x 64
 * quadrant per stored half block, 0.54 GB; DD_FX_CLASS_SPARSE=0 keeps the full blocks), plus a
 * transient dense n_Γ^2 (2.1 GB) during setup; under a pole split each rank keeps its rows of F and
 * of γ F + K S_unit instead.
 * Returns DD_EINVAL for dim not in {2,3}, N < 2, gamma_face != 0, K <= 0, mu_inv < 0,
 * a pole >= 0 or not finite, n_param < 1, n_poles < 0, max_cols < 1.
 */
dd_status dd_setup(const dd_mesh* mesh, int n_param, const double* K, const double* mu_inv,
                   int n_poles, const double* poles, const double* residues, const double* c0,
                   int max_cols, int device, void* cuda_stream, const dd_dist* dist,
                   dd_ctx** out);

/* dd_setup with a general fractional perturbation (dd_frac above; NULL = Eq.(2): t = -1/2,
 * unshifted, dense F).  Extra DD_EINVAL cases: t not in (-1, 1), shifted not in {0, 1},
 * mode unknown, DD_FRAC_RA with a pole >= 0 / non-finite coefficient. */
dd_status dd_setup_ex(const dd_mesh* mesh, const dd_frac* frac, int n_param, const double* K,
                      const double* mu_inv, int n_poles, const double* poles, const double* residues,
                      const double* c0, int max_cols, int device, void* cuda_stream,
                      const dd_dist* dist, dd_ctx** out);

/* n_Γ = N-1 (2D) or (N-1)^2 (3D); -1 for a NULL handle. */
int dd_interface_size(const dd_ctx* ctx);

/*
 * dd_apply_schur — y = S x per column:
 *   y_c = K_c (A^ii - A^i0 (A^00)^-1 A^0i) x_c + γ_c F x_c,  (K_c, γ_c) = set col_param[c].
 * The interior solve (A^00)^-1 is exact (fast diagonalisation; "exactly").
 *   col_param  DEVICE int[ncols], each in [0, n_param) (out-of-range entries are clamped on
 *              the device and not reported by this asynchronous call; see "Errors" above)
 *   x, y       DEVICE n_Γ x ncols column-major; x and y must not overlap.
 * 0 <= ncols <= max_cols (ncols = 0 is a no-op).
 */
dd_status dd_apply_schur(dd_ctx* ctx, int ncols, const int* col_param, const double* x, double* y);

/*
 * dd_apply_precond — z = P r per column with the column's RA (Eq.(8)),
 * shifted solves summed in the fixed order: M term, then poles in the given order.
 * 2D handles solve the 1D shifted systems directly (tridiagonal, long-double tables); 3D handles
 * solve the face systems iteratively to a 1e-13 relative accuracy (reading A12':
 * Chebyshev semi-iteration with a-priori spectral bounds), so 3D P is exact up to that.
 */
dd_status dd_apply_precond(dd_ctx* ctx, int ncols, const int* col_param, const double* r, double* z);

/*
 * dd_pcg_solve — x = S^-1 b per column by PCG from x0 = 0, stopping a
 * column when its preconditioned residual norm η_k <= rtol * η_0, where
 *   norm_kind 0: η = sqrt(r.Pr) (default)     1: η = ||Pr||_2.
 * Columns freeze individually on convergence (x, r untouched afterwards).
 *   b, x       DEVICE n_Γ x ncols (b may equal x? no: must not overlap)
 *   iters      HOST int[ncols]: S applications until convergence (or maxit)
 *   rel_res    HOST double[ncols]: final η / η0
 *   hist       HOST double[maxit+1] or NULL: η history of column 0 (η0 first); entries
 *              after column 0 converged are left untouched
 *   maxit      >= 0; with hist != NULL also maxit + 1 <= 4096 (else DD_EINVAL)
 * Returns DD_ENOCONV if any column reached maxit (outputs valid), DD_ENOTSPD on p.Sp <= 0
 * or r.Pr < 0 (outputs are the iterate at that point), DD_EINVAL after the solve when a
 * col_param entry was out of range (x written, contents undefined).
 */
dd_status dd_pcg_solve(dd_ctx* ctx, int ncols, const int* col_param, const double* b, double* x,
                       double rtol, int maxit, int norm_kind, int* iters, double* rel_res,
                       double* hist);

/* As dd_pcg_solve but b, x and col_param are HOST pointers: the call copies col_param
 * host->device, solves, and copies x device->host (synchronous, one synchronisation).  b is
 * read once, by the solve's first kernel: page-locked (pinned) host memory is read there in
 * place over PCIe (UVA), overlapping the transfer with that kernel; pageable memory is
 * staged by a copy first.  x likewise (2D, n_Γ >= 64): into a page-locked x the kernel that
 * freezes a column writes that column's final iterate directly, so the device->host transfer
 * of early-converging columns overlaps the iterations of the others; a pageable x, or a solve
 * stopped by DD_ENOTSPD / maxit = 0, gets one copy after the loop.  (DD_NO_ZERO_COPY=1 forces
 * both copies.) */
dd_status dd_pcg_solve_host(dd_ctx* ctx, int ncols, const int* col_param_host,
                            const double* b_host, double* x_host, double rtol, int maxit,
                            int norm_kind, int* iters, double* rel_res, double* hist);

/*
 * dd_bulk_solve — the full DD solve of the discrete Eq.(2) on a BULK right-hand side (SURVEY
 * §8(f) NEXT-1): block elimination with the exact leading block (PAPER.md: 123-145 Eq.(5),
 * 229-230 "(A^00)^-1 ... computed exactly"):
 *     g = b_Γ - A^{i0}(A^00)^-1 b_0,   x_Γ = S^-1 g (dd_pcg_solve),   x_0 = (A^00)^-1(b_0 - A^{0i} x_Γ)
 * with (A^00)^-1 by full-field fast diagonalisation (DST-I along every axis, batched DMMA).
 *   b, x   DEVICE.  2D: column c at c*(n^2 + n): [interior nodes (i h, j h), i, j = 1..n, at
 *          (i-1) n + (j-1)  (x-major);  Γ nodes (0, j h) at n^2 + (j-1)],  n = N - 1.
 *          3D: column c at c*(n^3 + n^2): [interior (i h, j h, k h) at (i-1) n^2 + (j-1) n + (k-1);
 *          Γ nodes (0, j h, k h) at n^3 + (j-1) n + (k-1)].
 *   rtol, maxit, norm_kind, iters, rel_res: as dd_pcg_solve (for the interface PCG)
 * Allocates its workspaces on first use (2D: 2 max_cols x Kpad^2 fields; 3D: 3 max_cols x n x
 * ldf^2 fields and a layer-major copy).  Otherwise as dd_pcg_solve.  Synchronous.
 */
dd_status dd_bulk_solve(dd_ctx* ctx, int ncols, const int* col_param, const double* b, double* x,
                        double rtol, int maxit, int norm_kind, int* iters, double* rel_res);

/*
 * dd_bulk_pcg_solve — the paper's protocol (Figs. 2-3): PCG on the BULK system
 * 𝒜 x = b (the discrete Eq.(2) on all free nodes, 𝒜 = K A_h + γ T^T F T) from x0 = 0,
 * preconditioned by the DD preconditioner 𝓑 of Eq.(5) with the leading block
 * exact (fast diagonalisation) and S_Γ^-1 realised by the handle's RA (Eq.(8)); stops when
 * sqrt(r·𝓑r) <= rtol · sqrt(r0·𝓑r0).  Same vector layout as dd_bulk_solve (2D and 3D handles).
 * In DD_FRAC_RA mode the operator's fractional term is the RA-evaluated γ M r_F(L) M (Remark 1,
 * operator and preconditioner both by RA).  iters / rel_res: HOST [ncols] or
 * NULL.  Allocates 4 max_cols x (bulk size) vectors on first use.  Synchronous.
 */
dd_status dd_bulk_pcg_solve(dd_ctx* ctx, int ncols, const int* col_param, const double* b, double* x,
                            double rtol, int maxit, int* iters, double* rel_res);

dd_status dd_destroy(dd_ctx* ctx);
const char* dd_last_error(void);

/* 128-byte ncclUniqueId for dd_dist (rank 0 calls it and broadcasts the bytes). */
dd_status dd_nccl_unique_id(void* out128);
/* 3D handles: inner iterations of the last preconditioner apply — the shifted face systems'
 * operator applications (Chebyshev default: max_s K_s - 1, the first step being P^-1 b; with
 * DD_INNER_CG=1 the inner CG iterations). */
dd_status dd_inner_iterations(const dd_ctx* ctx, int* iters);

/* 2D handles: how dd_apply_schur and the PCG apply S = K_c S_unit + γ_c F (
 * SURVEY §8(a) rows a-2, a-3).  Both give the same operator up to rounding order:
 *   DD_SCHUR_FACTORED (0): per apply, the interior solve by fast diagonalisation,
 *        T' = (K_c s) ∘ (S_dst X) then Y = [S_dst | F] [T' ; γ X]   (6 n^2 flops per column);
 *   DD_SCHUR_ASSEMBLED (1; the default in DD_FRAC_RA mode): the parameter-independent interior
 *        solve is applied once at setup to the identity, G = S_dst diag(s) S_dst = S_unit (n x n,
 *        beside F in the handle), and each apply is one GEMM  Y = [F | G] [γ X ; K X]
 *        (4 n^2 flops per column); in DD_FRAC_RA mode Y = G (K X) + γ M r_F(L) M X.
 *   DD_SCHUR_GROUPED (2; THE DEFAULT with the dense F): each apply is one grouped GEMM
 *        Y[:, c] = (K_p G + γ_p F) X[:, c] (2 n^2 flops per column) over 32-column tiles holding one
 *        parameter set each.  The per-parameter operators H_p = K_p G + γ_p F (n_param x n^2
 *        doubles) are formed when the mode is selected if they fit in 16 GiB; otherwise (or with
 *        DD_GROUPED_PAIR=1) the GEMM forms each tile's operator in registers from the shared pair
 *        (G, F) (2 n^2 doubles).  A call whose 32-column tiles mix parameter sets computes the
 *        assembled product instead (same result, checked on the device, no host synchronisation).
 * mode outside {0,1,2}, a 3D handle, or GROUPED in DD_FRAC_RA mode: DD_EINVAL.  (3D with the dense
 * F folds K S_unit into the packed-symmetric stream at setup, H = γ F + K S_unit — one parameter set
 * per 3D handle; with RA-evaluated F or a pole-split row shard it applies the interior solve per
 * apply.)  The environment variable DD_SCHUR_MODE=0|1|2 sets the mode at setup. */
#define DD_SCHUR_FACTORED 0
#define DD_SCHUR_ASSEMBLED 1
#define DD_SCHUR_GROUPED 2
dd_status dd_set_schur_mode(dd_ctx* ctx, int mode);

/* ---------------------------------------------------------------- instrumentation
 * Per-kernel-class device time (CUDA events on the handle's stream, recorded around each
 * launch while enabled; graphs are bypassed while enabled).  Classes: */
#define DD_KCLASS_GEMM_DST 0      /* K1: T = S_dst X with the Schur-weight epilogue (factored) */
#define DD_KCLASS_GEMM_SCHUR 1    /* K2: Y = [S_dst | F] [T ; γX]  or assembled [F | G] [γX ; KX] */
#define DD_KCLASS_POLESUM 2       /* K3 (+K4): fused PCG update + pole sum + dots           */
#define DD_KCLASS_OTHER 3         /* init / copies / allreduce                              */
#define DD_NKCLASS 4
dd_status dd_profile_enable(dd_ctx* ctx, int on);
/* ms[DD_NKCLASS] total milliseconds, launches[DD_NKCLASS]; resets the counters. */
dd_status dd_profile_read(dd_ctx* ctx, double* ms, long long* launches);
/* Device time of the last dd_pcg_solve / dd_pcg_solve_host in ms: CUDA events on the handle's
 * stream around the whole solve (parameter check, init, iterations), excluding the final
 * device->host read of iters/rel_res and, for the host variant, the staging copies. */
dd_status dd_last_solve_ms(dd_ctx* ctx, double* ms);
/* Number of this library's kernel launches since the last call (resets). */
long long dd_launch_count(dd_ctx* ctx);
/* Launch configuration actually used (for reports): splitk of the two GEMMs, pole-sum
 * warps per CTA, whether the CUDA-graph WHILE loop is used. */
dd_status dd_query_config(const dd_ctx* ctx, int* splitk_dst, int* splitk_schur, int* ps_warps,
                          int* uses_graph);

/* ---------------------------------------------------------------- test hooks
 * C = A B in fp64 with the library's DMMA GEMM: A row-major M x K (lda), B column-major
 * K x N (ldb), C column-major M x N (ldc); device pointers; K % 16 == 0, lda % 2 == 0,
 * ldb % 2 == 0 and 16-byte aligned A/B; rows of A up to round_up(M, 64) and columns of B
 * up to round_up(N, 64) must be readable.  Used by the parity tests only. */
dd_status dd_test_dgemm(int M, int N, int K, const double* A, int lda, const double* B, int ldb,
                        double* C, int ldc, int splitk, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* DD_API_H */
