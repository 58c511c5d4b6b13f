// Full DD solve of the bulk problem on a bulk right-hand side (2D).
//
// The discrete Eq.(2) on all free nodes, split V = V0 ⊕ VΓ (Eq.(4)):
//     [ K L00       -K E ] [x0]   [b0]          L00 = 5-point Laplacian on the n x n interior
//     [ -K E^T   S_ΓΓ    ] [xΓ] = [bΓ]          grid (Dirichlet), E = injection of Γ node (0, j)
// (A^{0i} couples Γ node (0, j) only to (h, jh) with -1: SURVEY §8 "verified stencils").
// Block elimination (the exact leading block of Eq.(5), "computed exactly"):
//     g  = bΓ - A^{i0} (A^00)^-1 b0 = bΓ + [L00^-1 b0]_{i=1}            (K cancels)
//     xΓ = S^-1 g                                                        (Schur PCG, dd_pcg_solve)
//     x0 = (A^00)^-1 (b0 - A^{0i} xΓ) = L00^-1 (b0 / K + E xΓ).
// L00^-1 by full-field fast diagonalisation: L00 = (S ⊗ S) diag(σ_a + σ_b) (S ⊗ S), S the
// orthonormal DST-I (S_dst, the left half of the 2D handle's W), applied to a field Y (row-major,
// rows = x index i, padded to ldf = Kpad) as two batched DMMA slab passes Out = (Y S)^T, each an
// n x n x Kpad GEMM per right-hand side.  With Ŷ = (S B0 S) / Σ:
//     [L00^-1 b0]_{i=1, j} = Σ_b (Σ_a s1_a Ŷ_ab) S_bj,    s1 = S[1, :]
//     x̂0 = Ŷ / K + (s1 ⊗ S xΓ) / Σ     (the transform of E xΓ is the rank-1 s1 (S xΓ)^T)
// so the whole solve is 4 slab passes, two skinny GEMMs and elementwise kernels.
#include "dd_internal.h"
#include "dgemm_tile.cuh"

namespace dd {

using CfgBulk = DgemmCfg<64, 64, 16, 2, 2, 4, 2>;

struct EpiBulkStore {          // Out[b] (slab b, row-major transposed store) = v · w[row + col ldf] (w optional)
    double* out; long long sC; int ldf; const double* w;
    __device__ __forceinline__ void operator()(int b, int row, int col, double v) const {
        const size_t i = row + (size_t)col * ldf;
        out[(size_t)b * sC + i] = w ? v * w[i] : v;
    }
};

// Out = (Y S)^T per slab: Y row-major ldf x ldf (rows >= n zero), S symmetric with row stride lds.
cudaError_t bulk_slab_pass(const double* in, double* out, int nslab, int n, int ldf, const double* S, int lds,
                           const double* w, cudaStream_t st) {
    DgemmProblem g{n, n, ldf, in, ldf, S, lds};
    g.sA = (long long)ldf * ldf;
    g.sB = 0;
    g.batch = nslab;
    g.a_static = 0;
    return dgemm_launch<CfgBulk>(g, 1, EpiBulkStore{out, (long long)ldf * ldf, ldf, w}, st);
}

// b (column c at c*ldb: [b0 (n x n, i-major), bΓ (n)]) -> slab c (row-major ldf x ldf, zero
// padded) and bΓ -> gout (ld ldg)
__global__ void k_bulk_in(int n, int ldf, int ncols, const double* __restrict__ b, long long ldb, double* __restrict__ slab,
                          double* __restrict__ gout, int ldg) {
    const long long NP = (long long)ldf * ldf;
    const long long total = NP * ncols;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(idx / NP);
        const int r = (int)(idx % NP);
        const int i = r / ldf, j = r % ldf;
        slab[idx] = (i < n && j < n) ? b[(size_t)c * ldb + (size_t)i * n + j] : 0.0;
        if (i == 0 && j < ldg) gout[(size_t)c * ldg + j] = j < n ? b[(size_t)c * ldb + (size_t)n * n + j] : 0.0;
    }
}

// w_c[b] = Σ_a s1[a] Ŷ_c[a][b]  (fixed a order; one thread per (c, b))
__global__ void k_bulk_row1(int n, int ldf, int ncols, const double* __restrict__ Yh, const double* __restrict__ s1,
                            double* __restrict__ w, int ldw) {
    const long long NP = (long long)ldf * ldf;
    const int total = ncols * ldf;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const int c = idx / ldf, bb = idx % ldf;
        double acc = 0.0;
        if (bb < n) {
            const double* y = Yh + (size_t)c * NP + bb;
            for (int a = 0; a < n; a++) acc = fma(s1[a], y[(size_t)a * ldf], acc);
        }
        w[(size_t)c * ldw + bb] = acc;
    }
}

// x̂_c[a][b] = Ŷ_c[a][b] / K_c + s1[a] u_c[b] Σinv[a][b]
__global__ void k_bulk_update(int n, int ldf, int ncols, double* __restrict__ Yh, const double* __restrict__ s1,
                              const double* __restrict__ u, int ldu, const double* __restrict__ sinv,
                              const int* __restrict__ col_param, int n_param, const double* __restrict__ Kp) {
    const long long NP = (long long)ldf * ldf;
    const long long total = NP * ncols;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(idx / NP);
        const int r = (int)(idx % NP);
        const int a = r / ldf, bb = r % ldf;
        if (a >= n || bb >= n) continue;
        int p = col_param[c];
        p = p < 0 ? 0 : (p >= n_param ? n_param - 1 : p);
        Yh[idx] = fma(s1[a] * u[(size_t)c * ldu + bb], sinv[r], Yh[idx] / Kp[p]);
    }
}

// x (column c at c*ldx: [x0 (n x n), xΓ (n)]) <- slab c and xΓ (ld ldg)
__global__ void k_bulk_out(int n, int ldf, int ncols, const double* __restrict__ slab, const double* __restrict__ xg,
                           int ldg, double* __restrict__ x, long long ldx) {
    const long long per = (long long)n * n + n;
    const long long total = per * ncols;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(idx / per);
        const long long r = idx % per;
        double v;
        if (r < (long long)n * n) {
            const int i = (int)(r / n), j = (int)(r % n);
            v = slab[(size_t)c * ldf * ldf + (size_t)i * ldf + j];
        } else {
            v = xg[(size_t)c * ldg + (r - (long long)n * n)];
        }
        x[(size_t)c * ldx + r] = v;
    }
}

static int grid_for(long long total) {
    long long b = (total + 255) / 256;
    return (int)(b > 148 * 16 ? 148 * 16 : (b < 1 ? 1 : b));
}

cudaError_t bulk_in(int n, int ldf, int ncols, const double* b, long long ldb, double* slab, double* gout, int ldg,
                    cudaStream_t st) {
    k_bulk_in<<<grid_for((long long)ldf * ldf * ncols), 256, 0, st>>>(n, ldf, ncols, b, ldb, slab, gout, ldg);
    return cudaGetLastError();
}
cudaError_t bulk_row1(int n, int ldf, int ncols, const double* Yh, const double* s1, double* w, int ldw,
                      cudaStream_t st) {
    k_bulk_row1<<<grid_for((long long)ncols * ldf), 256, 0, st>>>(n, ldf, ncols, Yh, s1, w, ldw);
    return cudaGetLastError();
}
cudaError_t bulk_update(int n, int ldf, int ncols, double* Yh, const double* s1, const double* u, int ldu,
                        const double* sinv, const int* col_param, int n_param, const double* Kp, cudaStream_t st) {
    k_bulk_update<<<grid_for((long long)ldf * ldf * ncols), 256, 0, st>>>(n, ldf, ncols, Yh, s1, u, ldu, sinv,
                                                                         col_param, n_param, Kp);
    return cudaGetLastError();
}
cudaError_t bulk_out(int n, int ldf, int ncols, const double* slab, const double* xg, int ldg, double* x, long long ldx,
                     cudaStream_t st) {
    k_bulk_out<<<grid_for(((long long)n * n + n) * ncols), 256, 0, st>>>(n, ldf, ncols, slab, xg, ldg, x, ldx);
    return cudaGetLastError();
}

}  // namespace dd

// ------------------------------------------------------------------------------------------------
// PCG on the bulk system with the DD preconditioner Eq.(5) (the
// paper's own protocol).  Bulk vectors use the dd_bulk_solve layout
// (column c at c*nb: interior nodes x-major, then Γ), nb = n^2 + n.
namespace dd {

// y = 𝒜 x = K A_h x + γ T^T F T x:   interior rows: K (4 x_ij - x_i±1,j - x_i,j±1) (i = 1 couples
// to the Γ node (0, j)); Γ rows: K (2 x_j - x_j±1 / 2 - x_1j) + γ (F xΓ)_j  (SURVEY §8 verified
// stencils; Dirichlet elsewhere).  fx: F xΓ (ld ldfx), computed by the GEMM core beforehand.
__global__ void k_bulk_apply(int n, int ncols, const double* __restrict__ x, long long nb, const double* __restrict__ fx,
                             int ldfx, const int* __restrict__ col_param, int n_param, const double* __restrict__ Kp,
                             const double* __restrict__ gp, double* __restrict__ y) {
    const long long total = nb * ncols;
    const long long nn = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(idx / nb);
        const long long r = idx % nb;
        int p = col_param[c];
        p = p < 0 ? 0 : (p >= n_param ? n_param - 1 : p);
        const double* xc = x + (size_t)c * nb;
        const double* xg = xc + nn;
        double v;
        if (r < nn) {
            const int i = (int)(r / n), j = (int)(r % n);
            const double up = i > 0 ? xc[r - n] : xg[j];            // i = 1 row couples to Γ node (0, j)
            const double dn = i + 1 < n ? xc[r + n] : 0.0;
            const double lf = j > 0 ? xc[r - 1] : 0.0;
            const double rt = j + 1 < n ? xc[r + 1] : 0.0;
            v = Kp[p] * (4.0 * xc[r] - up - dn - lf - rt);
        } else {
            const int j = (int)(r - nn);
            const double lf = j > 0 ? xg[j - 1] : 0.0;
            const double rt = j + 1 < n ? xg[j + 1] : 0.0;
            v = fma(gp[p], fx[(size_t)c * ldfx + j], Kp[p] * (2.0 * xg[j] - 0.5 * (lf + rt) - xc[j]));
        }
        y[(size_t)c * nb + r] = v;
    }
}

__device__ __forceinline__ double bpcg_block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); q++) s += red[q];   // fixed order: deterministic
    __syncthreads();
    return s;
}

// one CTA per column: α = ρ / p·q; x += α p; r -= α q  (active columns)
__global__ void k_bpcg_a(long long nb, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                         const double* __restrict__ q, const double* __restrict__ rho, int* __restrict__ active,
                         int* __restrict__ status) {
    __shared__ double red[32];
    const int c = blockIdx.x;
    if (!active[c]) return;
    const size_t off = (size_t)c * nb;
    double pq = 0.0;
    for (long long i = threadIdx.x; i < nb; i += blockDim.x) pq = fma(p[off + i], q[off + i], pq);
    pq = bpcg_block_sum(pq, red);
    if (!(pq > 0.0)) {
        if (threadIdx.x == 0) { atomicExch(status, (int)DD_ENOTSPD); active[c] = 0; }
        return;
    }
    const double alpha = rho[c] / pq;
    for (long long i = threadIdx.x; i < nb; i += blockDim.x) {
        x[off + i] = fma(alpha, p[off + i], x[off + i]);
        r[off + i] = fma(-alpha, q[off + i], r[off + i]);
    }
}

// one CTA per column after z = B r:  ρ' = r·z; η test; β = ρ'/ρ; p = z + β p.  init: p = z, η0.
__global__ void k_bpcg_b(long long nb, const double* __restrict__ r, const double* __restrict__ z, double* __restrict__ p,
                         double* __restrict__ rho, double* __restrict__ eta0, double* __restrict__ relres,
                         int* __restrict__ active, int* __restrict__ iters, int k, double rtol, int maxit, int init,
                         int* __restrict__ n_active, int* __restrict__ status) {
    __shared__ double red[32];
    const int c = blockIdx.x;
    if (!init && !active[c]) return;
    const size_t off = (size_t)c * nb;
    double rz = 0.0;
    for (long long i = threadIdx.x; i < nb; i += blockDim.x) rz = fma(r[off + i], z[off + i], rz);
    rz = bpcg_block_sum(rz, red);
    const double eta = sqrt(fmax(rz, 0.0));
    if (init) {
        for (long long i = threadIdx.x; i < nb; i += blockDim.x) p[off + i] = z[off + i];
        if (threadIdx.x == 0) {
            eta0[c] = eta; rho[c] = rz; iters[c] = 0; relres[c] = eta > 0.0 ? 1.0 : 0.0;
            if (rz < 0.0) atomicExch(status, (int)DD_ENOTSPD);
            const bool act = eta > 0.0 && rz >= 0.0;
            active[c] = act;
            if (act) atomicAdd(n_active, 1);
        }
        return;
    }
    const bool conv = eta <= rtol * eta0[c];
    if (threadIdx.x == 0) {
        iters[c] = k;
        relres[c] = eta0[c] > 0.0 ? eta / eta0[c] : 0.0;
        if (rz < 0.0) atomicExch(status, (int)DD_ENOTSPD);
    }
    if (conv || rz < 0.0 || k >= maxit) {
        if (threadIdx.x == 0) active[c] = 0;
        return;
    }
    const double beta = rz / rho[c];
    for (long long i = threadIdx.x; i < nb; i += blockDim.x) p[off + i] = fma(beta, p[off + i], z[off + i]);
    __syncthreads();
    if (threadIdx.x == 0) { rho[c] = rz; atomicAdd(n_active, 1); }
}

cudaError_t bulk_apply(int n, int ncols, const double* x, long long nb, const double* fx, int ldfx, const int* col_param,
                       int n_param, const double* Kp, const double* gp, double* y, cudaStream_t st) {
    k_bulk_apply<<<grid_for(nb * ncols), 256, 0, st>>>(n, ncols, x, nb, fx, ldfx, col_param, n_param, Kp, gp, y);
    return cudaGetLastError();
}
// ---- long columns, few of them (3D bulk: 2 M entries x 8 columns): NBLK CTAs per column; the
// dot products go through per-CTA partials summed in CTA order (deterministic), the scalar
// recurrences run in one thread per column
constexpr int NBLK = 64;
__global__ void k_coldot(long long nb, const double* __restrict__ a, const double* __restrict__ b,
                         const int* __restrict__ active, int all, double* __restrict__ part) {
    __shared__ double red[32];
    const int c = blockIdx.y, blk = blockIdx.x;
    if (!all && !active[c]) return;
    const long long chunk = (nb + NBLK - 1) / NBLK, i0 = blk * chunk, i1 = min(nb, i0 + chunk);
    const size_t off = (size_t)c * nb;
    double s = 0.0;
    for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) s = fma(a[off + i], b[off + i], s);
    s = bpcg_block_sum(s, red);
    if (threadIdx.x == 0) part[(size_t)c * NBLK + blk] = s;
}
__device__ __forceinline__ double part_sum(const double* part, int c) {
    double s = 0.0;
    for (int b = 0; b < NBLK; b++) s += part[(size_t)c * NBLK + b];
    return s;
}
__global__ void k_bpcg_a2(long long nb, double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                          const double* __restrict__ q, const double* __restrict__ rho, int* __restrict__ active,
                          int* __restrict__ status, const double* __restrict__ part) {
    const int c = blockIdx.y, blk = blockIdx.x;
    if (!active[c]) return;
    const double pq = part_sum(part, c);
    if (!(pq > 0.0)) {
        if (blk == 0 && threadIdx.x == 0) { atomicExch(status, (int)DD_ENOTSPD); active[c] = 0; }
        return;
    }
    const double alpha = rho[c] / pq;
    const long long chunk = (nb + NBLK - 1) / NBLK, i0 = blk * chunk, i1 = min(nb, i0 + chunk);
    const size_t off = (size_t)c * nb;
    for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        x[off + i] = fma(alpha, p[off + i], x[off + i]);
        r[off + i] = fma(-alpha, q[off + i], r[off + i]);
    }
}
// scalar step of k_bpcg_b per column: beta[c] = β (update p) or NaN (frozen / init)
__global__ void k_bpcg_b2(int ncols, double* __restrict__ rho, double* __restrict__ eta0, double* __restrict__ relres,
                          int* __restrict__ active, int* __restrict__ iters, int k, double rtol, int maxit, int init,
                          int* __restrict__ n_active, int* __restrict__ status, const double* __restrict__ part,
                          double* __restrict__ beta) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= ncols) return;
    beta[c] = __longlong_as_double(0x7ff8000000000000ll);
    if (!init && !active[c]) return;
    const double rz = part_sum(part, c);
    const double eta = sqrt(fmax(rz, 0.0));
    if (init) {
        eta0[c] = eta; rho[c] = rz; iters[c] = 0; relres[c] = eta > 0.0 ? 1.0 : 0.0;
        if (rz < 0.0) atomicExch(status, (int)DD_ENOTSPD);
        const bool act = eta > 0.0 && rz >= 0.0;
        active[c] = act;
        if (act) atomicAdd(n_active, 1);
        return;
    }
    const bool conv = eta <= rtol * eta0[c];
    iters[c] = k;
    relres[c] = eta0[c] > 0.0 ? eta / eta0[c] : 0.0;
    if (rz < 0.0) atomicExch(status, (int)DD_ENOTSPD);
    if (conv || rz < 0.0 || k >= maxit) { active[c] = 0; return; }
    beta[c] = rz / rho[c];
    rho[c] = rz;
    atomicAdd(n_active, 1);
}
__global__ void k_bpcg_b3(long long nb, const double* __restrict__ z, double* __restrict__ p, int init,
                          const double* __restrict__ beta) {
    const int c = blockIdx.y, blk = blockIdx.x;
    const double bt = beta[c];
    if (!init && isnan(bt)) return;
    const long long chunk = (nb + NBLK - 1) / NBLK, i0 = blk * chunk, i1 = min(nb, i0 + chunk);
    const size_t off = (size_t)c * nb;
    for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x)
        p[off + i] = init ? z[off + i] : fma(bt, p[off + i], z[off + i]);
}
static bool bpcg_wide(int ncols, long long nb) { return ncols < 148 && nb >= (1ll << 18); }
static double* bpcg_ws(int ncols) {
    static double* ws = nullptr;
    static int cap = 0;
    if (ncols > cap) {
        if (ws) cudaFree(ws);
        cap = ncols < 64 ? 64 : ncols;
        if (cudaMalloc(&ws, sizeof(double) * (size_t)cap * (NBLK + 1)) != cudaSuccess) { ws = nullptr; cap = 0; }
    }
    return ws;
}

cudaError_t bpcg_a(int ncols, long long nb, double* x, double* r, const double* p, const double* q, const double* rho,
                   int* active, int* status, cudaStream_t st) {
    if (bpcg_wide(ncols, nb)) {
        double* part = bpcg_ws(ncols);
        if (!part) return cudaErrorMemoryAllocation;
        k_coldot<<<dim3(NBLK, ncols), 512, 0, st>>>(nb, p, q, active, 0, part);
        k_bpcg_a2<<<dim3(NBLK, ncols), 512, 0, st>>>(nb, x, r, p, q, rho, active, status, part);
        return cudaGetLastError();
    }
    k_bpcg_a<<<ncols, 1024, 0, st>>>(nb, x, r, p, q, rho, active, status);
    return cudaGetLastError();
}
cudaError_t bpcg_b(int ncols, long long nb, const double* r, const double* z, double* p, double* rho, double* eta0,
                   double* relres, int* active, int* iters, int k, double rtol, int maxit, int init, int* n_active,
                   int* status, cudaStream_t st) {
    if (bpcg_wide(ncols, nb)) {
        double* part = bpcg_ws(ncols);
        if (!part) return cudaErrorMemoryAllocation;
        double* beta = part + (size_t)ncols * NBLK;
        k_coldot<<<dim3(NBLK, ncols), 512, 0, st>>>(nb, r, z, active, init, part);
        k_bpcg_b2<<<(ncols + 127) / 128, 128, 0, st>>>(ncols, rho, eta0, relres, active, iters, k, rtol, maxit, init,
                                                      n_active, status, part, beta);
        k_bpcg_b3<<<dim3(NBLK, ncols), 512, 0, st>>>(nb, z, p, init, beta);
        return cudaGetLastError();
    }
    k_bpcg_b<<<ncols, 1024, 0, st>>>(nb, r, z, p, rho, eta0, relres, active, iters, k, rtol, maxit, init, n_active,
                                      status);
    return cudaGetLastError();
}

}  // namespace dd
