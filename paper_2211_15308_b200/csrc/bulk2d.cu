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
