// Full DD solve on a bulk right-hand side, 3D (Eq.(5) with
// the exact leading block, 229-230): block elimination
//     g = b_Γ - A^{i0}(A^00)^-1 b_0,   x_Γ = S^-1 g,   x_0 = (A^00)^-1 (b_0 - A^{0i} x_Γ)
// on the Kuhn mesh of (0,1)^3, Γ = {x = 0}.  The interior block is K h (T ⊕ T ⊕ T) (the 7-point
// stencil) and the Γ coupling is -K h on the first layer, so with L = T ⊕ T ⊕ T
//     g = b_Γ + (L^-1 b_0)|_{i=1},        x_0 = L^-1 (b_0 / (K h) + e_1 ⊗ x_Γ),
// and L^-1 = (Q⊗Q⊗Q) diag(1/(σ_a+σ_b+σ_c)) (Q⊗Q⊗Q) by full-field fast diagonalisation (Q the
// orthonormal DST-I, σ = 4 sin^2(θ/2)).  The two face axes are the face slab passes of the Schur
// apply (batched DMMA over (column, layer) faces); the normal axis is one batched DMMA GEMM per
// column over a [column][face][layer] copy that the second face pass writes directly.
#include "dd_internal.h"
#include "dgemm_tile.cuh"

namespace dd {

namespace {
using CfgB3 = DgemmCfg<64, 64, 16, 2, 2, 4, 2>;

// face pass writing the [column][face][layer] layout (layer contiguous, row stride lk)
struct EpiToLayerMajor {
    double* out; int n, ldf, lk; long long NP;
    __device__ __forceinline__ void operator()(int b, int row, int col, double v) const {
        const int c = b / n, i = b % n;
        out[((size_t)c * NP + row + (size_t)col * ldf) * lk + i] = v;
    }
};
// normal-axis transform: C[face][a] -> out[c][a][face], optionally / (σ_a + σ_j + σ_k)
struct EpiNormal {
    double* out; int n, ldf; long long NP; const double* sig; int scale;
    __device__ __forceinline__ void operator()(int c, int face, int a, double v) const {
        const int j = face % ldf, k = face / ldf;       // face = j + k ldf (column-major face store)
        if (j >= n || k >= n) return;
        out[((size_t)c * n + a) * NP + face] = scale ? v / (sig[a] + sig[j] + sig[k]) : v;
    }
};
}  // namespace

// one face pass over nslab faces whose output goes to the layer-major layout
static cudaError_t face_pass_to_layer_major(const double* in, double* out, int nslab, int n, int ldf, int lk,
                                            long long NP, const double* S, cudaStream_t st) {
    DgemmProblem g{n, n, ldf, in, ldf, S, ldf};
    g.sA = (long long)ldf * ldf;
    g.sB = 0;
    g.batch = nslab;
    return dgemm_launch_s<CfgB3, EpiToLayerMajor, 1>(g, EpiToLayerMajor{out, n, ldf, lk, NP}, st, false);
}

// out[c][a][face] = Σ_i S[a][i] in[c][face][i]  (rows = faces, K = layers padded to lk)
static cudaError_t normal_pass(const double* in, double* out, int ncols, int n, int ldf, int lk, long long NP,
                               const double* S, const double* sig, bool scale, cudaStream_t st) {
    DgemmProblem g{(int)NP, n, lk, in, lk, S, ldf};
    g.sA = NP * lk;
    g.sB = 0;
    g.batch = ncols;
    return dgemm_launch_s<CfgB3, EpiNormal, 1>(g, EpiNormal{out, n, ldf, NP, sig, scale ? 1 : 0}, st, false);
}

// product layout -> padded faces: interior b_0 (scaled by s_c) into X[c][i][face]; b_Γ into G[c][face]
__global__ void k_b3_in(int n, int ldf, long long NP, int ncols, const double* __restrict__ b, long long ldb,
                        double* __restrict__ X, double* __restrict__ G) {
    const long long n2 = (long long)n * n, n3 = n2 * n;
    const long long per = n3 + n2;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < per * ncols;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long c = idx / per, e = idx % per;
        const double v = b[c * ldb + e];
        if (e < n3) {
            const long long i = e / n2, jk = e % n2;
            const int j = (int)(jk / n), k = (int)(jk % n);
            X[(c * n + i) * NP + j * ldf + k] = v;      // face (j, k): row j, column k of a ldf x ldf face
        } else {
            const long long jk = e - n3;
            G[c * NP + (jk / n) * ldf + jk % n] = v;
        }
    }
}
// w[c][face] = Σ_a s1_a Ŷ[c][a][face]   (s1 = row 1 of Q: the first interior layer)
__global__ void k_b3_layer1(int n, long long NP, int ncols, const double* __restrict__ Y, const double* __restrict__ s1,
                            double* __restrict__ w) {
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < NP * ncols;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long c = idx / NP, f = idx % NP;
        double acc = 0.0;
        for (int a = 0; a < n; a++) acc = fma(s1[a], Y[(c * n + a) * NP + f], acc);
        w[idx] = acc;
    }
}
// x̂_0[c][a][face] = Ŷ / (K_c h) + s1_a X̂_Γ[c][face] / (σ_a + σ_j + σ_k)
__global__ void k_b3_combine(int n, int ldf, long long NP, int ncols, double* __restrict__ Y,
                             const double* __restrict__ XG, const double* __restrict__ s1, const double* __restrict__ sig,
                             const int* __restrict__ col_param, int n_param, const double* __restrict__ Kp, double h) {
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)ncols * n * NP;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long f = idx % NP, ca = idx / NP;
        const int a = (int)(ca % n), c = (int)(ca / n);
        const int j = (int)(f % ldf), k = (int)(f / ldf);
        if (j >= n || k >= n) continue;
        int p = col_param[c];
        p = p < 0 ? 0 : (p >= n_param ? n_param - 1 : p);
        Y[idx] = Y[idx] / (Kp[p] * h) + s1[a] * XG[(long long)c * NP + f] / (sig[a] + sig[j] + sig[k]);
    }
}
// g (user face layout, n^2 per column) = b_Γ + w
__global__ void k_b3_g(int n, int ldf, long long NP, int ncols, const double* __restrict__ G, const double* __restrict__ W,
                       double* __restrict__ g) {
    const long long n2 = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n2 * ncols;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long c = idx / n2, jk = idx % n2;
        const long long f = (jk / n) * ldf + jk % n;
        g[idx] = G[c * NP + f] + W[c * NP + f];
    }
}
// x_Γ (user face layout, column stride lds) -> padded faces
__global__ void k_b3_pad(int n, int ldf, long long NP, int ncols, const double* __restrict__ xg, long long lds,
                         double* __restrict__ P) {
    const long long n2 = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n2 * ncols;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long c = idx / n2, jk = idx % n2;
        P[c * NP + (jk / n) * ldf + jk % n] = xg[c * lds + jk];
    }
}
// padded x_0 faces and x_Γ -> product layout
__global__ void k_b3_out(int n, int ldf, long long NP, int ncols, const double* __restrict__ X,
                         const double* __restrict__ xg, double* __restrict__ x, long long ldx) {
    const long long n2 = (long long)n * n, n3 = n2 * n;
    const long long per = n3 + n2;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < per * ncols;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long c = idx / per, e = idx % per;
        if (e < n3) {
            const long long i = e / n2, jk = e % n2;
            x[c * ldx + e] = X[(c * n + i) * NP + (jk / n) * ldf + jk % n];
        } else {
            x[c * ldx + e] = xg[c * n2 + (e - n3)];
        }
    }
}

// out = 𝒜 x on the bulk product layout: K h (7-point interior stencil; Γ rows 3, -1/2 in-face,
// -1 to the first layer) + γ F x_Γ on the Γ rows (fx: padded faces, γ already applied)
__global__ void k_b3_apply(int n, int ldf, long long NP, int ncols, const double* __restrict__ x, long long ldx,
                           const double* __restrict__ fx, const int* __restrict__ col_param, int n_param,
                           const double* __restrict__ Kp, double h, double* __restrict__ out) {
    const long long n2 = (long long)n * n, n3 = n2 * n;
    const long long per = n3 + n2;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < per * ncols;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long c = idx / per, e = idx % per;
        const double* xc = x + c * ldx;
        int p = col_param[c];
        p = p < 0 ? 0 : (p >= n_param ? n_param - 1 : p);
        const double Kh = Kp[p] * h;
        if (e < n3) {
            const int i = (int)(e / n2), j = (int)((e % n2) / n), k = (int)(e % n);
            double v = 6.0 * xc[e];
            v -= i > 0 ? xc[e - n2] : xc[n3 + (long long)j * n + k];          // i = 1 couples to Γ
            if (i + 1 < n) v -= xc[e + n2];
            if (j > 0) v -= xc[e - n];
            if (j + 1 < n) v -= xc[e + n];
            if (k > 0) v -= xc[e - 1];
            if (k + 1 < n) v -= xc[e + 1];
            out[c * ldx + e] = Kh * v;
        } else {
            const long long jk = e - n3;
            const int j = (int)(jk / n), k = (int)(jk % n);
            const double* g = xc + n3;
            double v = 3.0 * g[jk] - xc[jk];                                   // xc[jk]: layer 1, same (j, k)
            double nb = 0.0;
            if (j > 0) nb += g[jk - n];
            if (j + 1 < n) nb += g[jk + n];
            if (k > 0) nb += g[jk - 1];
            if (k + 1 < n) nb += g[jk + 1];
            v -= 0.5 * nb;
            out[c * ldx + e] = fma(Kh, v, fx[c * NP + (long long)j * ldf + k]);
        }
    }
}

static int grid_of(long long total) {
    long long b = (total + 255) / 256;
    return (int)(b < 1 ? 1 : (b > 148 * 16 ? 148 * 16 : b));
}

// L^-1 applied in mode space: in X (physical, [c][i][face]) -> Y (modes / Σ, [c][a][face]);
// T: face-pass scratch ([c][i][face]); Lk: [c][face][layer] scratch
cudaError_t bulk3_forward(int n, int ldf, int lk, long long NP, int ncols, const double* S, const double* sig,
                          const double* X, double* T, double* Lk, double* Y, cudaStream_t st) {
    cudaError_t e = face_slab_pass(X, T, ncols * n, n, ldf, S, st);
    if (e == cudaSuccess) e = face_pass_to_layer_major(T, Lk, ncols * n, n, ldf, lk, NP, S, st);
    if (e == cudaSuccess) e = normal_pass(Lk, Y, ncols, n, ldf, lk, NP, S, sig, true, st);
    return e;
}
// mode space -> physical (no scaling): in Y ([c][a][face]) -> X ([c][i][face])
cudaError_t bulk3_inverse(int n, int ldf, int lk, long long NP, int ncols, const double* S, const double* Y, double* T,
                          double* Lk, double* X, cudaStream_t st) {
    cudaError_t e = face_slab_pass(Y, T, ncols * n, n, ldf, S, st);
    if (e == cudaSuccess) e = face_pass_to_layer_major(T, Lk, ncols * n, n, ldf, lk, NP, S, st);
    if (e == cudaSuccess) e = normal_pass(Lk, X, ncols, n, ldf, lk, NP, S, nullptr, false, st);
    return e;
}
cudaError_t bulk3_in(int n, int ldf, long long NP, int ncols, const double* b, long long ldb, double* X, double* G,
                     cudaStream_t st) {
    const long long per = (long long)n * n * n + (long long)n * n;
    k_b3_in<<<grid_of(per * ncols), 256, 0, st>>>(n, ldf, NP, ncols, b, ldb, X, G);
    return cudaGetLastError();
}
cudaError_t bulk3_layer1(int n, long long NP, int ncols, const double* Y, const double* s1, double* w, cudaStream_t st) {
    k_b3_layer1<<<grid_of(NP * ncols), 256, 0, st>>>(n, NP, ncols, Y, s1, w);
    return cudaGetLastError();
}
cudaError_t bulk3_g(int n, int ldf, long long NP, int ncols, const double* G, const double* W, double* g, cudaStream_t st) {
    k_b3_g<<<grid_of((long long)n * n * ncols), 256, 0, st>>>(n, ldf, NP, ncols, G, W, g);
    return cudaGetLastError();
}
cudaError_t bulk3_pad(int n, int ldf, long long NP, int ncols, const double* xg, long long lds, double* P,
                      cudaStream_t st) {
    k_b3_pad<<<grid_of((long long)n * n * ncols), 256, 0, st>>>(n, ldf, NP, ncols, xg, lds, P);
    return cudaGetLastError();
}
cudaError_t bulk3_combine(int n, int ldf, long long NP, int ncols, double* Y, const double* XG, const double* s1,
                          const double* sig, const int* col_param, int n_param, const double* Kp, double h,
                          cudaStream_t st) {
    k_b3_combine<<<grid_of((long long)ncols * n * NP), 256, 0, st>>>(n, ldf, NP, ncols, Y, XG, s1, sig, col_param,
                                                                      n_param, Kp, h);
    return cudaGetLastError();
}
cudaError_t bulk3_apply(int n, int ldf, long long NP, int ncols, const double* x, long long ldx, const double* fx,
                        const int* col_param, int n_param, const double* Kp, double h, double* out, cudaStream_t st) {
    const long long per = (long long)n * n * n + (long long)n * n;
    k_b3_apply<<<grid_of(per * ncols), 256, 0, st>>>(n, ldf, NP, ncols, x, ldx, fx, col_param, n_param, Kp, h, out);
    return cudaGetLastError();
}
cudaError_t bulk3_out(int n, int ldf, long long NP, int ncols, const double* X, const double* xg, double* x, long long ldx,
                      cudaStream_t st) {
    const long long per = (long long)n * n * n + (long long)n * n;
    k_b3_out<<<grid_of(per * ncols), 256, 0, st>>>(n, ldf, NP, ncols, X, xg, x, ldx);
    return cudaGetLastError();
}

}  // namespace dd
