// 3D path (Γ = face {x = 0} of the unit cube, SURVEY §8(a) rows a-2..a-6 for config 4).
//
// Face vectors live in a padded layout: column c, node (j, k) (1-based grid indices j, k <= n)
// at c*NP + (j-1)*ldf + (k-1), ldf = round_up(n, 16), NP = ldf^2, padding zero.
//
// * Interior solve (row a-2): the 2D sine transform of a face slab, X̂ = S X S, is two batched
//   DMMA GEMM passes Out = (Y S^T)^T (dgemm_tile.cuh, batch = columns); the Schur weights
//   s_ab = h(3 - cos θ_a - cos θ_b) - h Σ_m S[1,m]^2/(σ_m + σ_a + σ_b) scale X̂ in the second
//   pass's epilogue, and two more passes transform back.
// * Fractional term (row a-3): q = γ F p + (back transform) as one stream-K DMMA GEMM with
//   BN = 8 columns (HBM-bound: F is read once per apply).
// * Pole sum (row a-4, 2D Γ): every system (A_Γ - p_k M_Γ) (5-point A, 7-point consistent mass)
//   and M_Γ is solved by batched preconditioned CG over all (system, column) pairs; the
//   preconditioner is the sine-diagonal part of the pair, 1/(α_ab - p μ̃_ab) with
//   α = σ_a + σ_b and μ̃ = (h^2/12)(6 + 2c_a + 2c_b + 2 c_a c_b) (spectrally equivalent, κ <= 3,
//   SURVEY V10), applied with the same slab transforms.  Converged pairs freeze.
//   The weighted sum over systems runs in fixed system order; across ranks (pole split) the
//   partial sums are added by one NCCL allreduce (row a-6, in dd_api.cpp).
#include <algorithm>
#include <cstdlib>

#include "dd_internal.h"
#include "dgemm_tile.cuh"
#include <cooperative_groups.h>

namespace dd {

using CfgSlab = DgemmCfg<64, 64, 16, 2, 2, 4, 2>;
// F x for a handful of columns (HBM-bound stream of F): 256 rows x 8 cols x 32-deep stages, 8 warps,
// one 223 KB CTA per SM — 5.86 TB/s (91 % of the measured HBM copy rate) vs 4.80 TB/s for the
// earlier 128x8x16, 2 CTAs/SM (tools/gemm_lab6.cu)
using CfgFv = DgemmCfg<256, 8, 32, 8, 1, 3, 1>;
constexpr int OCC_FV = 1;

// ------------------------------------------------------------------------------------ epilogues
struct EpiSlabStore {          // Out[b] (col-major, ldc = ldf) = v   (staged: 16-byte row-pair stores)
    double* out; long long sC; int ldf;
    static constexpr bool kStaged = true;
    struct Blk {};
    struct Ctx {};
    __device__ __forceinline__ void operator()(int b, int row, int col, double v) const {   // split-K form
        out[(size_t)b * sC + row + (size_t)col * ldf] = v;
    }
    __device__ __forceinline__ Blk block(int) const { return {}; }
    __device__ __forceinline__ void load(int, int, int, const Blk&, Ctx&) const {}
    __device__ __forceinline__ void store(int b, int row, int col, bool pair, const Blk&, const Ctx&, double2 v) const {
        double* o = out + (size_t)b * sC + row + (size_t)col * ldf;
        if (pair) *reinterpret_cast<double2*>(o) = v;
        else o[0] = v.x;
    }
};
struct EpiSlabScale {          // Out[b] = v * scale(b) * w[b's table][row + col ldf]
    double* out; long long sC; int ldf;
    const double* w; long long sW;          // weight table per slab group (sW = 0: shared)
    int group;                              // slabs b share table b / group
    const double* colscale;                 // per slab scalar (or null)
    __device__ __forceinline__ void operator()(int b, int row, int col, double v) const {
        const size_t i = row + (size_t)col * ldf;
        double s = w[(size_t)(b / group) * sW + i];
        if (colscale) s *= colscale[b];
        out[(size_t)b * sC + i] = v * s;
    }
};
struct EpiInnerOp {            // q̂_part[b] = cs[s] v,  s = b / C: the D̂ ⊗ D̂ part of the sine-domain operator; the
    double* q; const double* p; long long NP; int ldf, C;   // diagonal part dg ∘ p̂ is added where q̂ is
    const double* dg; const double* cs;                     // consumed (k_inner_update_cl), coalesced
    __device__ __forceinline__ void operator()(int b, int row, int col, double v) const {
        const int s = b / C;
        const size_t i = row + (size_t)col * ldf;
        q[(size_t)b * NP + i] = cs[s] * v;
    }
};
struct EpiInnerCheb {          // one Chebyshev step of pair b = s*C + c at element i (v = (D̂ T D̂^T)_i of x̂_j):
    double* x; double* d; const double* bh; long long NP; int ldf, C;   // r = b̂ - dg∘x̂ - cs v;
    const double* dg; const double* idg; const double* cs;              // d = c1[j] d + c2[j] idg∘r; x̂ += d
    const double* c1; const double* c2; int kstride; const int* kiter;
    static constexpr bool kStaged = true;                              // x̂, d̂ updated in place
    struct Blk { double cs, c1, c2; size_t e0, t0, b0; bool first; };   // first: step 0, d_0 = x̂_1 (not stored)
    struct Ctx { double2 x, d, b, g, ig; };
    __device__ __forceinline__ void operator()(int b, int row, int col, double v) const {   // split-K form
        const Blk k = block(b);
        const size_t i = row + (size_t)col * ldf;
        const double xv = x[k.e0 + i];
        const double r = bh[k.b0 + i] - fma(dg[k.t0 + i], xv, k.cs * v);
        const double dn = fma(k.c1, k.first ? xv : d[k.e0 + i], k.c2 * (idg[k.t0 + i] * r));
        d[k.e0 + i] = dn;
        x[k.e0 + i] = xv + dn;
    }
    __device__ __forceinline__ Blk block(int b) const {
        const int s = b / C, c = b - s * C;
        const int j = *kiter;
        return Blk{cs[s], c1[(size_t)s * kstride + j], c2[(size_t)s * kstride + j], (size_t)b * NP, (size_t)s * NP,
                   (size_t)c * NP, j == 0};
    }
    __device__ __forceinline__ void load(int, int row, int col, const Blk& k, Ctx& cx) const {
        const size_t i = row + (size_t)col * ldf;
        cx.x = *reinterpret_cast<const double2*>(x + k.e0 + i);
        cx.d = k.first ? cx.x : *reinterpret_cast<const double2*>(d + k.e0 + i);
        cx.b = __ldg(reinterpret_cast<const double2*>(bh + k.b0 + i));
        cx.g = __ldg(reinterpret_cast<const double2*>(dg + k.t0 + i));
        cx.ig = __ldg(reinterpret_cast<const double2*>(idg + k.t0 + i));
    }
    __device__ __forceinline__ void store(int, int row, int col, bool pair, const Blk& k, const Ctx& cx, double2 v) const {
        const size_t i = row + (size_t)col * ldf;
        const double r0 = cx.b.x - fma(cx.g.x, cx.x.x, k.cs * v.x), r1 = cx.b.y - fma(cx.g.y, cx.x.y, k.cs * v.y);
        const double d0 = fma(k.c1, cx.d.x, k.c2 * (cx.ig.x * r0)), d1 = fma(k.c1, cx.d.y, k.c2 * (cx.ig.y * r1));
        if (pair) {
            *reinterpret_cast<double2*>(d + k.e0 + i) = make_double2(d0, d1);
            *reinterpret_cast<double2*>(x + k.e0 + i) = make_double2(cx.x.x + d0, cx.x.y + d1);
        } else {
            d[k.e0 + i] = d0;
            x[k.e0 + i] = cx.x.x + d0;
        }
    }
};
struct EpiFaceFx {             // q[c] = γ_c v + D[c]  (padded face layout; rows offset by row0 for a row shard of F)
    double* q; const double* D; long long ldq; const int* col_param; int n_param; const double* gp; int row0;
    __device__ __forceinline__ void operator()(int, int row, int col, double v) const {
        int p = col_param[col];
        p = p < 0 ? 0 : (p >= n_param ? n_param - 1 : p);
        const size_t i = row0 + row + (size_t)col * ldq;
        const double g = gp ? gp[p] : 1.0;               // gp = NULL: the folded H (γ inside)
        q[i] = D ? fma(g, v, D[i]) : g * v;
    }
};
struct EpiFaceScatter {        // dense n^2 x n^2 product -> padded NP x NP row-major matrix
    double* F; int n, ldf; long long NP;
    __device__ __forceinline__ void operator()(int, int row, int col, double v) const {
        const size_t r = (size_t)(row / n) * ldf + row % n;
        const size_t c = (size_t)(col / n) * ldf + col % n;
        F[r * NP + c] = v;
    }
};

// split-K for small slab batches: the config-4 Schur apply transforms 8 slabs = 32 output tiles,
// a quarter of the SMs; split the K range over a cluster so that the tiles x splits reach the SM
// count (results: partials summed in fixed rank order over DSMEM)
static int slab_splitk(int nslab, int n) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    const long long tiles = (long long)nslab * ((n + CfgSlab::BM - 1) / CfgSlab::BM) * ((n + CfgSlab::BN - 1) / CfgSlab::BN);
    int sk = 1;
    while (sk < 8 && tiles * sk * 2 <= sms) sk *= 2;
    return sk;
}
cudaError_t face_slab_pass(const double* in, double* out, int nslab, int n, int ldf, const double* S, cudaStream_t st) {
    DgemmProblem g{n, n, ldf, in, ldf, S, ldf};
    g.sA = (long long)ldf * ldf;
    g.sB = 0;
    g.batch = nslab;
    return dgemm_launch<CfgSlab>(g, slab_splitk(nslab, n), EpiSlabStore{out, (long long)ldf * ldf, ldf}, st);
}

cudaError_t face_slab_pass_scaled(const double* in, double* out, int nslab, int n, int ldf, const double* S,
                                  const double* w, long long sW, int group, const double* colscale, cudaStream_t st) {
    DgemmProblem g{n, n, ldf, in, ldf, S, ldf};
    g.sA = (long long)ldf * ldf;
    g.sB = 0;
    g.batch = nslab;
    return dgemm_launch<CfgSlab>(g, slab_splitk(nslab, n), EpiSlabScale{out, (long long)ldf * ldf, ldf, w, sW, group, colscale},
                                 st);
}

// Out = (Y B^T)^T per active slab (B = D̂ for the sine-domain operator; kpar: its parity-block
// edge, see DgemmProblem::kpar)
cudaError_t face_slab_pass_active(const double* in, double* out, int nslab, int n, int ldf, const double* B,
                                  const int* active, int kpar, cudaStream_t st) {
    DgemmProblem g{n, n, ldf, in, ldf, B, ldf};
    g.sA = (long long)ldf * ldf;
    g.sB = 0;
    g.batch = nslab;
    g.active = active;
    g.kpar = kpar;
    return dgemm_launch<CfgSlab>(g, 1, EpiSlabStore{out, (long long)ldf * ldf, ldf}, st);
}
// second pass of q̂ = dg ∘ p̂ + cs D̂ p̂ D̂^T over active pairs
cudaError_t face_inner_op_pass(const double* in, double* q, const double* p, int nslab, int C, int n, int ldf,
                               const double* B, const double* dg, const double* cs, const int* active, int kpar,
                               cudaStream_t st) {
    DgemmProblem g{n, n, ldf, in, ldf, B, ldf};
    g.sA = (long long)ldf * ldf;
    g.sB = 0;
    g.batch = nslab;
    g.active = active;
    g.kpar = kpar;
    return dgemm_launch<CfgSlab>(g, 1, EpiInnerOp{q, p, (long long)ldf * ldf, ldf, C, dg, cs}, st);
}
// second pass of the Chebyshev step: the operator's D̂ ⊗ D̂ part of x̂_j, the residual and both
// updates in the epilogue (EpiInnerCheb)
cudaError_t face_inner_cheb_pass(const double* in, const InnerArgs& a, const double* bh, const double* B, int kpar,
                                 cudaStream_t st) {
    DgemmProblem g{a.n, a.n, a.ldf, in, a.ldf, B, a.ldf};
    g.sA = a.NP;
    g.sB = 0;
    g.batch = a.npair;
    g.active = a.active;
    g.kpar = kpar;
    return dgemm_launch<CfgSlab>(g, 1, EpiInnerCheb{a.x, a.p, bh, a.NP, a.ldf, a.C, a.dg, a.idg, a.cs, a.cc1, a.cc2,
                                                    a.kstride, a.kiter}, st);
}

// q = γ F p + D over ncols columns (F: NP x NP row-major padded; vectors NP per column).
size_t face_fx_ws_doubles(long long NP, int ncols, int num_sms) {
    return dgemm_streamk_ws_doubles<CfgFv>((int)NP, ncols, num_sms * OCC_FV);
}
// rows [row0, row0 + rows) of q only, F = those rows of the full operator (row-sharded F, §8(e))
cudaError_t face_fx(const double* F, long long NP, const double* p, double* q, const double* D, int ncols,
                    const int* col_param, int n_param, const double* gp, double* ws, int* counters, int num_sms,
                    cudaStream_t st, int row0, int rows) {
    if (rows < 0) rows = (int)NP;
    DgemmProblem g{rows, ncols, (int)NP, F, (int)NP, p, (int)NP};
    StreamK sk{ws, counters, 0};
    const int G = dgemm_streamk_grid<CfgFv>(rows, ncols, (int)NP, num_sms, OCC_FV);
    return dgemm_launch_streamk<CfgFv>(g, G, sk, EpiFaceFx{q, D, NP, col_param, n_param, gp, row0}, st);
}

// Row-sharded F: rank rows [r0, r0 + rows) of each column packed contiguously (count rows_max per
// column, zero padded) for ncclAllGather, and the gathered blocks scattered back into the columns
__global__ void k_fx_pack(const double* __restrict__ q, long long NP, int ncols, int r0, int rows, int rows_max,
                          double* __restrict__ buf) {
    const long long tot = (long long)ncols * rows_max;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot; idx += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(idx / rows_max), i = (int)(idx % rows_max);
        buf[idx] = i < rows ? q[(size_t)c * NP + r0 + i] : 0.0;
    }
}
__global__ void k_fx_unpack(const double* __restrict__ buf, long long NP, int ncols, int world, int rows_max,
                            const int* __restrict__ r0s, double* __restrict__ q) {
    const long long tot = (long long)world * ncols * rows_max;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot; idx += (long long)gridDim.x * blockDim.x) {
        const int rk = (int)(idx / ((long long)ncols * rows_max));
        const long long rem = idx % ((long long)ncols * rows_max);
        const int c = (int)(rem / rows_max), i = (int)(rem % rows_max);
        const int r0 = r0s[rk], r1 = r0s[rk + 1];
        if (r0 + i < r1) q[(size_t)c * NP + r0 + i] = buf[idx];
    }
}
// no communicator (ranks emulated in one process): the rows this rank does not own are zero, so
// the ranks' outputs add up to the full product
__global__ void k_fx_zero_outside(long long NP, int ncols, int r0, int r1, double* __restrict__ q) {
    const long long tot = (long long)ncols * NP;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot; idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(idx % NP);
        if (i < r0 || i >= r1) q[idx] = 0.0;
    }
}
cudaError_t fx_pack(const double* q, long long NP, int ncols, int r0, int rows, int rows_max, double* buf,
                    cudaStream_t st) {
    k_fx_pack<<<592, 256, 0, st>>>(q, NP, ncols, r0, rows, rows_max, buf);
    return cudaGetLastError();
}
cudaError_t fx_unpack(const double* buf, long long NP, int ncols, int world, int rows_max, const int* r0s, double* q,
                      cudaStream_t st) {
    k_fx_unpack<<<592, 256, 0, st>>>(buf, NP, ncols, world, rows_max, r0s, q);
    return cudaGetLastError();
}
cudaError_t fx_zero_outside(long long NP, int ncols, int r0, int r1, double* q, cudaStream_t st) {
    k_fx_zero_outside<<<592, 256, 0, st>>>(NP, ncols, r0, r1, q);
    return cudaGetLastError();
}
int face_fx_tiles(long long NP, int ncols) { return dgemm_tiles<CfgFv>((int)NP, ncols); }

// F = B B^T scattered into the padded layout (B: n2 x n2 row-major, n2 = n^2, K padded to kp).
cudaError_t face_gram_scatter(const double* B, int n2, int kp, double* F, int n, int ldf, long long NP,
                              int num_sms, cudaStream_t st) {
    DgemmProblem g{n2, n2, kp, B, kp, B, kp};
    const int sk = dgemm_pick_splitk<CfgSlab>(n2, n2, kp, num_sms, 2);
    return dgemm_launch<CfgSlab>(g, sk, EpiFaceScatter{F, n, ldf, NP}, st);
}

// ------------------------------------------------------------------------------------ layouts
__global__ void k_face_copy_in(int n, int ldf, long long NP, int ncols, const double* __restrict__ src, int lds,
                               double* __restrict__ dst) {
    const long long n2 = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n2 * ncols;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long c = idx / n2, i = idx % n2;
        dst[c * NP + (i / n) * ldf + i % n] = src[c * lds + i];
    }
}
__global__ void k_face_copy_out(int n, int ldf, long long NP, int ncols, const double* __restrict__ src,
                                double* __restrict__ dst, int ldd) {
    const long long n2 = (long long)n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n2 * ncols;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long c = idx / n2, i = idx % n2;
        dst[c * ldd + i] = src[c * NP + (i / n) * ldf + i % n];
    }
}
cudaError_t face_copy_in(int n, int ldf, long long NP, int ncols, const double* src, int lds, double* dst,
                         cudaStream_t st) {
    k_face_copy_in<<<1184, 256, 0, st>>>(n, ldf, NP, ncols, src, lds, dst);
    return cudaGetLastError();
}
cudaError_t face_copy_out(int n, int ldf, long long NP, int ncols, const double* src, double* dst, int ldd,
                          cudaStream_t st) {
    k_face_copy_out<<<1184, 256, 0, st>>>(n, ldf, NP, ncols, src, dst, ldd);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------ stencils
// Face pair (SURVEY §8 "verified stencils", oracle pin test_face_pair_3d):
//   A_Γ = [4; -1 at (±1,0),(0,±1)],  M_Γ = (h^2/12)[6; 1 at (±1,0),(0,±1),(1,1),(-1,-1)].
__device__ __forceinline__ double face_at(const double* v, int j, int k, int n, int ldf) {
    return (j < 0 || k < 0 || j >= n || k >= n) ? 0.0 : v[j * ldf + k];
}
// y = a A v + b M v on one padded slab (0-based j, k)
__device__ __forceinline__ double face_op(const double* v, int j, int k, int n, int ldf, double a, double bm) {
    const double c = v[j * ldf + k];
    const double nb = face_at(v, j - 1, k, n, ldf) + face_at(v, j + 1, k, n, ldf) + face_at(v, j, k - 1, n, ldf) +
                      face_at(v, j, k + 1, n, ldf);
    const double dg = face_at(v, j + 1, k + 1, n, ldf) + face_at(v, j - 1, k - 1, n, ldf);
    return a * (4.0 * c - nb) + bm * (6.0 * c + nb + dg);
}

// out_c = s_c M_Γ v_c (+ add_c) on padded face vectors (s: per-column scale or null = 1; add or null)
__global__ void k_face_mass_axpy(int n, int ldf, long long NP, int ncols, double hh12, const double* __restrict__ v,
                                 const double* __restrict__ scale, const double* __restrict__ add, double* __restrict__ out) {
    const long long total = NP * ncols;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(idx / NP);
        const int r = (int)(idx % NP);
        const int j = r / ldf, k = r % ldf;
        double y = 0.0;
        if (j < n && k < n) {
            y = face_op(v + (size_t)c * NP, j, k, n, ldf, 0.0, hh12);
            if (scale) y *= scale[c];
            if (add) y += add[idx];
        }
        out[idx] = y;
    }
}
cudaError_t face_mass_axpy(int n, int ldf, long long NP, int ncols, double hh12, const double* v, const double* scale,
                           const double* add, double* out, cudaStream_t st) {
    long long blocks = (NP * ncols + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    k_face_mass_axpy<<<(int)blocks, 256, 0, st>>>(n, ldf, NP, ncols, hh12, v, scale, add, out);
    return cudaGetLastError();
}

// M applied to the columns of a dense column-major n2 x ncol matrix (setup: B = M V).
__global__ void k_face_mass_cols(int n, double hh12, const double* __restrict__ V, double* __restrict__ out, int n2,
                                 int ncol, int ldo) {
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n2 * ncol;
         idx += (long long)gridDim.x * blockDim.x) {
        const int col = (int)(idx / n2), i = (int)(idx % n2);
        const int j = i / n, k = i % n;
        const double* v = V + (size_t)col * n2;
        out[(size_t)col * ldo + i] = face_op(v, j, k, n, n, 0.0, hh12);
    }
}
// dense assembly of the face pair (setup only, for the generalised eigensolver)
__global__ void k_face_dense(int n, double hh12, double* __restrict__ A, double* __restrict__ M) {
    const int n2 = n * n;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n2;
         idx += (long long)gridDim.x * blockDim.x) {
        const int i = (int)idx, j = i / n, k = i % n;
        auto setp = [&](int jj, int kk, double av, double mv) {
            if (jj < 0 || kk < 0 || jj >= n || kk >= n) return;
            const size_t col = (size_t)jj * n + kk;
            A[col * n2 + i] = av;   // column-major (symmetric anyway)
            M[col * n2 + i] = mv;
        };
        setp(j, k, 4.0, 6.0 * hh12);
        setp(j - 1, k, -1.0, hh12); setp(j + 1, k, -1.0, hh12);
        setp(j, k - 1, -1.0, hh12); setp(j, k + 1, -1.0, hh12);
        setp(j + 1, k + 1, 0.0, hh12); setp(j - 1, k - 1, 0.0, hh12);
    }
}
// scale columns and transpose: Out (row-major n2 x kp) = (V diag(w))^T^T ... Out[i][j] = V[i + j n2] w[j]
__global__ void k_scale_transpose(const double* __restrict__ V, const double* __restrict__ w, int n2, double* __restrict__ out,
                                  int kp) {
    __shared__ double tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int j = by + r, i = bx + threadIdx.x;   // read V[i + j n2] (coalesced in i)
        tile[r][threadIdx.x] = (i < n2 && j < n2) ? V[(size_t)j * n2 + i] * w[j] : 0.0;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int i = bx + r, j = by + threadIdx.x;   // write out[i][j] (coalesced in j)
        if (i < n2 && j < kp) out[(size_t)i * kp + j] = (j < n2) ? tile[threadIdx.x][r] : 0.0;
    }
}

__global__ void k_face_identity_cols(int n, int ldf, long long NP, int j0, int nb, double* __restrict__ X) {
    const long long tot = (long long)nb * NP;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(e / NP);
        const long long i = e - (long long)c * NP;
        const int j = j0 + c;
        const long long jp = (long long)(j / n) * ldf + j % n;
        X[e] = i == jp ? 1.0 : 0.0;
    }
}
__global__ void k_face_fold_rows(double* __restrict__ F, long long NP, int n, int ldf, int j0, int nb, double gamma,
                                 const double* __restrict__ Y) {
    const long long tot = (long long)nb * NP;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(e / NP);
        const long long i = e - (long long)c * NP;
        const int j = j0 + c;
        const long long jp = (long long)(j / n) * ldf + j % n;
        double* row = F + jp * NP;
        row[i] = fma(gamma, row[i], Y[e]);
    }
}
cudaError_t face_identity_cols(int n, int ldf, long long NP, int j0, int nb, double* X, cudaStream_t st) {
    k_face_identity_cols<<<1184, 256, 0, st>>>(n, ldf, NP, j0, nb, X);
    return cudaGetLastError();
}
cudaError_t face_fold_rows(double* F, long long NP, int n, int ldf, int j0, int nb, double gamma, const double* Y,
                           cudaStream_t st) {
    k_face_fold_rows<<<1184, 256, 0, st>>>(F, NP, n, ldf, j0, nb, gamma, Y);
    return cudaGetLastError();
}
__global__ void k_face_gather_cols(const double* __restrict__ B, int rows, int ldb, int j0, int nb, int n, int ldf,
                                   long long NP, double* __restrict__ X) {
    const long long tot = (long long)rows * nb;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e / nb), cc = (int)(e % nb);              // consecutive threads: consecutive columns
        X[(size_t)cc * NP + (size_t)(i / n) * ldf + i % n] = B[(size_t)i * ldb + j0 + cc];
    }
}
__global__ void k_face_scatter_cols(const double* __restrict__ X, int rows, int ldb, int j0, int nb, int n, int ldf,
                                    long long NP, double* __restrict__ B) {
    const long long tot = (long long)rows * nb;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(e / nb), cc = (int)(e % nb);
        B[(size_t)i * ldb + j0 + cc] = X[(size_t)cc * NP + (size_t)(i / n) * ldf + i % n];
    }
}
__global__ void k_face_hat_diag(double* __restrict__ F, long long NP, double gamma, double K, const double* __restrict__ w) {
    const long long tot = NP * NP;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
        const long long i = e / NP, j = e - i * NP;
        const double v = gamma * F[e];
        F[e] = i == j ? fma(K, w[i], v) : v;
    }
}
cudaError_t face_gather_cols(const double* B, int rows, int ldb, int j0, int nb, int n, int ldf, long long NP, double* X,
                             cudaStream_t st) {
    k_face_gather_cols<<<1184, 256, 0, st>>>(B, rows, ldb, j0, nb, n, ldf, NP, X);
    return cudaGetLastError();
}
cudaError_t face_scatter_cols(const double* X, int rows, int ldb, int j0, int nb, int n, int ldf, long long NP, double* B,
                              cudaStream_t st) {
    k_face_scatter_cols<<<1184, 256, 0, st>>>(X, rows, ldb, j0, nb, n, ldf, NP, B);
    return cudaGetLastError();
}
cudaError_t face_hat_diag(double* F, long long NP, int n, int ldf, double gamma, double K, const double* w,
                          cudaStream_t st) {
    (void)n; (void)ldf;
    k_face_hat_diag<<<1184 * 4, 256, 0, st>>>(F, NP, gamma, K, w);
    return cudaGetLastError();
}
cudaError_t face_dense_pair(int n, double hh12, double* A, double* M, cudaStream_t st) {
    k_face_dense<<<1184, 256, 0, st>>>(n, hh12, A, M);
    return cudaGetLastError();
}
cudaError_t face_mass_cols(int n, double hh12, const double* V, double* out, int ncol, int ldo, cudaStream_t st) {
    k_face_mass_cols<<<1184, 256, 0, st>>>(n, hh12, V, out, n * n, ncol, ldo);
    return cudaGetLastError();
}
cudaError_t scale_transpose(const double* V, const double* w, int n2, double* out, int kp, cudaStream_t st) {
    dim3 grid((n2 + 31) / 32, (kp + 31) / 32);
    k_scale_transpose<<<grid, dim3(32, 8), 0, st>>>(V, w, n2, out, kp);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------ inner PCG
// Pair layout: pair q = s * C + c (system s of this rank, column c); vectors NP each.

// deterministic block reduction
__device__ __forceinline__ double block_sum(double a, double* red) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    __syncthreads();
    if (lane == 0) red[warp] = a;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < W; w++) s += red[w];
    __syncthreads();
    return s;
}

// ---- sine-domain inner CG: the operator of system s is  dg_s ∘ v + cs_s D̂ v D̂^T  and the
// preconditioner is 1/dg_s (the sine-diagonal part), both exact algebra of the face pair
// (M = M̃ + (h^2/24) D⊗D, D = central difference).
// init: r̂ = b̂_c, x̂ = 0, ẑ = r̂ / dg, ρ = ρ0 = r̂·ẑ, p̂ = ẑ
__global__ void k_inner_init_hat(InnerArgs a, const double* __restrict__ bh) {
    __shared__ double red[32];
    const int pq = blockIdx.x;
    const int c = pq % a.C, s = pq / a.C;
    const size_t off = (size_t)pq * a.NP;
    const double* idg = a.idg + (size_t)s * a.NP;
    double rho = 0.0;
    for (long long i = threadIdx.x; i < a.NP; i += blockDim.x) {
        const double r = bh[(size_t)c * a.NP + i];
        const double z = r * idg[i];
        a.r[off + i] = r;
        a.x[off + i] = 0.0;
        a.p[off + i] = z;
        rho = fma(r, z, rho);
    }
    rho = block_sum(rho, red);
    if (threadIdx.x == 0) {
        a.rho[pq] = rho;
        a.rho0[pq] = rho;
        a.active[pq] = rho > 0.0 ? 1 : 0;
    }
}
// given q̂ = Â p̂: α = ρ/(p̂·q̂); x̂ += αp̂; r̂ -= αq̂; ẑ = r̂/dg; ρ' = r̂·ẑ; stop if ρ' <= rtol^2 ρ0;
// else p̂ = ẑ + (ρ'/ρ) p̂   (one CTA per pair; fixed-order reductions)
// CG update of one (system, column) pair by a cluster of ICL CTAs, each owning NP/ICL of the
// pair's entries; the two dot products are reduced over DSMEM in fixed rank order (deterministic):
//   q̂ = dg ∘ p̂ + q̂_part;  α = ρ/p̂·q̂;  x̂ += α p̂;  r̂ -= α q̂;  ρ' = r̂·(idg ∘ r̂);  p̂ = idg ∘ r̂ + β p̂
constexpr int ICL = 4;
template <int NCL>
__device__ __forceinline__ double cluster_allsum(double v, double* red, double* slot, bool trailing_sync = true) {
    // block sum -> this CTA's slot; cluster barrier; every CTA sums the ICL slots in rank order.
    // trailing_sync = false when the caller's next cluster barrier (or one before exiting) already
    // orders the slot reads before any overwrite or exit
    v = block_sum(v, red);
    cg::cluster_group cl = cg::this_cluster();
    if (threadIdx.x == 0) *slot = v;
    cl.sync();
    double s = 0.0;
    for (int q = 0; q < NCL; q++) s += *cl.map_shared_rank(slot, q);
    if (trailing_sync) cl.sync();                // nobody leaves / overwrites before all have read
    return s;
}
template <int NCL>
__global__ void __cluster_dims__(NCL, 1, 1) k_inner_update_cl(InnerArgs a, int* n_active) {
    __shared__ double red[32];
    __shared__ double slot[2];                   // one per reduction: the second needs no barrier before reuse
    const int pq = blockIdx.y;
    const int rank = blockIdx.x;                 // cluster rank (cluster spans blockIdx.x)
    if (!a.active[pq]) return;                   // uniform across the cluster
    const int s = pq / a.C;
    const long long chunk = (a.NP + NCL - 1) / NCL;
    const long long i0 = rank * chunk, i1 = min(a.NP, i0 + chunk);
    const size_t off = (size_t)pq * a.NP;
    const double* dg = a.dg + (size_t)s * a.NP;
    const double* idg = a.idg + (size_t)s * a.NP;
    // ρ read once, before the first cluster barrier: rank 0 overwrites it at the end, after the
    // other CTAs have passed both reductions (no read may follow that store)
    const double rho_old = a.rho[pq];
    double d = 0.0;
    for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const double pv = a.p[off + i];
        const double qv = fma(dg[i], pv, a.q[off + i]);
        a.q[off + i] = qv;
        d = fma(pv, qv, d);
    }
    d = cluster_allsum<NCL>(d, red, &slot[0], false);
    if (!(d > 0.0)) {
        cg::this_cluster().sync();               // slot[0] reads done before any CTA exits
        if (rank == 0 && threadIdx.x == 0) a.active[pq] = 0;
        return;
    }
    const double alpha = rho_old / d;
    double rho = 0.0;
    for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        a.x[off + i] = fma(alpha, a.p[off + i], a.x[off + i]);
        const double r = fma(-alpha, a.q[off + i], a.r[off + i]);
        a.r[off + i] = r;
        rho = fma(r, r * idg[i], rho);
    }
    rho = cluster_allsum<NCL>(rho, red, &slot[1]);
    if (!(rho > a.rtol * a.rtol * a.rho0[pq])) {
        if (rank == 0 && threadIdx.x == 0) a.active[pq] = 0;
        return;
    }
    const double beta = rho / rho_old;
    for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x)
        a.p[off + i] = fma(beta, a.p[off + i], a.r[off + i] * idg[i]);
    if (rank == 0 && threadIdx.x == 0) {
        a.rho[pq] = rho;
        atomicAdd(n_active, 1);
    }
}
// inner-loop WHILE-graph condition: one more iteration while any pair is active and it < maxit
// (handle 0: the host-driven loop, counter only)
__global__ void k_inner_cond(int* n_active, int* counter, int maxit, unsigned long long handle) {
    const int it = *counter + 1;
    *counter = it;
    counter[2] += 1;          // cumulative inner iterations (launch accounting; see dd_launch_count)
    const int na = *n_active;
    *n_active = 0;
    if (handle) cudaGraphSetConditional((cudaGraphConditionalHandle)handle, (na > 0 && it < maxit) ? 1u : 0u);
}

// ---- Chebyshev semi-iteration for the shifted face systems (reading A12'): with the rigorous
// spectral bounds 1 -/+ δ_s of the sine-diagonal preconditioned system (centre 1), x_0 = 0 and
// d_0 = P^-1 b, x_1 = d_0; step j = 0.. K_s-2 (face_inner_cheb_pass):
//   r = b - A x_{j+1},  d_{j+1} = c1[j] d_j + c2[j] P^-1 r,  x_{j+2} = x_{j+1} + d_{j+1}
// — the three-term recurrence written with the true residual, so the state is (x̂, d̂) only and
// K_s steps cost K_s - 1 operator applications.  No inner products: a pair stops after its
// a-priori step count K_s.
__global__ void k_inner_init_cheb(InnerArgs a, const double* __restrict__ bh) {
    const int pq = blockIdx.y;
    const int c = pq % a.C, s = pq / a.C;
    const size_t off = (size_t)pq * a.NP;
    const double* idg = a.idg + (size_t)s * a.NP;
    const bool live = a.kmax[s] > 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.NP; i += (long long)gridDim.x * blockDim.x) {
        a.x[off + i] = live ? bh[(size_t)c * a.NP + i] * idg[i] : 0.0;   // x̂_1 = d_0 (step 0 reads d from x̂)
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.active[pq] = a.kmax[s] > 1 ? 1 : 0;
}
// after step j = counter[0]: j + 1 steps done; pair q stays active while j + 3 <= K_s; the WHILE
// graph continues while any pair is active and j + 1 < maxit (handle 0: host-driven loop, which
// polls *n_active)
__global__ void k_inner_cond_cheb(InnerArgs a, int* n_active, int* counter, int maxit, unsigned long long handle) {
    const int j = counter[0] + 1;
    int na = 0;
    for (int pq = threadIdx.x; pq < a.npair; pq += blockDim.x) {
        const int on = j + 1 < a.kmax[pq / a.C] ? 1 : 0;
        a.active[pq] = on;
        na += on;
    }
    na = __syncthreads_count(na > 0);
    if (threadIdx.x == 0) {
        counter[0] = j;
        counter[2] += 1;       // cumulative steps (launch accounting; see dd_launch_count)
        *n_active = na;
        if (handle) cudaGraphSetConditional((cudaGraphConditionalHandle)handle, (na > 0 && j < maxit) ? 1u : 0u);
    }
}
// ---- fused Chebyshev step for n_e = 64 (N = 128: ldf = 128, two 64-wide parity blocks o, e).
// With D̂ = [[0, E], [-E^T, 0]] (antisymmetric, exact in the table) the operator's D̂ X̂ D̂^T splits
// into four independent 64x64 blocks, each from ONE block of X̂:
//   V_AB = L_A X̂_{Ā B̄} M_B^T,  L_o = M_o = E,  L_e = M_e = E^T,  sign -1 when A != B.
// Work item = (pair, output block AB), 4 per pair, strided over a persistent grid of one CTA per
// SM with warp-specialised roles (174 KB smem: E, X̂ block, Y, two V buffers):
//   8 MMA warps   X̂ block (cp.async, the next item's streams in during GEMM 2) -> Y = L X̂ (DMMA,
//                 K = 64) -> Y to smem -> V = Y M^T (DMMA) -> V to smem buffer t & 1;
//   8 epilogue    per V buffer: r = b̂ - dg∘x̂ - cs V, d = c1 d + c2 idg∘r, x̂' = x̂ + d over
//     warps       16-byte row pairs (coalesced, 4 independent loads batches per thread).
// FULL/EMPTY named barriers (bar.arrive / bar.sync) hand the V buffers over, so item t's
// epilogue (global-memory latency) overlaps item t+1's GEMMs (tensor pipe).  x̂ ping-pongs
// between a.x and a.x1 by step parity (the items of one pair read each other's blocks); d̂ is
// updated in place (read and written by its own item only).  The last CTA to finish advances
// the step counter, the active flags and the WHILE condition.  Same arithmetic as the two-pass
// form up to summation order.
constexpr int CF_LD = 68;                        // smem row stride: conflict-free fragment loads
constexpr int CF_MMA = 256, CF_EPI = 256, CF_T = CF_MMA + CF_EPI;
constexpr int CF_NI = 2;                         // MMA warp tile 32 x 16 (2 x 4 warps over the 64x64 block)
constexpr size_t CF_BLK = size_t(64) * CF_LD;    // doubles per 64x64 smem block
constexpr size_t CF_SMEM = 5 * CF_BLK * sizeof(double);
bool cheb_fused_ok(int n, int ldf) { return ldf == 128 && (n + 1) / 2 == 64; }

__device__ __forceinline__ void cf_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void cf_bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int NT>
__device__ __forceinline__ void cf_load_block(double* dst, const double* src, int ldf, int tid) {
#pragma unroll
    for (int j = 0; j < 64 * 32 / NT; j++) {
        const int c = tid + NT * j, row = c >> 5, ch = c & 31;
        dg_cp_async16(dst + row * CF_LD + 2 * ch, src + (size_t)row * ldf + 2 * ch);
    }
}
// C = L B over K = 64 for this warp's (16 MI) x (8 NI) sub-tile at (row0, col0): L[i][k] = Ls[i*l1 + k*l2],
// B[k][j] = Bs[k*b1 + j*b2]
template <int MI, int NI>
__device__ __forceinline__ void cf_gemm(double (&acc)[MI][NI][4], const double* Ls, int l1, int l2, const double* Bs,
                                        int b1, int b2, int row0, int col0, int gq, int tq) {
#pragma unroll
    for (int mi = 0; mi < MI; mi++)
#pragma unroll
        for (int ni = 0; ni < NI; ni++)
#pragma unroll
            for (int r = 0; r < 4; r++) acc[mi][ni][r] = 0.0;
    const double* la = Ls + (row0 + gq) * l1 + tq * l2;
    const double* bb = Bs + tq * b1 + (col0 + gq) * b2;
#pragma unroll 4
    for (int kk = 0; kk < 64; kk += 4) {
        double af[MI][2], bf[NI];
#pragma unroll
        for (int mi = 0; mi < MI; mi++) {
            af[mi][0] = la[(mi * 16) * l1 + kk * l2];
            af[mi][1] = la[(mi * 16 + 8) * l1 + kk * l2];
        }
#pragma unroll
        for (int ni = 0; ni < NI; ni++) bf[ni] = bb[kk * b1 + (ni * 8) * b2];
#pragma unroll
        for (int mi = 0; mi < MI; mi++)
#pragma unroll
            for (int ni = 0; ni < NI; ni++) dg_mma(acc[mi][ni], af[mi][0], af[mi][1], bf[ni]);
    }
}
template <int MI, int NI>
__device__ __forceinline__ void cf_store_acc(double* Ys, const double (&acc)[MI][NI][4], int row0, int col0, int gq,
                                             int tq) {
#pragma unroll
    for (int mi = 0; mi < MI; mi++)
#pragma unroll
        for (int ni = 0; ni < NI; ni++) {
            const int row = row0 + mi * 16 + gq, col = col0 + ni * 8 + 2 * tq;
            *reinterpret_cast<double2*>(&Ys[row * CF_LD + col]) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
            *reinterpret_cast<double2*>(&Ys[(row + 8) * CF_LD + col]) = make_double2(acc[mi][ni][2], acc[mi][ni][3]);
        }
}
// the 8 MMA warps' tiling of an item of HR output rows x 64 columns: WMW x (8 / WMW) warps of
// (16 MI) x (8 NI)
template <int HR> struct CfTile;
template <> struct CfTile<64> { static constexpr int MI = 2, NI = 2, WMW = 2; };
template <> struct CfTile<32> { static constexpr int MI = 1, NI = 2, WMW = 2; };
template <> struct CfTile<16> { static constexpr int MI = 1, NI = 1, WMW = 1; };

// MMA-warp part of one work item (rows h HR .. of output block AB): GEMM 1, the next unit's X̂ block
// prefetch (src_next, or none), Y to smem, GEMM 2, V to buffer t & 1
template <int HR>
__device__ __forceinline__ void cf_mma_item(int A, int B, int h, int t, const double* src_next, int ldf, double* Es,
                                            double* Xs, double* Ys, double* Vs, int tid) {
    using TL = CfTile<HR>;
    const int warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
    const int row0 = (warp % TL::WMW) * 16 * TL::MI, col0 = (warp / TL::WMW) * 8 * TL::NI;
    dg_cp_wait<0>();
    cf_bar_sync(1, CF_MMA);                           // X̂ block (and E) landed for every MMA warp
    double acc[TL::MI][TL::NI][4];
    // Y = L X̂ for the item's HR rows of L (= E, or E^T read transposed)
    cf_gemm<TL::MI, TL::NI>(acc, Es + (A ? h * HR : h * HR * CF_LD), A ? 1 : CF_LD, A ? CF_LD : 1, Xs, CF_LD, 1, row0,
                            col0, gq, tq);
    cf_bar_sync(1, CF_MMA);                           // X̂ consumed; previous GEMM 2 done with Ys
    if (src_next) cf_load_block<CF_MMA>(Xs, src_next, ldf, tid);
    dg_cp_commit();
    cf_store_acc<TL::MI, TL::NI>(Ys, acc, row0, col0, gq, tq);
    cf_bar_sync(1, CF_MMA);
    cf_gemm<TL::MI, TL::NI>(acc, Ys, CF_LD, 1, Es, B ? CF_LD : 1, B ? 1 : CF_LD, row0, col0, gq, tq);   // V = Y M^T
    const int b = t & 1;
    if (t >= 2) cf_bar_sync(4 + b, CF_T);             // EMPTY[b]: item t-2's epilogue is done with it
    cf_store_acc<TL::MI, TL::NI>(Vs + b * CF_BLK, acc, row0, col0, gq, tq);
    cf_bar_arrive(2 + b, CF_T);                       // FULL[b]
}

// epilogue-warp part of one work item:  r = b̂ - dg∘x̂ - cs V;  d = c1 d + c2 idg∘r;  x̂' = x̂ + d
template <int HR>
__device__ __forceinline__ void cf_epi_item(const InnerArgs& a, const double* __restrict__ bh, const double* xin,
                                            double* xout, int q, int A, int B, int h, int j, int t, bool release,
                                            const double* Vs, int et) {
    constexpr int PAIRS = HR * 32 / CF_EPI, U = PAIRS < 4 ? PAIRS : 4;      // row pairs per thread, per batch
    const int s = q / a.C, c = q - s * a.C, ldf = a.ldf;
    const int b = t & 1;
    const double sg = A == B ? 1.0 : -1.0;
    const double cs = sg * a.cs[s], c1 = a.cc1[(size_t)s * a.kstride + j], c2 = a.cc2[(size_t)s * a.kstride + j];
    const size_t e0 = (size_t)q * a.NP, t0 = (size_t)s * a.NP, b0 = (size_t)c * a.NP;
    const size_t base = (size_t)(A * 64 + h * HR) * ldf + B * 64;
    const double* V = Vs + b * CF_BLK;
    cf_bar_sync(2 + b, CF_T);                         // FULL[b]
#pragma unroll 1
    for (int bb = 0; bb < PAIRS; bb += U) {
        double2 xv[U], dv[U], bv[U], gv[U], iv[U];
        size_t idx[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int e = (bb + u) * CF_EPI + et, row = e >> 5, cp = e & 31;
            idx[u] = base + (size_t)row * ldf + 2 * cp;
            xv[u] = *reinterpret_cast<const double2*>(xin + e0 + idx[u]);
            dv[u] = j == 0 ? xv[u] : *reinterpret_cast<const double2*>(a.p + e0 + idx[u]);
            bv[u] = __ldg(reinterpret_cast<const double2*>(bh + b0 + idx[u]));
            gv[u] = __ldg(reinterpret_cast<const double2*>(a.dg + t0 + idx[u]));
            iv[u] = __ldg(reinterpret_cast<const double2*>(a.idg + t0 + idx[u]));
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int e = (bb + u) * CF_EPI + et, row = e >> 5, cp = e & 31;
            const double2 v = *reinterpret_cast<const double2*>(&V[row * CF_LD + 2 * cp]);
            const double r0 = bv[u].x - fma(gv[u].x, xv[u].x, cs * v.x);
            const double r1 = bv[u].y - fma(gv[u].y, xv[u].y, cs * v.y);
            const double d0 = fma(c1, dv[u].x, c2 * (iv[u].x * r0));
            const double d1 = fma(c1, dv[u].y, c2 * (iv[u].y * r1));
            *reinterpret_cast<double2*>(a.p + e0 + idx[u]) = make_double2(d0, d1);
            *reinterpret_cast<double2*>(xout + e0 + idx[u]) = make_double2(xv[u].x + d0, xv[u].y + d1);
        }
    }
    if (release) cf_bar_arrive(4 + b, CF_T);          // EMPTY[b] (only when the MMA warps will wait for it)
}

// HR: output rows per work item — 64 (a whole parity block) or 32 (half a block: twice the items,
// for batches whose pairs do not fill the SMs, e.g. the ranks of a pole split).  With HR = 64 the
// items left over after the whole rounds (nitem mod G) are cut into 16-row quarters spread over
// every CTA when that leaves at most two quarters per CTA (9 columns: 756 = 5 x 148 + 16 blocks ->
// one quarter each instead of a sixth round; 572 -> 508 us per apply).
// MULTI = false: one step (j = counter[0]) per launch, the last CTA advances the counter and sets the
// WHILE condition.  MULTI = true: all nsteps steps in one cooperative launch with a grid-wide
// barrier between steps — E stays in shared memory and the per-step launch / ramp / tail goes away.
// A block item is active at step j iff j + 1 < K_s of its system (the pair's a-priori step count).
// Work units of a step, strided over the CTAs: u < nmain  -> block item u (HR rows);
//                                    u >= nmain -> quarter (u - nmain) % 4 of block item nmain + (u - nmain) / 4
template <int HR, bool MULTI>
__global__ void __launch_bounds__(CF_T, 1) k_cheb_step(InnerArgs a, const double* __restrict__ bh,
                                                       const double* __restrict__ Dh, int* n_active, int* counter,
                                                       int* done, int maxit, unsigned long long handle, int nsteps) {
    constexpr int NH = 64 / HR, IPP = 4 * NH;         // items per block, per pair
    constexpr bool TAIL = HR == 64;                   // quarter the leftover items
    extern __shared__ __align__(16) double smem[];
    double* Es = smem;
    double* Xs = smem + CF_BLK;
    double* Ys = smem + 2 * CF_BLK;
    double* Vs = smem + 3 * CF_BLK;                   // two buffers
    __shared__ int last;
    const int tid = threadIdx.x;
    const int j0 = MULTI ? 0 : counter[0];
    const int J1 = MULTI ? nsteps : j0 + 1;
    const int nitem = a.npair * IPP;
    const int ldf = a.ldf;
    const int G = gridDim.x;
    // quarters only pay when they leave at most 2 per CTA: a quarter item runs at ~1/3 of a block
    // item's time (measured), so 3 quarters cost a whole round (config 4's 80 leftover blocks -> 320
    // quarters -> 3 per CTA: kept whole)
    const int rem = nitem % G;
    const bool split = TAIL && rem != 0 && (4 * rem + G - 1) / G <= 2;
    const int nmain = split ? nitem - rem : nitem;
    const int nunit = nmain + 4 * (nitem - nmain);
    // unit -> (block item, quarter or -1 for a whole item)
    auto item_of = [&](int u) { return u < nmain ? u : nmain + (u - nmain) / 4; };
    auto next = [&](int u, int j) {
        while (u < nunit && !(j + 1 < a.kmax[(item_of(u) / IPP) / a.C])) u += G;
        return u;
    };
    // this CTA's units over all its steps: the EMPTY hand-over looks two units ahead across steps
    int T_total = 0;
    for (int j = j0; j < J1; j++)
        for (int u = next(blockIdx.x, j); u < nunit; u = next(u + G, j)) T_total++;
    if (tid < CF_MMA) cf_load_block<CF_MMA>(Es, Dh + 64, ldf, tid);        // E = D̂[o rows][e cols], once
    int t = 0;
    for (int j = j0; j < J1; j++) {
        const double* xin = (j & 1) ? a.x1 : a.x;
        double* xout = (j & 1) ? a.x : a.x1;
        auto xblk = [&](int item) {
            const int q = item / IPP, blk = (item / NH) & 3, A = blk >> 1, B = blk & 1;
            return xin + (size_t)q * a.NP + (size_t)(1 - A) * 64 * ldf + (1 - B) * 64;
        };
        const int u0 = next(blockIdx.x, j);
        if (tid < CF_MMA) {
            // ------------------------------------------------ MMA warps
            if (u0 < nunit) cf_load_block<CF_MMA>(Xs, xblk(item_of(u0)), ldf, tid);
            dg_cp_commit();
            for (int u = u0; u < nunit; t++) {
                const int it = item_of(u), blk = (it / NH) & 3, A = blk >> 1, B = blk & 1;
                const int nu = next(u + G, j);                // within this step (the next step's X̂ is not final)
                const double* src = nu < nunit ? xblk(item_of(nu)) : nullptr;
                if (u < nmain) cf_mma_item<HR>(A, B, it % NH, t, src, ldf, Es, Xs, Ys, Vs, tid);
                else if constexpr (TAIL) cf_mma_item<16>(A, B, (u - nmain) % 4, t, src, ldf, Es, Xs, Ys, Vs, tid);
                u = nu;
            }
            dg_cp_wait<0>();
        } else {
            // ------------------------------------------------ epilogue warps
            const int et = tid - CF_MMA;
            for (int u = u0; u < nunit; t++) {
                const int it = item_of(u), q = it / IPP, blk = (it / NH) & 3, A = blk >> 1, B = blk & 1;
                const int nu = next(u + G, j);
                if (u < nmain) cf_epi_item<HR>(a, bh, xin, xout, q, A, B, it % NH, j, t, t + 2 < T_total, Vs, et);
                else if constexpr (TAIL)
                    cf_epi_item<16>(a, bh, xin, xout, q, A, B, (u - nmain) % 4, j, t, t + 2 < T_total, Vs, et);
                u = nu;
            }
        }
        if (MULTI && j + 1 < J1) {
            __syncthreads();
            cg::this_grid().sync();                           // step j's x̂, d̂ final everywhere
        }
    }
    if (MULTI) {
        if (blockIdx.x == 0 && tid == 0) {
            counter[0] = J1;
            counter[2] += J1 - j0;
            *n_active = 0;
        }
        return;
    }
    // the last CTA to finish: step counter, active flags, loop condition
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        last = atomicAdd(done, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    const int jn = j0 + 1;
    int na = 0;
    for (int pq = tid; pq < a.npair; pq += CF_T) {
        const int on = jn + 1 < a.kmax[pq / a.C] ? 1 : 0;
        a.active[pq] = on;
        na += on;
    }
    na = __syncthreads_count(na > 0);
    if (tid == 0) {
        *done = 0;
        counter[0] = jn;
        counter[2] += 1;
        *n_active = na;
        if (handle) cudaGraphSetConditional((cudaGraphConditionalHandle)handle, (na > 0 && jn < maxit) ? 1u : 0u);
    }
}
template <int HR, bool MULTI>
static cudaError_t cheb_launch(int G, const InnerArgs& a, const double* bh, const double* Dh, int* n_active,
                               int* counter, int* done, int maxit, unsigned long long handle, int nsteps,
                               cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_cheb_step<HR, MULTI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)CF_SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (!MULTI) {
        k_cheb_step<HR, false><<<G, CF_T, CF_SMEM, st>>>(a, bh, Dh, n_active, counter, done, maxit, handle, nsteps);
        return cudaGetLastError();
    }
    void* args[] = {(void*)&a, (void*)&bh, (void*)&Dh, (void*)&n_active, (void*)&counter, (void*)&done, (void*)&maxit,
                    (void*)&handle, (void*)&nsteps};
    return cudaLaunchCooperativeKernel((const void*)k_cheb_step<HR, true>, dim3(G), dim3(CF_T), args, CF_SMEM, st);
}
// nsteps > 0: all steps in one cooperative launch (MULTI); nsteps = 0: one step (the WHILE-loop form)
cudaError_t cheb_step_fused(const InnerArgs& a, const double* bh, const double* Dh, int* n_active, int* counter,
                            int* done, int maxit, unsigned long long handle, int num_sms, cudaStream_t st, int nsteps) {
    // whole parity blocks when they give every SM two or more items; half blocks otherwise
    if (a.npair * 4 >= 2 * num_sms) {
        const int G = num_sms;
        return nsteps > 0 ? cheb_launch<64, true>(G, a, bh, Dh, n_active, counter, done, maxit, handle, nsteps, st)
                          : cheb_launch<64, false>(G, a, bh, Dh, n_active, counter, done, maxit, handle, 0, st);
    }
    const int G = std::min(num_sms, std::max(1, a.npair * 8));
    return nsteps > 0 ? cheb_launch<32, true>(G, a, bh, Dh, n_active, counter, done, maxit, handle, nsteps, st)
                      : cheb_launch<32, false>(G, a, bh, Dh, n_active, counter, done, maxit, handle, 0, st);
}
cudaError_t inner_init_cheb(const InnerArgs& a, const double* bh, cudaStream_t st) {
    k_inner_init_cheb<<<dim3(8, a.npair), 256, 0, st>>>(a, bh);
    return cudaGetLastError();
}
cudaError_t inner_cond_cheb(const InnerArgs& a, int* n_active, int* counter, int maxit, unsigned long long handle,
                            cudaStream_t st) {
    k_inner_cond_cheb<<<1, 256, 0, st>>>(a, n_active, counter, maxit, handle);
    return cudaGetLastError();
}
cudaError_t inner_cond(int* n_active, int* counter, int maxit, unsigned long long handle, cudaStream_t st) {
    k_inner_cond<<<1, 1, 0, st>>>(n_active, counter, maxit, handle);
    return cudaGetLastError();
}

cudaError_t inner_init_hat(const InnerArgs& a, const double* bh, cudaStream_t st) {
    k_inner_init_hat<<<a.npair, 512, 0, st>>>(a, bh);
    return cudaGetLastError();
}
cudaError_t inner_update_hat(const InnerArgs& a, int* n_active, cudaStream_t st) {
    // 4-CTA clusters of 256 threads (cfg4: 203 solves/s vs 197 with 512 threads — one wave of
    // CTAs instead of 2.3; 2-CTA / 1-CTA clusters and 128 / 1024 threads measured slower)
    k_inner_update_cl<ICL><<<dim3(ICL, a.npair), 256, 0, st>>>(a, n_active);
    return cudaGetLastError();
}

// init: r = b_c, x = 0 (z, ρ set after the first preconditioner application)
__global__ void k_inner_init(InnerArgs a, const double* __restrict__ b) {
    const int pq = blockIdx.x;
    const int c = pq % a.C;
    const size_t off = (size_t)pq * a.NP;
    for (long long i = threadIdx.x; i < a.NP; i += blockDim.x) {
        a.r[off + i] = b[(size_t)c * a.NP + i];
        a.x[off + i] = 0.0;
    }
}
// after z = P0 r: ρ = r·z, ρ0 = ρ, p = z, active
__global__ void k_inner_start(InnerArgs a) {
    __shared__ double red[32];
    const int pq = blockIdx.x;
    const size_t off = (size_t)pq * a.NP;
    double s = 0.0;
    for (long long i = threadIdx.x; i < a.NP; i += blockDim.x) {
        s = fma(a.r[off + i], a.z[off + i], s);
        a.p[off + i] = a.z[off + i];
    }
    s = block_sum(s, red);
    if (threadIdx.x == 0) {
        a.rho[pq] = s;
        a.rho0[pq] = s;
        a.active[pq] = s > 0.0 ? 1 : 0;
    }
}
// q = (a A + b M) p, then α = ρ/(p·q), x += αp, r -= αq   (one CTA per pair)
__global__ void k_inner_step1(InnerArgs a) {
    __shared__ double red[32];
    const int pq = blockIdx.x;
    if (!a.active[pq]) return;
    const int s = pq / a.C;
    const double ca = a.sys_a[s], cb = a.sys_b[s] * a.hh12;
    const size_t off = (size_t)pq * a.NP;
    const double* pv = a.p + off;
    double d = 0.0;
    for (int i = threadIdx.x; i < a.n * a.ldf; i += blockDim.x) {
        const int j = i / a.ldf, k = i % a.ldf;
        if (k >= a.n) continue;
        const double qi = face_op(pv, j, k, a.n, a.ldf, ca, cb);
        a.q[off + i] = qi;
        d = fma(pv[i], qi, d);
    }
    d = block_sum(d, red);
    const double alpha = d > 0.0 ? a.rho[pq] / d : 0.0;
    for (int i = threadIdx.x; i < a.n * a.ldf; i += blockDim.x) {
        if (i % a.ldf >= a.n) continue;
        a.x[off + i] = fma(alpha, pv[i], a.x[off + i]);
        a.r[off + i] = fma(-alpha, a.q[off + i], a.r[off + i]);
    }
}
// after z = P0 r: ρ' = r·z; converged if sqrt(ρ'/ρ0) <= rtol; else p = z + (ρ'/ρ) p
__global__ void k_inner_step2(InnerArgs a, int* n_active) {
    __shared__ double red[32];
    const int pq = blockIdx.x;
    if (!a.active[pq]) return;
    const size_t off = (size_t)pq * a.NP;
    const double rho_old = a.rho[pq];            // before block_sum's barriers: thread 0 overwrites it below
    double s = 0.0;
    for (long long i = threadIdx.x; i < a.NP; i += blockDim.x) s = fma(a.r[off + i], a.z[off + i], s);
    s = block_sum(s, red);
    if (!(s > a.rtol * a.rtol * a.rho0[pq])) {
        if (threadIdx.x == 0) a.active[pq] = 0;
        return;
    }
    const double beta = s / rho_old;
    for (long long i = threadIdx.x; i < a.NP; i += blockDim.x) a.p[off + i] = fma(beta, a.p[off + i], a.z[off + i]);
    if (threadIdx.x == 0) {
        a.rho[pq] = s;
        atomicAdd(n_active, 1);
    }
}
// z_c = Σ_s w_s x_{s,c}  in fixed system order (rank-local partial sum)
__global__ void k_inner_combine(InnerArgs a, const double* __restrict__ w, int nsys, double* __restrict__ zout) {
    const long long tot = a.NP * a.C;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < tot;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long c = idx / a.NP, i = idx % a.NP;
        double acc = 0.0;
        for (int s = 0; s < nsys; s++) {
            // fused Chebyshev: x̂ of system s after its min(K_s - 1, J) loop steps is in x1 if that is odd
            const double* xs = a.x;
            if (a.x1 && (max(0, min(a.kmax[s] - 1, *a.kiter)) & 1)) xs = a.x1;
            acc = fma(w[s], xs[((size_t)s * a.C + c) * a.NP + i], acc);
        }
        zout[idx] = acc;
    }
}

cudaError_t inner_init(const InnerArgs& a, const double* b, cudaStream_t st) {
    k_inner_init<<<a.npair, 256, 0, st>>>(a, b);
    return cudaGetLastError();
}
cudaError_t inner_start(const InnerArgs& a, cudaStream_t st) {
    k_inner_start<<<a.npair, 256, 0, st>>>(a);
    return cudaGetLastError();
}
cudaError_t inner_step1(const InnerArgs& a, cudaStream_t st) {
    k_inner_step1<<<a.npair, 256, 0, st>>>(a);
    return cudaGetLastError();
}
cudaError_t inner_step2(const InnerArgs& a, int* n_active, cudaStream_t st) {
    k_inner_step2<<<a.npair, 256, 0, st>>>(a, n_active);
    return cudaGetLastError();
}
cudaError_t inner_combine(const InnerArgs& a, const double* w, int nsys, double* zout, cudaStream_t st) {
    k_inner_combine<<<1184, 256, 0, st>>>(a, w, nsys, zout);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------ outer PCG (3D)
__global__ void k_gather_param(int ncols, const int* col_param, int n_param, const double* src, double* dst) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncols; c += gridDim.x * blockDim.x) {
        int p = col_param[c];
        p = p < 0 ? 0 : (p >= n_param ? n_param - 1 : p);
        dst[c] = src[p];
    }
}
cudaError_t gather_param(int ncols, const int* col_param, int n_param, const double* src, double* dst, cudaStream_t st) {
    if (ncols <= 0) return cudaSuccess;
    k_gather_param<<<(ncols + 127) / 128, 128, 0, st>>>(ncols, col_param, n_param, src, dst);
    return cudaGetLastError();
}
// k = 0: r = b (already in r), z given: ρ = r·z, η0, p = z, x = 0
__global__ void k3_pcg_start(Pcg3 s) {
    __shared__ double red[32];
    const int c = blockIdx.x;
    const size_t off = (size_t)c * s.NP;
    double rz = 0.0, zz = 0.0;
    for (long long i = threadIdx.x; i < s.NP; i += blockDim.x) {
        const double zi = s.z[off + i];
        rz = fma(s.r[off + i], zi, rz);
        zz = fma(zi, zi, zz);
        s.p[off + i] = zi;
        s.x[off + i] = 0.0;
    }
    rz = block_sum(rz, red);
    zz = block_sum(zz, red);
    if (threadIdx.x == 0) {
        const double eta0 = s.norm_kind == 0 ? sqrt(fmax(rz, 0.0)) : sqrt(zz);
        s.rho[c] = rz; s.eta0[c] = eta0; s.iters[c] = 0; s.relres[c] = eta0 > 0.0 ? 1.0 : 0.0;
        s.active[c] = (eta0 > 0.0 && rz >= 0.0) ? 1 : 0;
        if (rz < 0.0) atomicExch(s.status, (int)DD_ENOTSPD);
        if (c == 0 && s.hist) s.hist[0] = eta0;
    }
}
// The per-iteration updates on a cluster of PCL CTAs per column (a column is NP = 16384 entries at
// config 4; one CTA per column left 8 CTAs streaming it): each CTA owns NP/PCL entries, the dots
// are reduced over DSMEM in fixed rank order (deterministic), rank 0 writes the scalars.
constexpr int PCL = 8;
__global__ void __cluster_dims__(PCL, 1, 1) k3_pcg_alpha_cl(Pcg3 s) {
    __shared__ double red[32];
    __shared__ double slot[1];
    const int c = blockIdx.y, rank = blockIdx.x;
    if (!s.active[c]) return;                    // uniform across the cluster
    const size_t off = (size_t)c * s.NP;
    const long long chunk = (s.NP + PCL - 1) / PCL;
    const long long i0 = rank * chunk, i1 = min(s.NP, i0 + chunk);
    double pq = 0.0;
    for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) pq = fma(s.p[off + i], s.q[off + i], pq);
    pq = cluster_allsum<PCL>(pq, red, &slot[0]);
    if (!(pq > 0.0)) {
        if (rank == 0 && threadIdx.x == 0) { atomicExch(s.status, (int)DD_ENOTSPD); s.active[c] = 0; }
        return;
    }
    const double alpha = s.rho[c] / pq;
    for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        s.x[off + i] = fma(alpha, s.p[off + i], s.x[off + i]);
        s.r[off + i] = fma(-alpha, s.q[off + i], s.r[off + i]);
    }
}
__global__ void __cluster_dims__(PCL, 1, 1) k3_pcg_beta_cl(Pcg3 s, int k, int maxit, int* n_active) {
    __shared__ double red[32];
    __shared__ double slot[2];
    const int c = blockIdx.y, rank = blockIdx.x;
    if (!s.active[c]) return;                    // uniform across the cluster
    const size_t off = (size_t)c * s.NP;
    const long long chunk = (s.NP + PCL - 1) / PCL;
    const long long i0 = rank * chunk, i1 = min(s.NP, i0 + chunk);
    // ρ read before the first cluster barrier: rank 0 overwrites it after the last one
    const double rho_old = s.rho[c];
    double rz = 0.0, zz = 0.0;
    for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
        const double zi = s.z[off + i];
        rz = fma(s.r[off + i], zi, rz);
        zz = fma(zi, zi, zz);
    }
    rz = cluster_allsum<PCL>(rz, red, &slot[0]);
    zz = cluster_allsum<PCL>(zz, red, &slot[1]);
    const double eta = s.norm_kind == 0 ? sqrt(fmax(rz, 0.0)) : sqrt(zz);
    const bool conv = eta <= s.rtol * s.eta0[c];
    if (rank == 0 && threadIdx.x == 0) {
        s.iters[c] = k;
        s.relres[c] = eta / s.eta0[c];
        if (c == 0 && s.hist) s.hist[k] = eta;
        if (rz < 0.0) atomicExch(s.status, (int)DD_ENOTSPD);
    }
    if (conv || rz < 0.0 || k >= maxit) {
        if (rank == 0 && threadIdx.x == 0) s.active[c] = 0;
        return;
    }
    const double beta = rz / rho_old;
    for (long long i = i0 + threadIdx.x; i < i1; i += blockDim.x) s.p[off + i] = fma(beta, s.p[off + i], s.z[off + i]);
    if (rank == 0 && threadIdx.x == 0) {
        s.rho[c] = rz;
        atomicAdd(n_active, 1);
    }
}
cudaError_t pcg3_start(const Pcg3& s, cudaStream_t st) {
    k3_pcg_start<<<s.ncols, 512, 0, st>>>(s);
    return cudaGetLastError();
}
cudaError_t pcg3_alpha(const Pcg3& s, cudaStream_t st) {
    if (s.ncols <= 0) return cudaSuccess;
    k3_pcg_alpha_cl<<<dim3(PCL, s.ncols), 256, 0, st>>>(s);
    return cudaGetLastError();
}
cudaError_t pcg3_beta(const Pcg3& s, int k, int maxit, int* n_active, cudaStream_t st) {
    if (s.ncols <= 0) return cudaSuccess;
    k3_pcg_beta_cl<<<dim3(PCL, s.ncols), 256, 0, st>>>(s, k, maxit, n_active);
    return cudaGetLastError();
}

}  // namespace dd
