// Pole sum of the RA preconditioner and the fused PCG vector updates (sm_100a).
//
// Preconditioner (Eq.(8)):
//     z = c0 M_Γ^-1 r + Σ_k c_k (A_Γ - p_k M_Γ)^-1 r
// 1D Γ: every system is symmetric Toeplitz tridiagonal (d, e) and SPD, strictly diagonally
// dominant for p < 0 (no pivoting).  One CTA owns one column; its W warps each solve one
// system per round with a chunked Thomas + warp-PCR scheme:
//   lane l owns rows [lL, lL+L): interior rows lL..lL+L-2 and separator row lL+L-1;
//   interiors: y = T^-1 r_int (Thomas, precomputed pivots), x_int = y - e g_{l-1} u - e g_l Ju;
//   separators: 32-row reduced tridiagonal system solved by PCR over __shfl (precomputed
//   multipliers, 5 steps).
// Rows >= n are padding with x = 0 (equivalent to the Dirichlet end of Γ).
// All per-column vectors live in shared memory in a transposed, padded layout
// [row-in-chunk][lane] (stride 33) so both the per-lane sweeps and the coalesced global
// loads are bank-conflict free.  Systems are summed in fixed order (round-major over warps)
// and every dot product is a fixed-order tree: results are bitwise reproducible.
//
// PCG: one fused kernel per iteration after the
// two GEMMs: α = ρ/(p·q); x += αp; r -= αq; z = P r; ρ' = r·z; η test; β = ρ'/ρ; p = z + βp.
#include "dd_internal.h"

namespace dd {

#define TI(i, l) ((i) * 33 + (l))

struct SysView {
    double w, d, e;
    const double *invb, *cpr, *ufull, *upart, *pa, *pb, *pinvb;
};

__device__ __forceinline__ SysView sys_view(const PoleTabs& t, int param, int k, int L) {
    SysView v;
    const size_t ps = (size_t)param * t.max_sys + k;
    v.w = t.w[ps]; v.d = t.d[ps]; v.e = t.e[ps];
    v.invb = t.invb + ps * L;
    v.cpr = t.cpr + ps * L;
    v.ufull = t.ufull + ps * L;
    v.upart = t.upart + ps * L;
    v.pa = t.pa + ps * 160;
    v.pb = t.pb + ps * 160;
    v.pinvb = t.pinvb + ps * 32;
    return v;
}

// One warp solves (tridiag(e, d, e)) x = r for the column held in R (transposed layout) into X.
__device__ void warp_tridiag_solve(const SysView& S, const PoleGeom& g, const double* __restrict__ R,
                                   double* __restrict__ X, int lane) {
    const int L = g.L;
    const int Lr = lane < g.part_lane ? L - 1 : (lane == g.part_lane ? g.Lr_part : 0);
    const bool sep_real = lane < g.part_lane;
    const double* u = lane < g.part_lane ? S.ufull : S.upart;
    const double e = S.e;

    // forward elimination  ỹ_i = (r_i - e ỹ_{i-1}) / b'_i
    double prev = 0.0;
    for (int i = 0; i < Lr; i++) {
        const double ib = __ldg(&S.invb[i]);
        const double yt = R[TI(i, lane)] * ib - (e * ib) * prev;
        X[TI(i, lane)] = yt;
        prev = yt;
    }
    // back substitution  y_i = ỹ_i - (e / b'_i) y_{i+1}
    double next = 0.0;
    for (int i = Lr - 1; i >= 0; i--) {
        const double y = X[TI(i, lane)] - __ldg(&S.cpr[i]) * next;
        X[TI(i, lane)] = y;
        next = y;
    }
    const double y_first = Lr > 0 ? X[TI(0, lane)] : 0.0;
    const double y_last = Lr > 0 ? X[TI(Lr - 1, lane)] : 0.0;
    const double y_first_next = __shfl_down_sync(0xffffffffu, y_first, 1);
    const int Lr_next = (lane + 1) < g.part_lane ? L - 1 : ((lane + 1) == g.part_lane ? g.Lr_part : 0);

    // reduced right-hand side at this lane's separator
    double rs = 0.0;
    if (sep_real) {
        rs = R[TI(L - 1, lane)];
        if (Lr > 0) rs -= e * y_last;
        if (lane < 31 && Lr_next > 0) rs -= e * y_first_next;
    }
    // PCR over the 32 separators (precomputed multipliers)
#pragma unroll
    for (int j = 0; j < 5; j++) {
        const int s = 1 << j;
        double rm = __shfl_up_sync(0xffffffffu, rs, s);
        double rp = __shfl_down_sync(0xffffffffu, rs, s);
        if (lane < s) rm = 0.0;
        if (lane + s > 31) rp = 0.0;
        rs = rs - __ldg(&S.pa[j * 32 + lane]) * rm - __ldg(&S.pb[j * 32 + lane]) * rp;
    }
    const double gsep = sep_real ? rs * __ldg(&S.pinvb[lane]) : 0.0;
    double gleft = __shfl_up_sync(0xffffffffu, gsep, 1);
    if (lane == 0) gleft = 0.0;

    // interior reconstruction
    const double eg0 = e * gleft, eg1 = e * gsep;
    for (int i = 0; i < Lr; i++) {
        X[TI(i, lane)] = X[TI(i, lane)] - eg0 * __ldg(&u[i]) - eg1 * __ldg(&u[Lr - 1 - i]);
    }
    for (int i = Lr; i < L - 1; i++) X[TI(i, lane)] = 0.0;
    X[TI(L - 1, lane)] = gsep;
}

// z = P r for the CTA's column: R (input, transposed) -> Z (output, transposed).  Xb: W buffers.
__device__ void block_polesum(const PoleTabs& t, const PoleGeom& g, int param, const double* R, double* Z,
                              double* Xb) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = blockDim.x >> 5;
    const int L = g.L;
    const int tot = L * 33;
    const int nsys = t.nsys[param];
    for (int i = threadIdx.x; i < tot; i += blockDim.x) Z[i] = 0.0;
    for (int r0 = 0; r0 < nsys; r0 += W) {
        const int k = r0 + warp;
        if (k < nsys) {
            SysView S = sys_view(t, param, k, L);
            warp_tridiag_solve(S, g, R, Xb + (size_t)warp * tot, lane);
        }
        __syncthreads();
        const int nw = min(W, nsys - r0);
        for (int i = threadIdx.x; i < tot; i += blockDim.x) {
            if ((i % 33) == 32) continue;
            double acc = Z[i];
            for (int w = 0; w < nw; w++) acc += t.w[(size_t)param * t.max_sys + r0 + w] * Xb[(size_t)w * tot + i];
            Z[i] = acc;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------------
// Register-resident fast path for chunk length L <= LMAX <= 32 (n_Γ <= 1023).
// Every lane keeps its chunk (y) and its share of the pole sum (z) in registers; sweeps are fully
// unrolled so the table loads (shared memory, broadcast) are hoisted off the FMA chain.  Warp w
// accumulates systems k = w, w+W, ... in registers; the W partial sums are combined in fixed
// warp order at the end (deterministic).  Tables of all systems are staged in shared memory
// once per CTA: [k][invb | cpr | ufull | upart] x L.
template <int LMAX>
__device__ void block_polesum_reg(const PoleTabs& t, const PoleGeom& g, int param, const double* R, double* Z,
                                  double* scratch) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = blockDim.x >> 5;
    const int L = g.L;
    const int tot = L * 33;
    const int nsys = t.nsys[param];
    double* Zw = scratch;                          // [W][tot]
    double* tab = scratch + (size_t)W * tot;       // [nsys][4][L]
    const size_t pbase = (size_t)param * t.max_sys;
    for (int idx = threadIdx.x; idx < nsys * 4 * L; idx += blockDim.x) {
        const int k = idx / (4 * L), rem = idx - k * 4 * L, which = rem / L, i = rem - which * L;
        const double* src = which == 0 ? t.invb : (which == 1 ? t.cpr : (which == 2 ? t.ufull : t.upart));
        tab[idx] = src[(pbase + k) * L + i];
    }
    __syncthreads();

    const int Lr = lane < g.part_lane ? L - 1 : (lane == g.part_lane ? g.Lr_part : 0);
    const int Lr_next = (lane + 1) < g.part_lane ? L - 1 : ((lane + 1) == g.part_lane ? g.Lr_part : 0);
    const bool sep_real = lane < g.part_lane;
    double z[LMAX];
#pragma unroll
    for (int i = 0; i < LMAX; i++) z[i] = 0.0;

    for (int k = warp; k < nsys; k += W) {
        const double* ib = tab + (size_t)k * 4 * L;
        const double* cp = ib + L;
        const double* u = lane < g.part_lane ? ib + 2 * L : ib + 3 * L;
        const double e = t.e[pbase + k], wk = t.w[pbase + k];
        const double* pa = t.pa + (pbase + k) * 160;
        const double* pb = t.pb + (pbase + k) * 160;
        double pav[5], pbv[5];
#pragma unroll
        for (int j = 0; j < 5; j++) { pav[j] = __ldg(&pa[j * 32 + lane]); pbv[j] = __ldg(&pb[j * 32 + lane]); }
        const double pinv = __ldg(&t.pinvb[(pbase + k) * 32 + lane]);
        double y[LMAX];
        // forward:  ỹ_i = r_i/b'_i - (e/b'_i) ỹ_{i-1}
        double prev = 0.0, y_last = 0.0;   // y_last = ỹ_{Lr-1} = y_{Lr-1} (untouched by the back sweep)
#pragma unroll
        for (int i = 0; i < LMAX; i++) {
            if (i < L - 1) {
                const double v = fma(-cp[i], prev, R[TI(i, lane)] * ib[i]);
                y[i] = i < Lr ? v : 0.0;
                if (i < Lr) y_last = v;
                prev = y[i];
            } else {
                y[i] = 0.0;
            }
        }
        // backward:  y_i = ỹ_i - (e/b'_i) y_{i+1}
        double next = 0.0;
#pragma unroll
        for (int i = LMAX - 1; i >= 0; i--) {
            if (i < L - 1) {
                y[i] = fma(-cp[i], next, y[i]);
                next = y[i];
            }
        }
        double y_first = y[0];
        if (Lr == 0) y_first = 0.0;
        const double y_first_next = __shfl_down_sync(0xffffffffu, y_first, 1);
        double rs = 0.0;
        if (sep_real) {
            rs = R[TI(L - 1, lane)];
            if (Lr > 0) rs -= e * y_last;
            if (lane < 31 && Lr_next > 0) rs -= e * y_first_next;
        }
#pragma unroll
        for (int j = 0; j < 5; j++) {
            const int s = 1 << j;
            double rm = __shfl_up_sync(0xffffffffu, rs, s);
            double rp = __shfl_down_sync(0xffffffffu, rs, s);
            if (lane < s) rm = 0.0;
            if (lane + s > 31) rp = 0.0;
            rs = rs - pav[j] * rm - pbv[j] * rp;
        }
        const double gsep = sep_real ? rs * pinv : 0.0;
        double gleft = __shfl_up_sync(0xffffffffu, gsep, 1);
        if (lane == 0) gleft = 0.0;
        const double eg0 = e * gleft, eg1 = e * gsep;
#pragma unroll
        for (int i = 0; i < LMAX; i++) {
            if (i < L - 1 && i < Lr) {
                const double x = y[i] - eg0 * u[i] - eg1 * u[Lr - 1 - i];
                z[i] = fma(wk, x, z[i]);
            }
        }
        // separator row (in-chunk index L-1)
#pragma unroll
        for (int i = 0; i < LMAX; i++)
            if (i == L - 1) z[i] = fma(wk, gsep, z[i]);
    }
    // fixed-order combine of the W warp partials
#pragma unroll
    for (int i = 0; i < LMAX; i++)
        if (i < L) Zw[(size_t)warp * tot + TI(i, lane)] = z[i];
    __syncthreads();
    for (int idx = threadIdx.x; idx < tot; idx += blockDim.x) {
        if ((idx % 33) == 32) continue;
        double acc = 0.0;
        for (int w = 0; w < W; w++) acc += Zw[(size_t)w * tot + idx];
        Z[idx] = acc;
    }
    __syncthreads();
}

// Deterministic block reduction of two values (fixed tree).
__device__ __forceinline__ void block_sum2(double& a, double& b, double* red) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int W = blockDim.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    __syncthreads();
    if (lane == 0) { red[warp] = a; red[32 + warp] = b; }
    __syncthreads();
    double sa = 0.0, sb = 0.0;
    for (int w = 0; w < W; w++) { sa += red[w]; sb += red[32 + w]; }
    a = sa; b = sb;
    __syncthreads();
}

__device__ __forceinline__ int clamp_param(int p, int n_param) { return p < 0 ? 0 : (p >= n_param ? n_param - 1 : p); }

// rows of the column in natural order <-> transposed smem index
__device__ __forceinline__ int tpos(int row, int L) { return TI(row % L, row / L); }

template <int LMAX>
__device__ __forceinline__ void polesum_dispatch(const PoleTabs& t, const PoleGeom& g, int param, const double* R,
                                                 double* Z, double* Xb) {
    if constexpr (LMAX > 0) block_polesum_reg<LMAX>(t, g, param, R, Z, Xb);
    else block_polesum(t, g, param, R, Z, Xb);
}

// ---------------------------------------------------------------------------- kernels
template <int LMAX>
__global__ void k_precond(int ncols, const int* __restrict__ col_param, PoleGeom g, PoleTabs t,
                          const double* __restrict__ r, int ldr, double* __restrict__ z, int ldz) {
    extern __shared__ __align__(16) double sm[];
    const int c = blockIdx.x;
    if (c >= ncols) return;
    const int L = g.L, tot = L * 33;
    double* R = sm; double* Z = sm + tot; double* Xb = sm + 2 * tot;
    for (int i = threadIdx.x; i < 32 * L; i += blockDim.x)
        R[tpos(i, L)] = i < g.n ? r[(size_t)c * ldr + i] : 0.0;
    __syncthreads();
    polesum_dispatch<LMAX>(t, g, clamp_param(col_param[c], t.n_param), R, Z, Xb);
    for (int i = threadIdx.x; i < g.n; i += blockDim.x) z[(size_t)c * ldz + i] = Z[tpos(i, L)];
}

__device__ __forceinline__ void finish_iteration(const PcgState& s, bool still_active) {
    // grid-wide bookkeeping: count active columns; last CTA publishes and sets the graph condition
    __shared__ int s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        if (still_active) atomicAdd(s.n_active_next, 1);
        __threadfence();
        const int prev = atomicAdd(s.done_ctas, 1);
        s_last = (prev == (int)gridDim.x - 1);
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        __threadfence();
        const int na = atomicAdd(s.n_active_next, 0);
        const int k = *s.kiter + 1;
        *s.kiter = k;
        *s.n_active = na;
        *s.n_active_next = 0;
        *s.done_ctas = 0;
        if (s.cond_handle) {
            cudaGraphSetConditional((cudaGraphConditionalHandle)s.cond_handle,
                                    (na > 0 && k < s.maxit && *s.status == 0) ? 1u : 0u);
        }
    }
}

template <int LMAX>
__global__ void k_pcg_init(PcgState s, PoleGeom g, PoleTabs t, const double* __restrict__ b, int ldb) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[64];
    const int c = blockIdx.x;
    const int L = g.L, tot = L * 33, n = g.n;
    double* R = sm; double* Z = sm + tot; double* Xb = sm + 2 * tot;
    const size_t off = (size_t)c * s.ldv;
    for (int i = threadIdx.x; i < 32 * L; i += blockDim.x) {
        const double v = i < n ? b[(size_t)c * ldb + i] : 0.0;
        R[tpos(i, L)] = v;
        if (i < n) { s.r[off + i] = v; s.x[(size_t)c * s.ldx + i] = 0.0; }
    }
    __syncthreads();
    const int param = clamp_param(s.col_param[c], t.n_param);
    polesum_dispatch<LMAX>(t, g, param, R, Z, Xb);
    double rz = 0.0, zz = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double zi = Z[tpos(i, L)];
        rz += R[tpos(i, L)] * zi;
        zz += zi * zi;
        s.p[off + i] = zi;
    }
    block_sum2(rz, zz, red);
    if (threadIdx.x == 0) {
        const double eta0 = s.norm_kind == 0 ? sqrt(fmax(rz, 0.0)) : sqrt(zz);
        s.rho[c] = rz;
        s.eta0[c] = eta0;
        s.iters[c] = 0;
        s.relres[c] = eta0 > 0.0 ? 1.0 : 0.0;
        const bool act = eta0 > 0.0 && rz >= 0.0;
        if (rz < 0.0) atomicExch(s.status, (int)DD_ENOTSPD);
        s.active[c] = act ? 1 : 0;
        if (c == 0 && s.hist) s.hist[0] = eta0;
        if (act) atomicAdd(s.n_active_next, 1);
        __threadfence();
        const int prev = atomicAdd(s.done_ctas, 1);
        if (prev == (int)gridDim.x - 1) {
            __threadfence();
            *s.n_active = atomicAdd(s.n_active_next, 0);
            *s.n_active_next = 0;
            *s.done_ctas = 0;
            *s.kiter = 0;
        }
    }
}

template <int LMAX>
__global__ void k_pcg_iter(PcgState s, PoleGeom g, PoleTabs t) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[64];
    __shared__ double s_alpha;
    __shared__ int s_work;
    const int c = blockIdx.x;
    const int L = g.L, tot = L * 33, n = g.n;
    double* R = sm; double* Z = sm + tot; double* Xb = sm + 2 * tot;
    const size_t off = (size_t)c * s.ldv;
    if (threadIdx.x == 0) s_work = s.active[c];
    __syncthreads();
    bool still = false;
    if (s_work) {
        const int k = *s.kiter + 1;
        // π = p·q
        double pq = 0.0, dummy = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) pq += s.p[off + i] * s.q[off + i];
        block_sum2(pq, dummy, red);
        if (threadIdx.x == 0) s_alpha = pq > 0.0 ? s.rho[c] / pq : 0.0;
        __syncthreads();
        const double alpha = s_alpha;
        if (!(pq > 0.0)) {
            if (threadIdx.x == 0) {
                atomicExch(s.status, (int)DD_ENOTSPD);
                s.active[c] = 0;
                s.iters[c] = k;
            }
        } else {
            // x += α p ; r -= α q
            for (int i = threadIdx.x; i < 32 * L; i += blockDim.x) {
                double ri = 0.0;
                if (i < n) {
                    const double pi = s.p[off + i];
                    s.x[(size_t)c * s.ldx + i] += alpha * pi;
                    ri = s.r[off + i] - alpha * s.q[off + i];
                    s.r[off + i] = ri;
                }
                R[tpos(i, L)] = ri;
            }
            __syncthreads();
            const int param = clamp_param(s.col_param[c], t.n_param);
            polesum_dispatch<LMAX>(t, g, param, R, Z, Xb);
            double rz = 0.0, zz = 0.0;
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                const double zi = Z[tpos(i, L)];
                rz += R[tpos(i, L)] * zi;
                zz += zi * zi;
            }
            block_sum2(rz, zz, red);
            const double eta = s.norm_kind == 0 ? sqrt(fmax(rz, 0.0)) : sqrt(zz);
            const bool notspd = rz < 0.0;
            const bool conv = eta <= s.rtol * s.eta0[c];
            if (threadIdx.x == 0) {
                s.iters[c] = k;
                s.relres[c] = eta / s.eta0[c];
                if (c == 0 && s.hist) s.hist[k] = eta;
                if (notspd) atomicExch(s.status, (int)DD_ENOTSPD);
            }
            if (conv || notspd || k >= s.maxit) {
                if (threadIdx.x == 0) s.active[c] = 0;
            } else {
                const double beta = rz / s.rho[c];
                for (int i = threadIdx.x; i < n; i += blockDim.x)
                    s.p[off + i] = Z[tpos(i, L)] + beta * s.p[off + i];
                __syncthreads();
                if (threadIdx.x == 0) s.rho[c] = rz;
                still = true;
            }
        }
    }
    finish_iteration(s, still);
}

__global__ void k_copy_cols(int n, int ncols, const double* __restrict__ src, int lds, double* __restrict__ dst,
                            int ldd) {
    const size_t total = (size_t)n * ncols;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const size_t c = idx / n, i = idx % n;
        dst[c * ldd + i] = src[c * lds + i];
    }
}

__global__ void k_check_params(int ncols, const int* col_param, int n_param, int* flag) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncols; c += gridDim.x * blockDim.x) {
        const int p = col_param[c];
        if (p < 0 || p >= n_param) atomicExch(flag, 1);
    }
}

// ---------------------------------------------------------------------------- host side
// Launch shape of the pole-sum kernels: register fast path (LMAX = L rounded up to a power of
// two, L <= 32) with 4-8 warps, or the shared-memory path for longer chunks.
static int lmax_of(int L) {
    if (L <= 1) return 1;
    if (L <= 2) return 2;
    if (L <= 4) return 4;
    if (L <= 8) return 8;
    if (L <= 16) return 16;
    if (L <= 32) return 32;
    return 0;
}

int polesum_warps(int L) {
    if (lmax_of(L) > 0) return L >= 32 ? 4 : 8;
    const size_t buf = (size_t)L * 33 * sizeof(double);
    const size_t budget = 200 * 1024;
    int w = (int)(budget / buf) - 2;
    return w < 1 ? 1 : (w > 8 ? 8 : w);
}

size_t polesum_smem(int L, int warps, int max_sys) {
    size_t d = (size_t)(2 + warps) * L * 33;
    if (lmax_of(L) > 0) d += (size_t)max_sys * 4 * L;
    return d * sizeof(double);
}

template <typename K>
static cudaError_t set_smem(K kern, size_t bytes) {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

#define DD_LMAX_SWITCH(L, ...)                  \
    switch (lmax_of(L)) {                        \
        case 1: { constexpr int LM = 1; __VA_ARGS__; } break;   \
        case 2: { constexpr int LM = 2; __VA_ARGS__; } break;   \
        case 4: { constexpr int LM = 4; __VA_ARGS__; } break;   \
        case 8: { constexpr int LM = 8; __VA_ARGS__; } break;   \
        case 16: { constexpr int LM = 16; __VA_ARGS__; } break; \
        case 32: { constexpr int LM = 32; __VA_ARGS__; } break; \
        default: { constexpr int LM = 0; __VA_ARGS__; } break;  \
    }

cudaError_t launch_pcg_init(const PcgState& s, const PoleGeom& g, const PoleTabs& t, const double* b, int ldb,
                            cudaStream_t st) {
    if (s.ncols <= 0) return cudaSuccess;
    const int W = polesum_warps(g.L);
    const size_t smem = polesum_smem(g.L, W, t.max_sys);
    cudaError_t e = cudaSuccess;
    DD_LMAX_SWITCH(g.L, {
        e = set_smem(k_pcg_init<LM>, smem);
        if (e == cudaSuccess) k_pcg_init<LM><<<s.ncols, 32 * W, smem, st>>>(s, g, t, b, ldb);
    });
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_pcg_iter(const PcgState& s, const PoleGeom& g, const PoleTabs& t, cudaStream_t st) {
    if (s.ncols <= 0) return cudaSuccess;
    const int W = polesum_warps(g.L);
    const size_t smem = polesum_smem(g.L, W, t.max_sys);
    cudaError_t e = cudaSuccess;
    DD_LMAX_SWITCH(g.L, {
        e = set_smem(k_pcg_iter<LM>, smem);
        if (e == cudaSuccess) k_pcg_iter<LM><<<s.ncols, 32 * W, smem, st>>>(s, g, t);
    });
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_precond(int ncols, const int* col_param, const PoleGeom& g, const PoleTabs& t, const double* r,
                           int ldr, double* z, int ldz, cudaStream_t st) {
    if (ncols <= 0) return cudaSuccess;
    const int W = polesum_warps(g.L);
    const size_t smem = polesum_smem(g.L, W, t.max_sys);
    cudaError_t e = cudaSuccess;
    DD_LMAX_SWITCH(g.L, {
        e = set_smem(k_precond<LM>, smem);
        if (e == cudaSuccess) k_precond<LM><<<ncols, 32 * W, smem, st>>>(ncols, col_param, g, t, r, ldr, z, ldz);
    });
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_copy_cols(int n, int ncols, const double* src, int lds, double* dst, int ldd, cudaStream_t st) {
    if (n <= 0 || ncols <= 0) return cudaSuccess;
    const size_t total = (size_t)n * ncols;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_copy_cols<<<blocks, 256, 0, st>>>(n, ncols, src, lds, dst, ldd);
    return cudaGetLastError();
}

cudaError_t launch_check_params(int ncols, const int* col_param, int n_param, int* flag, cudaStream_t st) {
    if (ncols <= 0) return cudaSuccess;
    k_check_params<<<(ncols + 255) / 256, 256, 0, st>>>(ncols, col_param, n_param, flag);
    return cudaGetLastError();
}

}  // namespace dd
