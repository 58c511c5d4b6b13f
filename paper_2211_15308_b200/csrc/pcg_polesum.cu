// Pole sum of the RA preconditioner and the fused PCG vector updates (sm_100a).
//
// Preconditioner (Eq.(8)):
//     z = c0 M_Γ^-1 r + Σ_k c_k (A_Γ - p_k M_Γ)^-1 r
// 1D Γ: every system is symmetric Toeplitz tridiagonal (d, e), SPD and diagonally dominant for
// p < 0 (no pivoting).  Partitioned solve ("group" = G warps = T = 32G threads per system):
//   thread τ owns rows [τ LL, (τ+1) LL): interior rows τLL .. τLL+LL-2, separator row τLL+LL-1;
//   interiors, in registers:  y = T^-1 r_int by Thomas with precomputed pivots (fully unrolled,
//   LL <= 32), then x_int = y - e g_{τ-1} u - e g_τ J u  (u = T^-1 e_1, precomputed);
//   separators: the T-row reduced tridiagonal system by parallel cyclic reduction — warp
//   shuffles when G = 1, a double-buffered shared-memory exchange with one named barrier per
//   step when G > 1 (log2 T steps, precomputed multipliers).
// Rows >= n are padding with x = 0 (the Dirichlet end of Γ).  The pivots, u and PCR multipliers
// are computed on the host in long double (dd_api.cpp), so the fp64 sweeps keep ~1e-15 accuracy
// even for the nearly singular pole closest to 0.
// A CTA owns one column; its NG groups take systems k ≡ group (mod NG), accumulate their share of
// the pole sum in registers, and the NG partial sums are combined in fixed group order:
// bitwise reproducible.
//
// PCG: one fused kernel per iteration after the two
// GEMMs: α = ρ/(p·q); x += αp; r -= αq; z = P r; ρ' = r·z; η test; β = ρ'/ρ; p = z + βp.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "dd_internal.h"

namespace dd {

// Programmatic dependent launch (no-ops unless the launch opted in): dependents may launch at
// entry; the wait precedes every read of data an earlier kernel of the stream writes.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait_prior() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename Kern, typename... Args>
static cudaError_t launch_ex(Kern k, int grid, int block, size_t smem, cudaStream_t st, bool pdl, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(block, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, args...);
}

// transposed, padded layout of a column in shared memory: [row-in-chunk i][thread τ], stride T+1
__device__ __forceinline__ int tix(int i, int tau, int T) { return i * (T + 1) + tau; }
__device__ __forceinline__ int clamp_param(int p, int n_param) { return p < 0 ? 0 : (p >= n_param ? n_param - 1 : p); }

template <int G>
__device__ __forceinline__ void group_sync(int group) {
    if constexpr (G == 1) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(1 + group), "r"(32 * G) : "memory");
    }
}

// Value of `v` held by thread τ+d of the group (0 outside [0, T)).  G = 1: shuffles.
template <int G>
__device__ __forceinline__ double group_shift(double v, int d, int tau, double* xb, int group) {
    constexpr int T = 32 * G;
    if constexpr (G == 1) {
        double r = d > 0 ? __shfl_down_sync(0xffffffffu, v, d) : __shfl_up_sync(0xffffffffu, v, -d);
        const int src = tau + d;
        return (src < 0 || src >= T) ? 0.0 : r;
    } else {
        xb[tau] = v;
        group_sync<G>(group);
        const int src = tau + d;
        const double r = (src < 0 || src >= T) ? 0.0 : xb[src];
        group_sync<G>(group);
        return r;
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Read-only global load issued where written (volatile: not sunk towards its first use).
__device__ __forceinline__ double ldg_early(const double* p) {
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}

// Asynchronously stage this parameter set's interior tables (4 contiguous blocks of nsys x LL
// doubles; v2: the parameter set's W + records block) into scratch with cp.async (LDGSTS);
// block_polesum waits for them.  Called at kernel entry so the copies overlap the vector passes.
__device__ __forceinline__ void stage_tables(const PoleTabs& t, const PoleGeom& g, int param, double* scratch) {
    if (t.v2) {
        const double* src = t.v2 + (size_t)param * t.v2_stride;
        const int cnt = (V2_WSZ + V2_REC * t.nsys[param]) / 2;          // 16-byte pieces
        for (int idx = threadIdx.x; idx < cnt; idx += blockDim.x) {
            const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(scratch + 2 * idx));
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src + 2 * idx));
        }
        asm volatile("cp.async.commit_group;\n" ::);
        return;
    }
    const int LL = g.LL;
    const int cnt = t.nsys[param] * LL;
    const size_t tstride = (size_t)t.max_sys * LL;
    const size_t src0 = (size_t)param * t.max_sys * LL;
#pragma unroll
    for (int which = 0; which < 4; which++) {
        const double* src = (which == 0 ? t.invb : (which == 1 ? t.cpr : (which == 2 ? t.ufull : t.upart))) + src0;
        double* dst = scratch + which * tstride;
        for (int idx = threadIdx.x; idx < cnt; idx += blockDim.x) {
            const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst + idx));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(src + idx));
        }
    }
    asm volatile("cp.async.commit_group;\n" ::);
}

// z = P r for the CTA's column.  R: input (transposed), Z: output (transposed, written by every
// thread for its own chunk after the fixed-order combine).  sm: scratch (tables already staged).
// FULL: the chunk length equals LMAX at compile time (n + 1 = T * LMAX; all BASELINE configs), so
// the unrolled sweeps carry no per-row branch and every table / R load hoists off the FMA chain.
template <int LMAX, int G, int NG, bool FULL>
__device__ void block_polesum_impl(const PoleTabs& t, const PoleGeom& g, int param, const double* R, double* Z,
                                   double* scratch, long long* dbg) {
#define DD_PS(i) \
    if (dbg && threadIdx.x == 0) dbg[i] = clock64()
    constexpr int T = 32 * G;
    const int LL = FULL ? LMAX : g.LL;
    const int tot = LL * (T + 1);
    const int tid = threadIdx.x;
    const int group = tid / T, tau = tid % T;
    const int nsys = t.nsys[param];
    const size_t pbase = (size_t)param * t.max_sys;
    const size_t tstride = (size_t)t.max_sys * LL;             // tables: [which][k][i], staged by stage_tables()
    double* tab = scratch;
    double* xbuf = scratch + 4 * tstride;                      // [NG][2][T] PCR exchange (G > 1)
    double* Zw = xbuf + 2 * NG * T;                            // [NG][tot] per-group partial sums
    double* zg = Zw + (size_t)group * tot;
#pragma unroll
    for (int i = 0; i < LMAX; i++)
        if (i < LL) zg[tix(i, tau, T)] = 0.0;
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    DD_PS(6);

    // FULL (n + 1 = T LL): every chunk has LL - 1 interior rows; only the last separator is padding
    const int Lr = FULL ? LMAX - 1 : (tau < g.part ? LL - 1 : (tau == g.part ? g.Lr_part : 0));
    const int Lr_next = FULL ? LMAX - 1 : ((tau + 1) < g.part ? LL - 1 : ((tau + 1) == g.part ? g.Lr_part : 0));
    const bool sep_real = FULL ? (tau < T - 1) : (tau < g.part);
    double* xb = xbuf + (size_t)group * 2 * T;

    for (int k = group; k < nsys; k += NG) {
        const double* ib = tab + (size_t)k * LL;
        const double* cp = ib + tstride;
        const double* u = (FULL || tau < g.part) ? ib + 2 * tstride : ib + 3 * tstride;
        // Per-system scalars and this thread's PCR multipliers: issued here (volatile loads are not
        // sunk by the compiler) so their global latency hides under the Thomas sweeps below.
        const double e = ldg_early(&t.e[pbase + k]), wk = ldg_early(&t.w[pbase + k]);
        const double* pa = t.pa + (pbase + k) * (size_t)g.J * T;
        const double* pb = t.pb + (pbase + k) * (size_t)g.J * T;
        constexpr int JM = G == 1 ? 5 : (G == 2 ? 6 : (G == 4 ? 7 : 8));   // log2(32 G)
        double pav[JM], pbv[JM];
#pragma unroll
        for (int j = 0; j < JM; j++) {
            pav[j] = ldg_early(&pa[j * T + tau]);
            pbv[j] = ldg_early(&pb[j * T + tau]);
        }
        const double pinv = ldg_early(&t.pinvb[(pbase + k) * T + tau]);

        // forward:  ỹ_i = r_i/b'_i - (e/b'_i) ỹ_{i-1}
        // (rows in batches of 8: the batch's shared-memory loads issue together, then the chain runs)
        constexpr int BT = LMAX < 8 ? LMAX : 8;
        double y[LMAX];
        double prev = 0.0, y_last = 0.0;
#pragma unroll
        for (int i0 = 0; i0 < LMAX; i0 += BT) {
            double rb[BT], cb[BT];
#pragma unroll
            for (int j = 0; j < BT; j++) {
                const int i = i0 + j;
                rb[j] = 0.0;
                cb[j] = 0.0;
                if (i < LL - 1) {
                    rb[j] = R[tix(i, tau, T)] * ib[i];
                    cb[j] = cp[i];
                }
            }
#pragma unroll
            for (int j = 0; j < BT; j++) {
                const int i = i0 + j;
                if (i < LL - 1) {
                    const double v = fma(-cb[j], prev, rb[j]);
                    y[i] = i < Lr ? v : 0.0;
                    if (i < Lr) y_last = v;
                    prev = y[i];
                } else {
                    y[i] = 0.0;
                }
            }
        }
        if (k == 0) DD_PS(7);
        // backward:  y_i = ỹ_i - (e/b'_i) y_{i+1}
        double next = 0.0;
#pragma unroll
        for (int i0 = LMAX - 1; i0 >= 0; i0 -= BT) {
            double cb[BT];
#pragma unroll
            for (int j = 0; j < BT; j++) {
                const int i = i0 - j;
                cb[j] = (i >= 0 && i < LL - 1) ? cp[i] : 0.0;
            }
#pragma unroll
            for (int j = 0; j < BT; j++) {
                const int i = i0 - j;
                if (i >= 0 && i < LL - 1) {
                    y[i] = fma(-cb[j], next, y[i]);
                    next = y[i];
                }
            }
        }
        const double y_first = Lr > 0 ? y[0] : 0.0;
        const double y_first_next = group_shift<G>(y_first, 1, tau, xb, group);
        double rs = 0.0;
        if (sep_real) {
            rs = R[tix(LL - 1, tau, T)];
            if (Lr > 0) rs -= e * y_last;
            if (tau < T - 1 && Lr_next > 0) rs -= e * y_first_next;
        }
        if (k == 0) DD_PS(8);
        // parallel cyclic reduction over the T separators
        if constexpr (G == 1) {
#pragma unroll
            for (int j = 0; j < 5; j++) {
                const int s = 1 << j;
                double rm = __shfl_up_sync(0xffffffffu, rs, s);
                double rp = __shfl_down_sync(0xffffffffu, rs, s);
                if (tau < s) rm = 0.0;
                if (tau + s > T - 1) rp = 0.0;
                rs = rs - pav[j] * rm - pbv[j] * rp;
            }
        } else {
            // double-buffered shared-memory exchange, one named barrier per step
#pragma unroll
            for (int j = 0; j < JM; j++) {
                const int s = 1 << j;
                double* buf = xb + (j & 1) * T;
                buf[tau] = rs;
                group_sync<G>(group);
                const double rm = (tau >= s) ? buf[tau - s] : 0.0;
                const double rp = (tau + s < T) ? buf[tau + s] : 0.0;
                rs = rs - pav[j] * rm - pbv[j] * rp;
            }
            group_sync<G>(group);
        }
        if (k == 0) DD_PS(9);
        const double gsep = sep_real ? rs * pinv : 0.0;
        const double gleft = group_shift<G>(gsep, -1, tau, xb, group);
        const double eg0 = e * gleft, eg1 = e * gsep;
        {
#pragma unroll
            for (int i0 = 0; i0 < LMAX; i0 += BT) {
                double ua[BT], ub[BT], zo[BT];
#pragma unroll
                for (int j = 0; j < BT; j++) {
                    const int i = i0 + j;
                    ua[j] = 0.0; ub[j] = 0.0; zo[j] = 0.0;
                    if (i < LL - 1 && i < Lr) {
                        ua[j] = u[i];
                        ub[j] = u[Lr - 1 - i];
                        zo[j] = zg[tix(i, tau, T)];
                    }
                }
#pragma unroll
                for (int j = 0; j < BT; j++) {
                    const int i = i0 + j;
                    if (i < LL - 1 && i < Lr) {
                        const double x = y[i] - eg0 * ua[j] - eg1 * ub[j];
                        zg[tix(i, tau, T)] = fma(wk, x, zo[j]);
                    }
                }
            }
            if (LL >= 1) {
                const int ix = tix(LL - 1, tau, T);
                zg[ix] = fma(wk, gsep, zg[ix]);
            }
        }
    }
    DD_PS(10);
    // fixed-order combine of the NG group partials: Z = z_0 + z_1 + ... + z_{NG-1}
    __syncthreads();
    for (int idx = tid; idx < tot; idx += blockDim.x) {
        double acc = Zw[idx];
        for (int gg = 1; gg < NG; gg++) acc += Zw[(size_t)gg * tot + idx];
        Z[idx] = acc;
    }
    __syncthreads();
#undef DD_PS
}

// FULL geometry (n + 1 = T LL: every chunk has LL - 1 interior rows, only the last separator is
// padding) — the BASELINE shapes.  Same arithmetic as block_polesum_impl, restructured for issue
// and latency: the group's share of the pole sum is accumulated in registers (no shared-memory
// read-modify-write per row and system), the broadcast table reads are 16-byte vector loads of
// a whole row pair, and the PCR multipliers / per-system scalars of the NEXT system are fetched
// from global memory while the current one is swept.
template <int LL, int G, int NG>
__device__ void block_polesum_full(const PoleTabs& t, int param, const double* R, double* Z, double* scratch,
                                   long long* dbg) {
    constexpr int T = 32 * G;
    constexpr int JM = G == 1 ? 5 : (G == 2 ? 6 : (G == 4 ? 7 : 8));   // log2(32 G)
    constexpr int tot = LL * (T + 1);
    static_assert(LL % 2 == 0, "row pairs");
    const int tid = threadIdx.x;
    const int group = tid / T, tau = tid % T;
    const int nsys = t.nsys[param];
    const size_t pbase = (size_t)param * t.max_sys;
    const size_t tstride = (size_t)t.max_sys * LL;
    const double* tab = scratch;
    double* xbuf = scratch + 4 * tstride;
    double* Zw = xbuf + 2 * NG * T;
    double* xb = xbuf + (size_t)group * 2 * T;
    const bool sep_real = tau < T - 1;
    const double* Rt = R + tau;              // row i of this thread's chunk: Rt[i * (T + 1)]

    double zacc[LL];
#pragma unroll
    for (int i = 0; i < LL; i++) zacc[i] = 0.0;
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    if (dbg && threadIdx.x == 0) dbg[6] = clock64();

    for (int k = group; k < nsys; k += NG) {
        // per-system scalars and this thread's PCR multipliers: issued first (volatile loads are not
        // sunk), their latency hides under the sweeps
        const double e = ldg_early(&t.e[pbase + k]), wk = ldg_early(&t.w[pbase + k]);
        double pav[JM], pbv[JM];
        {
            const double* pa = t.pa + (pbase + k) * (size_t)JM * T + tau;
            const double* pb = t.pb + (pbase + k) * (size_t)JM * T + tau;
#pragma unroll
            for (int j = 0; j < JM; j++) { pav[j] = ldg_early(&pa[j * T]); pbv[j] = ldg_early(&pb[j * T]); }
        }
        const double pinv = ldg_early(&t.pinvb[(pbase + k) * T + tau]);
        const double2* ib2 = reinterpret_cast<const double2*>(tab + (size_t)k * LL);
        const double2* cp2 = reinterpret_cast<const double2*>(tab + tstride + (size_t)k * LL);
        const double2* u2 = reinterpret_cast<const double2*>(tab + 2 * tstride + (size_t)k * LL);

        // forward:  ỹ_i = r_i/b'_i - (e/b'_i) ỹ_{i-1},  i = 0 .. LL-2
        double y[LL];
        double prev = 0.0;
#pragma unroll
        for (int i2 = 0; i2 < LL / 2; i2++) {
            const double2 ib = ib2[i2], cp = cp2[i2];
            const int i = 2 * i2;
            if (i < LL - 1) { prev = fma(-cp.x, prev, Rt[i * (T + 1)] * ib.x); y[i] = prev; }
            if (i + 1 < LL - 1) { prev = fma(-cp.y, prev, Rt[(i + 1) * (T + 1)] * ib.y); y[i + 1] = prev; }
        }
        const double y_last = y[LL - 2];
        // backward:  y_i = ỹ_i - (e/b'_i) y_{i+1}
#pragma unroll
        for (int i2 = (LL - 2) / 2; i2 >= 0; i2--) {
            const double2 cp = cp2[i2];
            const int i = 2 * i2;
            if (i + 1 <= LL - 3) y[i + 1] = fma(-cp.y, y[i + 2], y[i + 1]);
            if (i <= LL - 3) y[i] = fma(-cp.x, y[i + 1], y[i]);
        }
        const double y_first_next = group_shift<G>(y[0], 1, tau, xb, group);
        double rs = 0.0;
        if (sep_real) rs = Rt[(LL - 1) * (T + 1)] - e * y_last - e * y_first_next;
        // parallel cyclic reduction over the T separators
        if constexpr (G == 1) {
#pragma unroll
            for (int j = 0; j < 5; j++) {
                const int s = 1 << j;
                double rm = __shfl_up_sync(0xffffffffu, rs, s);
                double rp = __shfl_down_sync(0xffffffffu, rs, s);
                if (tau < s) rm = 0.0;
                if (tau + s > T - 1) rp = 0.0;
                rs = rs - pav[j] * rm - pbv[j] * rp;
            }
        } else {
#pragma unroll
            for (int j = 0; j < JM; j++) {
                const int s = 1 << j;
                double* buf = xb + (j & 1) * T;
                buf[tau] = rs;
                group_sync<G>(group);
                const double rm = (tau >= s) ? buf[tau - s] : 0.0;
                const double rp = (tau + s < T) ? buf[tau + s] : 0.0;
                rs = rs - pav[j] * rm - pbv[j] * rp;
            }
            group_sync<G>(group);
        }
        const double gsep = sep_real ? rs * pinv : 0.0;
        const double gleft = group_shift<G>(gsep, -1, tau, xb, group);
        const double eg0 = e * gleft, eg1 = e * gsep;
        // x_i = y_i - e g_{τ-1} u_i - e g_τ u_{LL-2-i};  z += w_k x
#pragma unroll
        for (int i2 = 0; i2 < LL / 2; i2++) {
            const double2 ua = u2[i2];
            const int i = 2 * i2;
            if (i < LL - 1) zacc[i] = fma(wk, y[i] - eg0 * ua.x - eg1 * tab[2 * tstride + (size_t)k * LL + (LL - 2 - i)], zacc[i]);
            if (i + 1 < LL - 1)
                zacc[i + 1] = fma(wk, y[i + 1] - eg0 * ua.y - eg1 * tab[2 * tstride + (size_t)k * LL + (LL - 3 - i)], zacc[i + 1]);
        }
        zacc[LL - 1] = fma(wk, gsep, zacc[LL - 1]);
        if (dbg && threadIdx.x == 0 && k == 0) dbg[7] = dbg[8] = dbg[9] = clock64();
    }
    if (dbg && threadIdx.x == 0) dbg[10] = clock64();
    // fixed-order combine of the NG group partials
    double* zg = Zw + (size_t)group * tot;
#pragma unroll
    for (int i = 0; i < LL; i++) zg[tix(i, tau, T)] = zacc[i];
    __syncthreads();
    for (int idx = tid; idx < tot; idx += blockDim.x) {
        double acc = Zw[idx];
        for (int gg = 1; gg < NG; gg++) acc += Zw[(size_t)gg * tot + idx];
        Z[idx] = acc;
    }
    __syncthreads();
}

// Merged-interior pole sum (FULL geometry, 16-row chunks, T = 32 G chunks, NT threads = Q
// sub-threads per chunk).  Same operator as block_polesum_full, reorganised so that no thread runs
// a per-system dependent chain or waits on a per-system barrier:
//   chunk interior of system k:  x_int = T_k^-1 r_int - e_k (g_k,τ-1 u_k + g_k,τ J u_k),  u_k = T_k^-1 e_1
//   Σ_k w_k x_int = W r_int - Σ_k w_k e_k (g_k,τ-1 u_k + g_k,τ J u_k),   W = Σ_k w_k T_k^-1 (host, long double)
//   separators: δ_k g_τ + ε_k (g_τ-1 + g_τ+1) = r_sep,τ - e_k (last(T_k^-1 r_int,τ) + first(T_k^-1 r_int,τ+1))
// Phase A (chunk-parallel): W r_int for the thread's rows and, for its share of the systems, the two
//   end rows of T_k^-1 r_int (dot products with tf_k = first row of T_k^-1; last row = tf_k reversed);
// Phase B (one warp per system): the T - 1 separator unknowns by parallel cyclic reduction on the
//   antisymmetric period-2T extension (g_0 = g_T = 0 by symmetry), whose multipliers are the same at
//   every position — log2(2T) steps with two scalars per step from the table, exchanges through the
//   system's own shared-memory rows and __syncwarp only;
// Phase C (chunk-parallel): the corrections Σ_k w_k e_k (...) and z_sep = Σ_k w_k g_k,τ.
// Three block barriers per pole sum.  scratch: [tables | hl (max_sys x (T+1)) | yf (same)].
template <int T, int NT>
__device__ void block_polesum_v2(const PoleTabs& t, int param, const double* R, double* Z, double* scratch,
                                 long long* dbg = nullptr) {
    constexpr int Q = NT / T;                    // sub-threads per chunk
    constexpr int RPT = V2_L / Q;                // output rows per thread
    constexpr int S = T / 32;                    // separators per lane in phase B
    constexpr int TP = T + 1;                    // row stride of hl / yf
    constexpr int NW = NT / 32;
    constexpr int JS = T == 32 ? 6 : (T == 64 ? 7 : (T == 128 ? 8 : 9));   // log2(2T)
    static_assert(Q >= 1 && V2_L % Q == 0 && T % 32 == 0, "v2 geometry");
    const double* tab = scratch;
    const int nsys = t.nsys[param];
    double* hl = scratch + t.v2_stride;
    double* yf = hl + (size_t)t.max_sys * TP;
    const int tid = threadIdx.x, tau = tid % T, q = tid / T;
    asm volatile("cp.async.wait_all;\n" ::);
    __syncthreads();
    if (dbg && threadIdx.x == 0) dbg[6] = clock64();
    // ---- phase A
    double r[V2_L];
#pragma unroll
    for (int i = 0; i < V2_L; i++) r[i] = R[i * (T + 1) + tau];
    double acc[RPT];
#pragma unroll
    for (int u = 0; u < RPT; u++) {
        const int i = q * RPT + u;               // contiguous rows per thread (phase C loads pairs)
        double a = 0.0;
        if (i < V2_L - 1) {
            const double2* wr = reinterpret_cast<const double2*>(tab + i * 16);
#pragma unroll
            for (int j2 = 0; j2 < 8; j2++) {
                const double2 wv = wr[j2];
                a = fma(wv.x, r[2 * j2], a);
                if (2 * j2 + 1 < V2_L - 1) a = fma(wv.y, r[2 * j2 + 1], a);
            }
        }
        acc[u] = a;
    }
#pragma unroll 2
    for (int k = q; k < ((t.v2_skip & 1) ? 0 : nsys); k += Q) {
        const double* rec = tab + V2_WSZ + k * V2_REC;
        const double2* tf2 = reinterpret_cast<const double2*>(rec);
        double f0 = 0.0, l0 = 0.0, f1 = 0.0, l1 = 0.0;        // two chains each (even / odd terms)
#pragma unroll
        for (int j2 = 0; j2 < 8; j2++) {
            const double2 tv = tf2[j2];
            const int j = 2 * j2;
            f0 = fma(tv.x, r[j], f0);
            l0 = fma(tv.x, r[V2_L - 2 - j], l0);
            if (j + 1 < V2_L - 1) {
                f1 = fma(tv.y, r[j + 1], f1);
                l1 = fma(tv.y, r[V2_L - 3 - j], l1);
            }
        }
        hl[k * TP + tau] = fma(-rec[V2_E], l0 + l1, r[V2_L - 1]);   // r_sep - e last(T^-1 r_int)
        yf[k * TP + tau] = f0 + f1;                                 // first(T^-1 r_int)
    }
    __syncthreads();
    if (dbg && threadIdx.x == 0) dbg[7] = clock64();
    // ---- phase B: separators of up to NSI systems per warp, interleaved (independent chains:
    // the PCR is latency-bound, so a warp advances its systems' steps together).  Each system's
    // values live in its own hl row (positions 0..T, v_0 = v_T = 0); the antisymmetric period-2T
    // extension is read through the reflection x -> -x (x < 0), 2T - x (x > T) with the sign
    // flipped — no halo buffer; read, __syncwarp, write, __syncwarp per step.
    if (!t.pcr_smem) {
        // Register form (default): lane owns σ = 32 sl + lane + 1, sl < S, for one system at a
        // time; distances below 32 by warp shuffles (the S registers shifted by st lanes, the
        // wrap into the neighbouring register, the reflections at σ < 0 and σ > T), distances
        // 32 m by register renaming plus a lane reversal where the reflection is read.  Same
        // operations in the same order as the shared-memory form (bitwise equal), without its
        // row stores and __syncwarp pairs.
        const int warp = tid >> 5, lane = tid & 31;
        for (int k = warp; k < ((t.v2_skip & 2) ? 0 : nsys); k += NW) {
            const double* rec = tab + V2_WSZ + k * V2_REC;
            double* A = hl + (size_t)k * TP;
            const double e = rec[V2_E];
            double v[S];
#pragma unroll
            for (int sl = 0; sl < S; sl++) {
                const int sg = 32 * sl + lane + 1;
                v[sl] = sg < T ? fma(-e, yf[k * TP + sg], A[sg - 1]) : 0.0;
            }
#pragma unroll
            for (int j = 0; j < JS; j++) {
                const int st = 1 << j;
                const double al = rec[V2_AL + j];
                double nv[S];
                if (st < 32) {
                    double a[S], b[S];
#pragma unroll
                    for (int sl = 0; sl < S; sl++) {
                        a[sl] = __shfl_sync(0xffffffffu, v[sl], (lane - st) & 31);
                        b[sl] = __shfl_sync(0xffffffffu, v[sl], (lane + st) & 31);
                    }
                    const double rl = __shfl_sync(0xffffffffu, v[0], max(st - lane - 2, 0));
                    const double rr = __shfl_sync(0xffffffffu, v[S - 1], min(max(62 - lane - st, 0), 31));
                    const double reflL = lane == st - 1 ? 0.0 : -rl;
#pragma unroll
                    for (int sl = 0; sl < S; sl++) {
                        const double left = lane >= st ? a[sl] : (sl >= 1 ? a[sl >= 1 ? sl - 1 : 0] : reflL);
                        const double right = lane + st <= 31 ? b[sl] : (sl <= S - 2 ? b[sl <= S - 2 ? sl + 1 : 0] : -rr);
                        nv[sl] = fma(-al, left + right, v[sl]);
                    }
                } else {
                    const int m = st >> 5;
                    // value at σ = 32 r + 31 - lane (lane 30 - lane of register r; lane 31: its own
                    // register r - 1, or 0 at σ = 0)
                    auto rev = [&](int r) {
                        const double x = __shfl_sync(0xffffffffu, v[r], (30 - lane) & 31);
                        const double own = r >= 1 ? v[r >= 1 ? r - 1 : 0] : 0.0;
                        return lane <= 30 ? x : own;
                    };
#pragma unroll
                    for (int sl = 0; sl < S; sl++) {
                        const double left = sl >= m ? v[sl >= m ? sl - m : 0] : -rev(m - sl - 1);
                        const double right = sl + m <= S - 1 ? v[sl + m <= S - 1 ? sl + m : 0] : -rev(2 * S - sl - m - 1);
                        nv[sl] = fma(-al, left + right, v[sl]);
                    }
                }
#pragma unroll
                for (int sl = 0; sl < S; sl++) v[sl] = (sl == S - 1 && lane == 31) ? 0.0 : nv[sl];   // σ = T stays 0
            }
            const double dinv = rec[V2_DINV];
            __syncwarp();                                   // the prologue's reads of this row precede the writes
#pragma unroll
            for (int sl = 0; sl < S; sl++) A[32 * sl + lane + 1] = v[sl] * dinv;   // g at σ (σ = T: 0)
            if (lane == 0) A[0] = 0.0;
        }
    } else {
        const int warp = tid >> 5, lane = tid & 31;
        constexpr int NSI = 3;
        for (int k0 = warp; k0 < ((t.v2_skip & 2) ? 0 : nsys); k0 += NW * NSI) {
            double rs[NSI][S];
            double* A[NSI];
#pragma unroll
            for (int i = 0; i < NSI; i++) {
                const int k = k0 + i * NW;
                A[i] = hl + (size_t)(k < nsys ? k : 0) * TP;
                if (k < nsys) {
                    const double e = tab[V2_WSZ + k * V2_REC + V2_E];
                    const double* B = yf + k * TP;
#pragma unroll
                    for (int sl = 0; sl < S; sl++) {
                        const int sg = 32 * sl + lane + 1;     // separator σ = τ + 1 in 1..T (σ = T: boundary)
                        rs[i][sl] = sg < T ? fma(-e, B[sg], A[i][sg - 1]) : 0.0;
                    }
                }
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < NSI; i++)
                if (k0 + i * NW < nsys) {
#pragma unroll
                    for (int sl = 0; sl < S; sl++) A[i][32 * sl + lane + 1] = rs[i][sl];   // v_T = 0 from σ = T
                    if (lane == 0) A[i][0] = 0.0;
                }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < JS; j++) {
                const int st = 1 << j;
#pragma unroll
                for (int i = 0; i < NSI; i++) {
                    const int k = k0 + i * NW;
                    if (k < nsys) {
                        const double al = tab[V2_WSZ + k * V2_REC + V2_AL + j];
#pragma unroll
                        for (int sl = 0; sl < S; sl++) {
                            const int sg = 32 * sl + lane + 1;
                            const int xl = sg - st, xr = sg + st;
                            const double vl = xl < 0 ? -A[i][-xl] : A[i][xl];
                            const double vr = xr > T ? -A[i][2 * T - xr] : A[i][xr];
                            rs[i][sl] = sg < T ? fma(-al, vl + vr, rs[i][sl]) : 0.0;
                        }
                    }
                }
                __syncwarp();
#pragma unroll
                for (int i = 0; i < NSI; i++)
                    if (k0 + i * NW < nsys) {
#pragma unroll
                        for (int sl = 0; sl < S; sl++) A[i][32 * sl + lane + 1] = rs[i][sl];
                    }
                __syncwarp();
            }
#pragma unroll
            for (int i = 0; i < NSI; i++) {
                const int k = k0 + i * NW;
                if (k < nsys) {
                    const double dinv = tab[V2_WSZ + k * V2_REC + V2_DINV];
#pragma unroll
                    for (int sl = 0; sl < S; sl++) A[i][32 * sl + lane + 1] = rs[i][sl] * dinv;   // g at σ (σ = T: 0)
                }
            }
        }
    }
    __syncthreads();
    if (dbg && threadIdx.x == 0) dbg[8] = clock64();
    // ---- phase C: corrections and separator rows
    double acc2[RPT];                            // second chain (odd systems)
#pragma unroll
    for (int u = 0; u < RPT; u++) acc2[u] = 0.0;
    // the thread's rows are contiguous (i = q RPT + u), so the coefficients w e tf_k[i] and their
    // mirror w e tf_k[14 - i] (stored reversed in the record) load as 16-byte pairs
    static_assert(RPT % 2 == 0, "row pairs");
    for (int k0 = 0; k0 < ((t.v2_skip & 4) ? 0 : nsys); k0 += 2) {
#pragma unroll
        for (int kk = 0; kk < 2; kk++) {
            const int k = k0 + kk;
            if (k < nsys) {
                const double* rec = tab + V2_WSZ + k * V2_REC;
                const double gl = hl[k * TP + tau], gr = hl[k * TP + tau + 1];    // g_k,τ-1 and g_k,τ
                const double wk = rec[V2_WK];
                const double2* wf2 = reinterpret_cast<const double2*>(rec + 16 + q * RPT);
                const double2* wr2 = reinterpret_cast<const double2*>(rec + V2_WREV + q * RPT);
                double* a = kk ? acc2 : acc;
#pragma unroll
                for (int v = 0; v < RPT / 2; v++) {
                    const double2 f = wf2[v], r2 = wr2[v];
                    const int i = q * RPT + 2 * v;
                    a[2 * v] = fma(-gl, f.x, fma(-gr, r2.x, a[2 * v]));
                    a[2 * v + 1] = (i + 1 < V2_L - 1) ? fma(-gl, f.y, fma(-gr, r2.y, a[2 * v + 1]))
                                                      : fma(wk, gr, a[2 * v + 1]);        // separator row
                }
            }
        }
    }
#pragma unroll
    for (int u = 0; u < RPT; u++) Z[(q * RPT + u) * (T + 1) + tau] = acc[u] + acc2[u];
    __syncthreads();
    if (dbg && threadIdx.x == 0) dbg[9] = dbg[10] = clock64();
}

template <int LMAX, int G, int NG, int V = 0>
__device__ __forceinline__ void block_polesum(const PoleTabs& t, const PoleGeom& g, int param, const double* R,
                                              double* Z, double* scratch, long long* dbg = nullptr) {
    if constexpr (V >= 1) {                      // t.v2 set: FULL geometry with 16-row chunks
        block_polesum_v2<32 * G, 32 * G * NG>(t, param, R, Z, scratch, dbg);
        return;
    } else {
    if (g.LL == LMAX && g.n + 1 == g.T * g.LL) {
        if constexpr (LMAX >= 2) {
            block_polesum_full<LMAX, G, NG>(t, param, R, Z, scratch, dbg);
            return;
        }
        block_polesum_impl<LMAX, G, NG, true>(t, g, param, R, Z, scratch, dbg);
    }
    else block_polesum_impl<LMAX, G, NG, false>(t, g, param, R, Z, scratch, dbg);
    }
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
    // no leading barrier: red is used by block_sum2 only, and every call ends with one after its reads
    if (lane == 0) { red[warp] = a; red[32 + warp] = b; }
    __syncthreads();
    double sa = 0.0, sb = 0.0;
    for (int w = 0; w < W; w++) { sa += red[w]; sb += red[32 + w]; }
    a = sa; b = sb;
    __syncthreads();
}

// smem index of natural row ρ of the column
__device__ __forceinline__ int tpos(int row, const PoleGeom& g) { return tix(row % g.LL, row / g.LL, g.T); }

struct Smem {
    double *R, *Z, *scratch;
};
__device__ __forceinline__ Smem carve(double* sm, const PoleGeom& g) {
    const int tot = g.LL * (g.T + 1);
    return Smem{sm, sm + tot, sm + 2 * tot};
}
// V = 2 (merged-interior pole sum, compact): Z shares the yf rows of block_polesum_v2 (yf is last
// read at the start of phase B, Z first written in phase C, after a block barrier), so the CTA
// needs tot + v2_stride + 2 max_sys (T + 1) doubles and three 256-thread CTAs fit on an SM.
template <int V>
__device__ __forceinline__ Smem carve_v(double* sm, const PoleGeom& g, const PoleTabs& t) {
    if constexpr (V == 2) {
        const int tot = g.LL * (g.T + 1);
        double* scratch = sm + tot;
        return Smem{sm, scratch + t.v2_stride + (size_t)t.max_sys * (g.T + 1), scratch};
    } else {
        return carve(sm, g);
    }
}

// ---------------------------------------------------------------------------- kernels
template <int LMAX, int G, int NG, int V>
__global__ void __launch_bounds__(32 * G * NG, (32 * G * NG) <= 256 ? (V == 2 ? 3 : 2) : 1) k_precond(int ncols, const int* __restrict__ col_param, PoleGeom g,
                                                         PoleTabs t, const double* __restrict__ r, int ldr,
                                                         double* __restrict__ z, int ldz) {
    extern __shared__ __align__(16) double sm[];
    const int c = blockIdx.x;
    if (c >= ncols) return;
    pdl_trigger();
    Smem S = carve_v<V>(sm, g, t);
    const int npad = g.T * g.LL;
    const int param = clamp_param(col_param[c], t.n_param);
    stage_tables(t, g, param, S.scratch);
    pdl_wait_prior();
    for (int i = threadIdx.x; i < npad; i += blockDim.x) S.R[tpos(i, g)] = i < g.n ? r[(size_t)c * ldr + i] : 0.0;
    __syncthreads();
    block_polesum<LMAX, G, NG, V>(t, g, param, S.R, S.Z, S.scratch);
    for (int i = threadIdx.x; i < g.n; i += blockDim.x) z[(size_t)c * ldz + i] = S.Z[tpos(i, g)];
}

// RA-evaluated fractional term (Remark 1; dd_frac mode DD_FRAC_RA):
//   u_c = γ_c M_Γ r_F(L) M_Γ x_c,   r_F(L) = fc0 M_Γ^-1 + Σ_k fc_k (A_Γ - fp_k M_Γ)^-1 ≈ L^t,
// i.e. the pole sum of block_polesum on the F tables (one parameter set) between two products
// with the 1D P1 mass M_Γ = (h/6) tridiag(1, 4, 1) (Dirichlet ends).
template <int LMAX, int G, int NG, int V>
__global__ void __launch_bounds__(32 * G * NG, (32 * G * NG) <= 256 ? (V == 2 ? 3 : 2) : 1) k_frac_ra(int ncols, const int* __restrict__ col_param,
                                                         int n_param, const double* __restrict__ gp, PoleGeom g,
                                                         PoleTabs t, const double* __restrict__ x, int ldx,
                                                         double* __restrict__ u, int ldu, double h6) {
    extern __shared__ __align__(16) double sm[];
    const int c = blockIdx.x;
    if (c >= ncols) return;
    pdl_trigger();
    Smem S = carve_v<V>(sm, g, t);
    const int npad = g.T * g.LL, n = g.n;
    stage_tables(t, g, 0, S.scratch);
    pdl_wait_prior();
    const double* xc = x + (size_t)c * ldx;
    for (int i = threadIdx.x; i < npad; i += blockDim.x) {
        double v = 0.0;
        if (i < n) v = h6 * ((i > 0 ? xc[i - 1] : 0.0) + 4.0 * xc[i] + (i + 1 < n ? xc[i + 1] : 0.0));
        S.R[tpos(i, g)] = v;
    }
    __syncthreads();
    block_polesum<LMAX, G, NG, V>(t, g, 0, S.R, S.Z, S.scratch);
    int p = col_param[c];
    p = p < 0 ? 0 : (p >= n_param ? n_param - 1 : p);
    const double gam = gp[p] * h6;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double zm = i > 0 ? S.Z[tpos(i - 1, g)] : 0.0;
        const double zp = i + 1 < n ? S.Z[tpos(i + 1, g)] : 0.0;
        u[(size_t)c * ldu + i] = gam * (zm + 4.0 * S.Z[tpos(i, g)] + zp);
    }
}

// Live column tiles of the batch (s.ntl_bn = 64, or 32 for the grouped Schur GEMM; GEMM output
// tiles with at least one unconverged column):
// every CTA keeps its tile's active-column count current (ntl_cnt, +1 at init, -1 when its column
// freezes); the last-arriving CTA compacts the live tile ids into s.ntl = [count, ids...] and the
// next iteration's GEMMs partition their work over those tiles only.
__device__ __forceinline__ void publish_live_tiles(const PcgState& s, int na) {
    // warp 0 of the last CTA.  All columns active (the common case until the last iterations):
    // the identity list, no memory round trip; otherwise one L2 round trip per 32 tiles (ballot +
    // prefix popcount over the per-tile counters).
    if (!s.ntl || threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    const int nt = (s.ncols + s.ntl_bn - 1) / s.ntl_bn;
    if (na == s.ncols) {
        for (int j = lane; j < nt; j += 32) s.ntl[1 + j] = j;
        if (lane == 0) s.ntl[0] = nt;
        return;
    }
    int total = 0;
    for (int base = 0; base < nt; base += 32) {
        const int j = base + lane;
        const bool live = j < nt && __ldcg(&s.ntl_cnt[j]) > 0;
        const unsigned m = __ballot_sync(0xffffffffu, live);
        if (live) s.ntl[1 + total + __popc(m & ((1u << lane) - 1u))] = j;
        total += __popc(m);
    }
    if (lane == 0) s.ntl[0] = total;
}

__device__ __forceinline__ void finish_iteration(const PcgState& s, bool still_active, bool was_active, bool flagged) {
    // grid-wide bookkeeping: count active columns; last CTA publishes and sets the graph condition.
    // One 64-bit arrival per CTA on the adjacent counters (n_active_next, done_ctas): low word +=
    // still-active, high word += 1 — the last arriver reads the total from the returned value.  Only a
    // CTA that also changed a live-tile counter or the status flag fences before arriving (release);
    // the last arriver fences after (acquire) before reading those.
    __shared__ int s_last, s_na;
    __syncthreads();
    if (threadIdx.x == 0) {
        const bool froze = was_active && !still_active && s.ntl;
        if (froze) atomicSub(&s.ntl_cnt[blockIdx.x / s.ntl_bn], 1);
        if (froze || flagged) __threadfence();
        const unsigned long long old = atomicAdd(reinterpret_cast<unsigned long long*>(s.n_active_next),
                                                 (1ull << 32) | (still_active ? 1ull : 0ull));
        s_last = (int)(old >> 32) == (int)gridDim.x - 1;
        s_na = (int)(old & 0xffffffffull) + (still_active ? 1 : 0);
        if (s_last) __threadfence();
    }
    __syncthreads();
    if (!s_last || threadIdx.x >= 32) return;
    const int na = s_na;
    publish_live_tiles(s, na);
    if (threadIdx.x == 0) {
        const int k = *s.kiter + 1;
        *s.kiter = k;
        *s.n_active = na;
        *s.n_active_next = 0;
        *s.done_ctas = 0;
        if (s.cond_handle) {
            cudaGraphSetConditional((cudaGraphConditionalHandle)s.cond_handle,
                                    (na > 0 && k < s.maxit && *(volatile int*)s.status == 0) ? 1u : 0u);
        }
    }
}

template <int LMAX, int G, int NG, int V>
__global__ void __launch_bounds__(32 * G * NG, (32 * G * NG) <= 256 ? (V == 2 ? 3 : 2) : 1) k_pcg_init(PcgState s, PoleGeom g, PoleTabs t,
                                                          const double* __restrict__ b, int ldb) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[64];
    __shared__ int s_init_last, s_act;
    const int c = blockIdx.x;
    const int n = g.n, npad = g.T * g.LL;
    pdl_trigger();
    Smem S = carve_v<V>(sm, g, t);
    const size_t off = (size_t)c * s.ldv;
    const int param = clamp_param(s.col_param[c], t.n_param);
    stage_tables(t, g, param, S.scratch);
    pdl_wait_prior();
    for (int i = threadIdx.x; i < npad; i += blockDim.x) {
        const double v = i < n ? b[(size_t)c * ldb + i] : 0.0;
        S.R[tpos(i, g)] = v;
        if (i < n) { s.r[off + i] = v; s.x[(size_t)c * s.ldx + i] = 0.0; }
    }
    __syncthreads();
    block_polesum<LMAX, G, NG, V>(t, g, param, S.R, S.Z, S.scratch);
    double rz = 0.0, zz = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double zi = S.Z[tpos(i, g)];
        rz += S.R[tpos(i, g)] * zi;
        zz += zi * zi;
        s.p[off + i] = zi;
        if (s.zs && (!s.zmixed || *s.zmixed)) {
            s.zs[(size_t)c * s.ldz + i] = s.gp[param] * zi;
            s.zs[(size_t)c * s.ldz + s.zhalf + i] = s.Kp[param] * zi;
        }
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
        s_act = act ? 1 : 0;
        if (c == 0 && s.hist) s.hist[0] = eta0;
        if (act) atomicAdd(s.n_active_next, 1);
        if (act && s.ntl) atomicAdd(&s.ntl_cnt[c / s.ntl_bn], 1);
        __threadfence();
        const int prev = atomicAdd(s.done_ctas, 1);
        s_init_last = prev == (int)gridDim.x - 1;
        if (s_init_last) __threadfence();
    }
    __syncthreads();
    if (s.xh && !s_act)                          // frozen at k = 0: x = 0 is final
        for (int i = threadIdx.x; i < n; i += blockDim.x) s.xh[(size_t)c * n + i] = 0.0;
    if (s_init_last && threadIdx.x < 32) {
        int na = 0;
        if (threadIdx.x == 0) na = atomicAdd(s.n_active_next, 0);
        na = __shfl_sync(0xffffffffu, na, 0);
        publish_live_tiles(s, na);
        if (threadIdx.x == 0) {
            *s.n_active = na;
            *s.n_active_next = 0;
            *s.done_ctas = 0;
            *s.kiter = 0;
        }
    }
}

// rows of thread tid: ρ = tid + j NT, j < RPT (coalesced); RPT = ceil(T LL / NT) <= ceil(LMAX / NG)
template <int LMAX, int G, int NG, int V>
__global__ void __launch_bounds__(32 * G * NG, (32 * G * NG) <= 256 ? (V == 2 ? 3 : 2) : 1) k_pcg_iter(PcgState s, PoleGeom g, PoleTabs t) {
    constexpr int NT = 32 * G * NG;
    constexpr int RPT = (LMAX + NG - 1) / NG;
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[64];
    const int c = blockIdx.x;
    const int n = g.n;
    Smem S = carve_v<V>(sm, g, t);
    const size_t off = (size_t)c * s.ldv;
    const size_t offx = (size_t)c * s.ldx;
    pdl_trigger();
    if (s.dbg && threadIdx.x == 0) s.dbg[16 + 2 * c] = (long long)gtimer();
    // constant inputs (column parameter, pole tables) before the wait on the preceding GEMM
    const int param = clamp_param(s.col_param[c], t.n_param);
    stage_tables(t, g, param, S.scratch);
    // Inside the WHILE graph the previous iteration's kernels have all completed when this one
    // starts (iterations of the conditional body are serialised; only the GEMM before this kernel
    // overlaps it through PDL), so p, x, r, the active flag and the iteration counter are final:
    // the v2 kernels load them before waiting on the GEMM and only q after it.
    const bool early = V >= 1 && s.cond_handle != 0;
    double pv[RPT], qv[RPT], xv[RPT], rv[RPT];
    int work = 0, k = 0;
    double rho_c = 0.0, eta0_c = 0.0;            // the column's ρ and η0 (written by earlier kernels only)
    auto load_pxr = [&]() {
        work = __ldcg(&s.active[c]);
        k = __ldcg(s.kiter) + 1;
        rho_c = __ldcg(&s.rho[c]);
        eta0_c = __ldcg(&s.eta0[c]);
        if (work) {
#pragma unroll
            for (int j = 0; j < RPT; j++) {
                const int i = threadIdx.x + j * NT;
                const bool ok = i < n;
                pv[j] = ok ? __ldcg(&s.p[off + i]) : 0.0;
                xv[j] = ok ? __ldcg(&s.x[offx + i]) : 0.0;
                rv[j] = ok ? __ldcg(&s.r[off + i]) : 0.0;
            }
        }
    };
    if (early) load_pxr();
    pdl_wait_prior();
    if (!early) load_pxr();
    bool still = false;
    bool flagged = false;
    bool froze = false;                          // this launch ends the column: x is final
#define DD_PHASE(i) \
    if (s.dbg && blockIdx.x == 0 && threadIdx.x == 0) s.dbg[i] = clock64()
    DD_PHASE(0);
    if (!work) asm volatile("cp.async.wait_all;\n" ::);
    if (work) {
#pragma unroll
        for (int j = 0; j < RPT; j++) {
            const int i = threadIdx.x + j * NT;
            qv[j] = i < n ? (s.qadd ? s.q[off + i] + s.qadd[off + i] : s.q[off + i]) : 0.0;
        }
        double pq = 0.0, dummy = 0.0;
#pragma unroll
        for (int j = 0; j < RPT; j++) pq = fma(pv[j], qv[j], pq);
        block_sum2(pq, dummy, red);
        DD_PHASE(1);
        if (!(pq > 0.0)) {
            flagged = true;
            froze = true;
            if (threadIdx.x == 0) {
                atomicExch(s.status, (int)DD_ENOTSPD);
                s.active[c] = 0;
                s.iters[c] = k;
            }
        } else {
            const double alpha = rho_c / pq;
#pragma unroll
            for (int j = 0; j < RPT; j++) {
                const int i = threadIdx.x + j * NT;
                if (i < n) {
                    s.x[offx + i] = fma(alpha, pv[j], xv[j]);
                    const double ri = fma(-alpha, qv[j], rv[j]);
                    s.r[off + i] = ri;
                    S.R[tpos(i, g)] = ri;
                } else if (i < g.T * g.LL) {
                    S.R[tpos(i, g)] = 0.0;
                }
            }
            for (int i = threadIdx.x + RPT * NT; i < g.T * g.LL; i += NT) S.R[tpos(i, g)] = 0.0;
            __syncthreads();
            DD_PHASE(2);
            block_polesum<LMAX, G, NG, V>(t, g, param, S.R, S.Z, S.scratch, blockIdx.x == 0 ? s.dbg : nullptr);
            DD_PHASE(3);
            if constexpr (V == 2) {
                // compact layout: p re-read from L2 (not held across the pole sum), issued before
                // the dot products so the round trip overlaps the block reduction
#pragma unroll
                for (int j = 0; j < RPT; j++) {
                    const int i = threadIdx.x + j * NT;
                    pv[j] = i < n ? __ldcg(&s.p[off + i]) : 0.0;
                }
            }
            double rz = 0.0, zz = 0.0;
            double zv[RPT];
#pragma unroll
            for (int j = 0; j < RPT; j++) {
                const int i = threadIdx.x + j * NT;
                zv[j] = 0.0;
                if (i < n) {
                    const int ps = tpos(i, g);
                    zv[j] = S.Z[ps];
                    rz = fma(S.R[ps], zv[j], rz);
                    zz = fma(zv[j], zv[j], zz);
                }
            }
            block_sum2(rz, zz, red);
            const double eta = s.norm_kind == 0 ? sqrt(fmax(rz, 0.0)) : sqrt(zz);
            const bool notspd = rz < 0.0;
            flagged = notspd;
            const bool conv = eta <= s.rtol * eta0_c;
            if (threadIdx.x == 0) {
                s.iters[c] = k;
                s.relres[c] = eta / eta0_c;
                if (c == 0 && s.hist) s.hist[k] = eta;
                if (notspd) atomicExch(s.status, (int)DD_ENOTSPD);
            }
            if (conv || notspd || k >= s.maxit) {
                froze = true;
                if (threadIdx.x == 0) s.active[c] = 0;
            } else {
                const double beta = rz / rho_c;
                if constexpr (V == 0) {
                    // p as at entry, re-read (L2) rather than held in registers across the pole sum
                    // (the partitioned pole sum needs every register)
#pragma unroll
                    for (int j = 0; j < RPT; j++) {
                        const int i = threadIdx.x + j * NT;
                        pv[j] = i < n ? __ldcg(&s.p[off + i]) : 0.0;
                    }
                }
                if (s.zs && (!s.zmixed || *s.zmixed)) {
                    // assembled Schur apply: the next GEMM's operand [γ p ; K p] written with p
                    const double gc = s.gp[param], Kc = s.Kp[param];
                    double* zc = s.zs + (size_t)c * s.ldz;
#pragma unroll
                    for (int j = 0; j < RPT; j++) {
                        const int i = threadIdx.x + j * NT;
                        if (i < n) {
                            const double pn = fma(beta, pv[j], zv[j]);
                            s.p[off + i] = pn;
                            zc[i] = gc * pn;
                            zc[s.zhalf + i] = Kc * pn;
                        }
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < RPT; j++) {
                        const int i = threadIdx.x + j * NT;
                        if (i < n) s.p[off + i] = fma(beta, pv[j], zv[j]);   // pv: p as loaded at entry
                    }
                }
                __syncthreads();
                if (threadIdx.x == 0) s.rho[c] = rz;
                still = true;
            }
        }
    }
    if (froze && s.xh) {
        // each thread's own x entries (written above by this thread, or untouched on a p.q <= 0 stop)
#pragma unroll
        for (int j = 0; j < RPT; j++) {
            const int i = threadIdx.x + j * NT;
            if (i < n) s.xh[(size_t)c * n + i] = s.x[offx + i];
        }
    }
    DD_PHASE(4);
    finish_iteration(s, still, work != 0, flagged);
    DD_PHASE(5);
    if (s.dbg && threadIdx.x == 0) s.dbg[17 + 2 * c] = (long long)gtimer();
#undef DD_PHASE
}

// ---------------------------------------------------------------------------------------------
// Persistent whole-PCG kernel for small interfaces (n <= 63): one CTA per column
// keeps [S_dst | F], the vectors and the pole-sum state in shared memory and runs every PCG
// iteration in one launch — the Schur apply as two fixed-order matvecs (same operator as the
// GEMM path: q = S_dst (K s ∘ S_dst p) + γ F p), the pole sum and the updates as in k_pcg_iter.
template <int LMAX, int NG>
__global__ void __launch_bounds__(32 * NG) k_pcg_small(PcgState s, PoleGeom g, PoleTabs t, const double* __restrict__ b,
                                                       int ldb, const double* __restrict__ W, int lda, int Kpad,
                                                       const double* __restrict__ sw, const double* __restrict__ Kp,
                                                       const double* __restrict__ gp) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[64];
    const int c = blockIdx.x;
    const int n = g.n, npad = g.T * g.LL;
    const int ldw = 2 * Kpad;
    const int lws = ldw + 1;                           // smem row stride (odd: rows of a warp hit different banks)
    double* Ws = sm;                                   // n x 2Kpad
    double* pv = Ws + (((size_t)n * lws + 1) & ~(size_t)1);   // p, T, x, q : 64 each (16-byte aligned)
    double* Tv = pv + 64;
    double* xv = Tv + 64;
    double* Qv = xv + 64;
    double* psm = Qv + 64;
    Smem S = carve(psm, g);
    const int param = clamp_param(s.col_param[c], t.n_param);
    stage_tables(t, g, param, S.scratch);
    for (int idx = threadIdx.x; idx < n * ldw; idx += blockDim.x) Ws[(idx / ldw) * lws + idx % ldw] = W[(size_t)(idx / ldw) * lda + idx % ldw];
    // matvecs: TPR threads per row (blockDim / 32 for n <= 31, / 64 for n <= 63), each a strided share of the
    // row, combined by a fixed xor-shuffle tree within the row's lane group
    const int TPR = (int)blockDim.x / (n <= 31 ? 32 : 64);
    const int mrow = threadIdx.x / TPR, msub = threadIdx.x % TPR;
    const double Kc = Kp[param], gc = gp[param];
    for (int i = threadIdx.x; i < npad; i += blockDim.x) {
        const double v = i < n ? b[(size_t)c * ldb + i] : 0.0;
        S.R[tpos(i, g)] = v;
        if (i < 64) xv[i] = 0.0;
    }
    __syncthreads();
    block_polesum<LMAX, 1, NG>(t, g, param, S.R, S.Z, S.scratch);
    double rz = 0.0, zz = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double zi = S.Z[tpos(i, g)];
        rz += S.R[tpos(i, g)] * zi;
        zz += zi * zi;
        pv[i] = zi;
    }
    block_sum2(rz, zz, red);
    const double eta0 = s.norm_kind == 0 ? sqrt(fmax(rz, 0.0)) : sqrt(zz);
    double rho = rz;
    int k = 0;
    double rel = eta0 > 0.0 ? 1.0 : 0.0;
    if (threadIdx.x == 0 && c == 0 && s.hist) s.hist[0] = eta0;
    if (rz < 0.0 && threadIdx.x == 0) atomicExch(s.status, (int)DD_ENOTSPD);
    bool run = eta0 > 0.0 && rz >= 0.0;
    while (run && k < s.maxit) {
        k++;
        // q = S_dst (K s ∘ (S_dst p)) + γ F p
        {
            double a = 0.0;
            if (mrow < n) {
                const double* wr = Ws + (size_t)mrow * lws;
                for (int j = msub; j < n; j += TPR) a = fma(wr[j], pv[j], a);
            }
            for (int o = TPR / 2; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (mrow < n && msub == 0) Tv[mrow] = Kc * sw[mrow] * a;
        }
        __syncthreads();
        {
            double a = 0.0, f = 0.0;
            if (mrow < n) {
                const double* wr = Ws + (size_t)mrow * lws;
                for (int j = msub; j < n; j += TPR) {
                    a = fma(wr[j], Tv[j], a);
                    f = fma(wr[Kpad + j], pv[j], f);
                }
            }
            for (int o = TPR / 2; o > 0; o >>= 1) {
                a += __shfl_xor_sync(0xffffffffu, a, o);
                f += __shfl_xor_sync(0xffffffffu, f, o);
            }
            if (mrow < n && msub == 0) Qv[mrow] = fma(gc, f, a);
        }
        __syncthreads();
        // n <= 63 < blockDim: thread i owns row i
        double pq = 0.0, dummy = 0.0, qi = 0.0;
        const int i = threadIdx.x;
        if (i < n) {
            qi = Qv[i];
            pq = pv[i] * qi;
        }
        block_sum2(pq, dummy, red);
        if (!(pq > 0.0)) {
            if (threadIdx.x == 0) atomicExch(s.status, (int)DD_ENOTSPD);
            break;
        }
        const double alpha = rho / pq;
        if (i < n) {
            xv[i] = fma(alpha, pv[i], xv[i]);
            const int ps = tpos(i, g);
            S.R[ps] = fma(-alpha, qi, S.R[ps]);
        }
        __syncthreads();
        block_polesum<LMAX, 1, NG>(t, g, param, S.R, S.Z, S.scratch);
        rz = 0.0; zz = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const double zi = S.Z[tpos(i, g)];
            rz = fma(S.R[tpos(i, g)], zi, rz);
            zz = fma(zi, zi, zz);
        }
        block_sum2(rz, zz, red);
        const double eta = s.norm_kind == 0 ? sqrt(fmax(rz, 0.0)) : sqrt(zz);
        rel = eta / eta0;
        if (threadIdx.x == 0 && c == 0 && s.hist) s.hist[k] = eta;
        if (rz < 0.0) {
            if (threadIdx.x == 0) atomicExch(s.status, (int)DD_ENOTSPD);
            break;
        }
        if (eta <= s.rtol * eta0) break;
        const double beta = rz / rho;
        for (int i = threadIdx.x; i < n; i += blockDim.x) pv[i] = fma(beta, pv[i], S.Z[tpos(i, g)]);
        __syncthreads();
        rho = rz;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) s.x[(size_t)c * s.ldx + i] = xv[i];
    if (threadIdx.x == 0) {
        s.iters[c] = k;
        s.relres[c] = rel;
        s.eta0[c] = eta0;
        s.active[c] = 0;
        atomicMax(s.kiter, k);
    }
}

__global__ void k_copy_cols(int n, int ncols, const double* __restrict__ src, int lds, double* __restrict__ dst,
                            int ldd) {
    const size_t total = (size_t)n * ncols;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const size_t c = idx / n, i = idx % n;
        dst[c * ldd + i] = src[c * lds + i];
    }
}

__global__ void k_schur_operand(int n, int ncols, const int* __restrict__ col_param, int n_param,
                                const double* __restrict__ Kp, const double* __restrict__ gp,
                                const double* __restrict__ x, int ldx, double* __restrict__ Z, int ldz, int zhalf) {
    const size_t total = (size_t)n * ncols;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const size_t c = idx / n, i = idx % n;
        const int p = clamp_param(col_param[c], n_param);
        const double v = x[c * ldx + i];
        Z[c * ldz + i] = gp[p] * v;
        Z[c * ldz + zhalf + i] = Kp[p] * v;
    }
}

// Solve prologue in one launch (one CTA): zero the solve's counters and live-tile list, then
// flag out-of-range parameter ids (ints[5]) and, for the grouped Schur apply, 32-column tiles
// that hold two parameter sets (ints[6]).
__global__ void __launch_bounds__(1024) k_solve_prep(int ncols, const int* __restrict__ col_param, int n_param,
                                                     int* ints, int nzero, int* ntl, int ntl_len, int check_tiles) {
    for (int i = threadIdx.x; i < nzero; i += blockDim.x) ints[i] = 0;
    for (int i = threadIdx.x; i < ntl_len; i += blockDim.x) ntl[i] = 0;
    int bad = 0, mixed = 0;
    for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
        const int p = col_param[c];
        bad |= (p < 0 || p >= n_param) ? 1 : 0;
        if (check_tiles) mixed |= (p != col_param[c - c % GEMM_BN_GROUPED]) ? 1 : 0;
    }
    bad = __syncthreads_or(bad);        // also orders the zeroing above before the flag stores
    mixed = __syncthreads_or(mixed);
    if (threadIdx.x == 0) {
        if (bad) ints[5] = 1;
        if (mixed) ints[6] = 1;
    }
}

// Grouped Schur apply: does any 32-column tile hold two parameter sets?  (*mixed |= 1)
__global__ void k_check_tiles(int ncols, const int* __restrict__ col_param, int* mixed) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncols; c += gridDim.x * blockDim.x) {
        const int c0 = c - c % GEMM_BN_GROUPED;
        if (col_param[c] != col_param[c0]) atomicExch(mixed, 1);
    }
}

// H_p = K_p G + γ_p F for every parameter set p (rows of n, row stride ldh; padded entries 0)
__global__ void k_group_operators(int n, int n_param, const double* __restrict__ W, int lda, int f_off, int g_off,
                                  const double* __restrict__ Kp, const double* __restrict__ gp, double* __restrict__ H,
                                  int ldh, long long sH) {
    const size_t total = (size_t)n * ldh;
    for (int p = 0; p < n_param; p++) {
        const double K = Kp[p], g = gp[p];
        for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
            const size_t i = idx / ldh, k = idx % ldh;
            H[p * sH + idx] = k < (size_t)n ? fma(K, W[i * lda + g_off + k], g * W[i * lda + f_off + k]) : 0.0;
        }
    }
}

__global__ void k_check_params(int ncols, const int* col_param, int n_param, int* flag) {
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncols; c += gridDim.x * blockDim.x) {
        const int p = col_param[c];
        if (p < 0 || p >= n_param) atomicExch(flag, 1);
    }
}

// ---------------------------------------------------------------------------- host side
PoleGeom make_pole_geom(int n) {
    PoleGeom g{};
    g.n = n;
    // chunks of <= 16 rows per thread (short Thomas chains, <= 128 registers), widening the
    // group (G warps, PCR over 32 G separators) as n grows; chunks grow to 32 only past n = 4095
    int G = 1;
    while (32 * G * 16 < n + 1 && G < 8) G *= 2;
    g.G = G;
    g.T = 32 * G;
    g.J = 0;
    while ((1 << g.J) < g.T) g.J++;
    g.LL = (n + 1 + g.T - 1) / g.T;
    g.part = n / g.LL;
    g.Lr_part = n - g.part * g.LL;
    return g;
}

bool pole_geom_supported(const PoleGeom& g) { return g.LL <= 32; }

static int lmax_of(int L) {
    int m = 1;
    while (m < L) m *= 2;
    return m;
}

int polesum_groups(const PoleGeom& g) {
    if (g.G >= 8) return g.LL <= 16 ? 2 : 1;
    if (g.G == 4) return 2;
    if (g.G == 2) return 4;
    return 8;
}

int polesum_warps(const PoleGeom& g) { return g.G * polesum_groups(g); }

static size_t polesum_v2_doubles(const PoleGeom& g, int max_sys) {
    (void)g;
    return (size_t)V2_WSZ + (size_t)V2_REC * max_sys        // tables
           + 2 * (size_t)max_sys * (g.T + 1);               // hl, yf (phase B works in the hl rows)
}

size_t polesum_smem(const PoleGeom& g, int max_sys) {
    const int NG = polesum_groups(g);
    const size_t tot = (size_t)g.LL * (g.T + 1);
    size_t d = 2 * tot                          // R, Z
               + (size_t)max_sys * 4 * g.LL     // tables
               + 2 * (size_t)NG * g.T           // PCR exchange
               + (size_t)NG * tot;              // group partials
    if (polesum_v2_supported(g, max_sys)) d = std::max(d, 2 * tot + polesum_v2_doubles(g, max_sys));
    return d * sizeof(double);
}

// The compact merged-interior layout (V = 2, three CTAs per SM): 128-chunk geometry (G = 4,
// 256 threads), at least LL systems (Z fits in the yf rows), within a third of the SM's shared
// memory.  DD_POLE_COMPACT=0 keeps the two-CTA layout (V = 1).
bool polesum_compact(const PoleGeom& g, int max_sys) {
    static const bool off = std::getenv("DD_POLE_COMPACT") && std::getenv("DD_POLE_COMPACT")[0] == '0';
    if (off || g.G != 4 || polesum_groups(g) != 2 || max_sys < g.LL || !polesum_v2_supported(g, max_sys)) return false;
    return polesum_smem_v(g, max_sys, 2) <= 74 * 1024;
}

size_t polesum_smem_v(const PoleGeom& g, int max_sys, int v) {
    if (v != 2) return polesum_smem(g, max_sys);
    const size_t tot = (size_t)g.LL * (g.T + 1);
    return (tot + polesum_v2_doubles(g, max_sys)) * sizeof(double);
}

bool polesum_v2_supported(const PoleGeom& g, int max_sys) {
    if (g.LL != V2_L || g.n + 1 != g.T * g.LL || g.T < 32 || g.T > 256) return false;
    const int NT = 32 * polesum_warps(g);
    if (NT % g.T != 0 || V2_L % (NT / g.T) != 0) return false;
    const size_t tot = (size_t)g.LL * (g.T + 1);
    return (2 * tot + polesum_v2_doubles(g, max_sys)) * sizeof(double) <= 220 * 1024;
}

// Dynamic shared memory of a pole-sum kernel, with the full shared-memory carveout (the layouts
// are sized for 2 or 3 resident CTAs per SM); DD_OCC_PRINT=1 prints the resident CTAs per SM.
template <typename K>
static cudaError_t set_smem(K kern, size_t bytes, int threads = 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    static const bool occ_print = std::getenv("DD_OCC_PRINT") && std::getenv("DD_OCC_PRINT")[0] == '1';
    if (e == cudaSuccess && occ_print && threads > 0) {
        int nb = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, threads, bytes);
        fprintf(stderr, "[dd] pole-sum kernel: %d threads, %zu B smem, %d CTAs/SM\n", threads, bytes, nb);
    }
    return e;
}

// Instantiated shapes (LMAX, G, NG): n <= 1023 with G = 1, and LL = 32 chunks with G = 2, 4, 8.
// V: 1 = merged-interior pole sum (tables t.v2; 16-row chunks only), 0 = partitioned Thomas + PCR
#define DD_POLE_SWITCH_V(g, t, ...)                                                                \
    DD_POLE_SWITCH(g, {                                                                          \
        if constexpr (LM == V2_L) {                                                              \
            if ((t).v2 && GG == 4 && polesum_compact(g, (t).max_sys)) {                          \
                if constexpr (GG == 4) { constexpr int VV = 2; __VA_ARGS__; }                    \
            } else if ((t).v2) { constexpr int VV = 1; __VA_ARGS__; }                            \
            else { constexpr int VV = 0; __VA_ARGS__; }                                          \
        } else { constexpr int VV = 0; __VA_ARGS__; }                                            \
    })

#define DD_POLE_SWITCH(g, ...)                                                                   \
    do {                                                                                         \
        const int _lm = lmax_of((g).LL), _G = (g).G;                                             \
        if (_G == 1 && _lm == 1) { constexpr int LM = 1, GG = 1, NGG = 8; __VA_ARGS__; }         \
        else if (_G == 1 && _lm == 2) { constexpr int LM = 2, GG = 1, NGG = 8; __VA_ARGS__; }    \
        else if (_G == 1 && _lm == 4) { constexpr int LM = 4, GG = 1, NGG = 8; __VA_ARGS__; }    \
        else if (_G == 1 && _lm == 8) { constexpr int LM = 8, GG = 1, NGG = 8; __VA_ARGS__; }    \
        else if (_G == 1 && _lm == 16) { constexpr int LM = 16, GG = 1, NGG = 8; __VA_ARGS__; }  \
        else if (_G == 2) { constexpr int LM = 16, GG = 2, NGG = 4; __VA_ARGS__; }               \
        else if (_G == 4) { constexpr int LM = 16, GG = 4, NGG = 2; __VA_ARGS__; }               \
        else if (_lm <= 16) { constexpr int LM = 16, GG = 8, NGG = 2; __VA_ARGS__; }             \
        else { constexpr int LM = 32, GG = 8, NGG = 1; __VA_ARGS__; }                            \
    } while (0)

cudaError_t launch_pcg_init(const PcgState& s, const PoleGeom& g, const PoleTabs& t, const double* b, int ldb,
                            cudaStream_t st) {
    if (s.ncols <= 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    DD_POLE_SWITCH_V(g, t, {
        const size_t smem = polesum_smem_v(g, t.max_sys, VV);
        e = set_smem(k_pcg_init<LM, GG, NGG, VV>, smem, 32 * GG * NGG);
        if (e == cudaSuccess) k_pcg_init<LM, GG, NGG, VV><<<s.ncols, 32 * GG * NGG, smem, st>>>(s, g, t, b, ldb);
    });
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_pcg_iter(const PcgState& s, const PoleGeom& g, const PoleTabs& t, cudaStream_t st, bool pdl) {
    if (s.ncols <= 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    DD_POLE_SWITCH_V(g, t, {
        const size_t smem = polesum_smem_v(g, t.max_sys, VV);
        e = set_smem(k_pcg_iter<LM, GG, NGG, VV>, smem, 32 * GG * NGG);
        if (e == cudaSuccess) e = launch_ex(k_pcg_iter<LM, GG, NGG, VV>, s.ncols, 32 * GG * NGG, smem, st, pdl, s, g, t);
    });
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_precond(int ncols, const int* col_param, const PoleGeom& g, const PoleTabs& t, const double* r,
                           int ldr, double* z, int ldz, cudaStream_t st, bool pdl) {
    if (ncols <= 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    DD_POLE_SWITCH_V(g, t, {
        const size_t smem = polesum_smem_v(g, t.max_sys, VV);
        e = set_smem(k_precond<LM, GG, NGG, VV>, smem, 32 * GG * NGG);
        if (e == cudaSuccess) e = launch_ex(k_precond<LM, GG, NGG, VV>, ncols, 32 * GG * NGG, smem, st, pdl, ncols, col_param, g, t, r, ldr, z, ldz);
    });
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_frac_ra(int ncols, const int* col_param, int n_param, const double* gp, const PoleGeom& g,
                           const PoleTabs& t, const double* x, int ldx, double* u, int ldu, double h6, cudaStream_t st,
                           bool pdl) {
    if (ncols <= 0) return cudaSuccess;
    cudaError_t e = cudaSuccess;
    DD_POLE_SWITCH_V(g, t, {
        const size_t smem = polesum_smem_v(g, t.max_sys, VV);
        e = set_smem(k_frac_ra<LM, GG, NGG, VV>, smem, 32 * GG * NGG);
        if (e == cudaSuccess)
            e = launch_ex(k_frac_ra<LM, GG, NGG, VV>, ncols, 32 * GG * NGG, smem, st, pdl, ncols, col_param, n_param, gp, g, t,
                          x, ldx, u, ldu, h6);
    });
    return e != cudaSuccess ? e : cudaGetLastError();
}

bool pcg_small_supported(int n) { return n <= 63; }

cudaError_t launch_pcg_small(const PcgState& s, const PoleGeom& g, const PoleTabs& t, const double* b, int ldb,
                             const double* W, int lda, int Kpad, const double* sw, const double* Kp, const double* gp,
                             cudaStream_t st) {
    if (s.ncols <= 0) return cudaSuccess;
    if (!pcg_small_supported(g.n) || g.G != 1) return cudaErrorInvalidValue;
    const size_t smem = ((size_t)g.n * (2 * Kpad + 1) + 1 + 256) * sizeof(double) + polesum_smem(g, t.max_sys);
    cudaError_t e = cudaSuccess;
    switch (lmax_of(g.LL)) {
        case 1: {
            e = set_smem(k_pcg_small<1, 8>, smem);
            if (e == cudaSuccess) k_pcg_small<1, 8><<<s.ncols, 256, smem, st>>>(s, g, t, b, ldb, W, lda, Kpad, sw, Kp, gp);
        } break;
        default: {
            e = set_smem(k_pcg_small<2, 8>, smem);
            if (e == cudaSuccess) k_pcg_small<2, 8><<<s.ncols, 256, smem, st>>>(s, g, t, b, ldb, W, lda, Kpad, sw, Kp, gp);
        } break;
    }
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

cudaError_t launch_schur_operand(int n, int ncols, const int* col_param, int n_param, const double* Kp,
                                 const double* gp, const double* x, int ldx, double* Z, int ldz, int zhalf,
                                 cudaStream_t st) {
    if (n <= 0 || ncols <= 0) return cudaSuccess;
    const size_t total = (size_t)n * ncols;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    k_schur_operand<<<blocks, 256, 0, st>>>(n, ncols, col_param, n_param, Kp, gp, x, ldx, Z, ldz, zhalf);
    return cudaGetLastError();
}

cudaError_t launch_solve_prep(int ncols, const int* col_param, int n_param, int* ints, int nzero, int* ntl,
                              int ntl_len, bool check_tiles, cudaStream_t st) {
    k_solve_prep<<<1, 1024, 0, st>>>(ncols, col_param, n_param, ints, nzero, ntl, ntl_len, check_tiles ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_check_tiles(int ncols, const int* col_param, int* mixed, cudaStream_t st) {
    if (ncols <= 0) return cudaSuccess;
    k_check_tiles<<<(ncols + 255) / 256, 256, 0, st>>>(ncols, col_param, mixed);
    return cudaGetLastError();
}

cudaError_t launch_group_operators(int n, int n_param, const double* W, int lda, int f_off, int g_off, const double* Kp,
                                   const double* gp, double* H, int ldh, long long sH, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_group_operators<<<148 * 8, 256, 0, st>>>(n, n_param, W, lda, f_off, g_off, Kp, gp, H, ldh, sH);
    return cudaGetLastError();
}

cudaError_t launch_check_params(int ncols, const int* col_param, int n_param, int* flag, cudaStream_t st) {
    if (ncols <= 0) return cudaSuccess;
    k_check_params<<<(ncols + 255) / 256, 256, 0, st>>>(ncols, col_param, n_param, flag);
    return cudaGetLastError();
}

}  // namespace dd
