// libdd, 3D interfaces (Γ = face {x = 0} of the unit cube; BASELINE.json config 4).
// Setup: sine matrix, Schur weights, the dense fractional term
// F = (M U) Λ^{-1/2} (M U)^T of the consistent P1 face pair from a generalised eigensolve
// (cuSOLVER Dsygvd — setup only, Eq.(7)), pole systems and their sine-diagonal
// preconditioners, and (pole split) the NCCL communicator.  Applies: see face3d.cu.
#include <cusolverDn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "dd_ctx.h"

namespace dd {

static const long double PI_L = 3.141592653589793238462643383279502884L;

#define SK(expr)                                                                                          \
    do {                                                                                                  \
        cusolverStatus_t _s = (expr);                                                                     \
        if (_s != CUSOLVER_STATUS_SUCCESS) return set_error(DD_ECUDA, std::string(#expr) + " failed");    \
    } while (0)
#define NK(expr)                                                                                                  \
    do {                                                                                                          \
        ncclResult_t _r = (expr);                                                                                 \
        if (_r != ncclSuccess) return set_error(DD_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(_r));   \
    } while (0)

// Chebyshev semi-iteration tables for systems a A + b M of the face pair (reading A12'):
// preconditioned by P = T_{a α + b m̃} (the sine-diagonal part), every eigenvalue of P^-1 (a A + b M)
// lies in 1 ± δ with δ = sup_θ |b (m - m̃)| / (a α + b m̃) — a bound on the Rayleigh quotient of
// these two-level Toeplitz matrices by the ratio of their stencil symbols
//   α = 4 - 2c1 - 2c2,  m = (h²/12)(6 + 2c1 + 2c2 + 2cos(θ1 + θ2)),  m̃ = (h²/12)(6 + 2c1 + 2c2 + 2c1c2)
// (m - m̃ = -(h²/6) s1 s2; for a = 0 the sup is (√3 - 1)/2).  δ from a 1024² grid of θ in [0, π]²,
// widened by 2 %; step count K = ceil(ln(2 √κ / ε) / ln(1/q)), q = (√κ - 1)/(√κ + 1),
// κ = (1 + δ)/(1 - δ): an energy-norm reduction of ε; coefficients of x += d, r -= A d,
// d = c1[k] d + c2[k] P^-1 r (centre 1, half-width δ).
static void build_cheb(const std::vector<std::pair<double, double>>& ab, long double hh12, double eps,
                       std::vector<double>& c1, std::vector<double>& c2, std::vector<int>& K, int& kmax_all) {
    const int ns = std::max(1, (int)ab.size());
    c1.assign((size_t)ns * CHEB_KMAX, 0.0);
    c2.assign((size_t)ns * CHEB_KMAX, 0.0);
    K.assign(ns, 0);
    kmax_all = 0;
    const int G = 1024;
    std::vector<long double> cs(G + 1), sn(G + 1);
    for (int i = 0; i <= G; i++) {
        const long double t = 3.141592653589793238462643383279502884L * i / G;
        cs[i] = cosl(t);
        sn[i] = sinl(t);
    }
    for (size_t k = 0; k < ab.size(); k++) {
        const long double a = ab[k].first, b = ab[k].second;
        long double dmax = 0.0L;
        for (int i = 0; i <= G; i++)
            for (int j = 0; j <= G; j++) {
                const long double den = a * (4.0L - 2.0L * cs[i] - 2.0L * cs[j]) +
                                        b * hh12 * (6.0L + 2.0L * cs[i] + 2.0L * cs[j] + 2.0L * cs[i] * cs[j]);
                if (den <= 0.0L) continue;
                const long double v = 2.0L * b * hh12 * sn[i] * sn[j] / den;
                if (v > dmax) dmax = v;
            }
        const long double d = std::min(0.999L, dmax * 1.02L);
        int steps = 1;
        if (d > 1e-300L) {
            const long double kap = (1.0L + d) / (1.0L - d), sq = sqrtl(kap);
            const long double qf = (sq - 1.0L) / (sq + 1.0L);
            steps = qf > 0.0L ? (int)ceill(logl(2.0L * sq / (long double)eps) / logl(1.0L / qf)) : 1;
        }
        steps = std::max(1, std::min(CHEB_KMAX, steps));
        K[k] = steps;
        kmax_all = std::max(kmax_all, steps);
        // ρ_0 = 1/σ = δ (θ = 1), ρ_{j+1} = 1/(2σ - ρ_j); c1 = ρ_{j+1} ρ_j, c2 = 2 ρ_{j+1}/δ
        const long double dd = std::max(d, 1e-300L), sig = 1.0L / dd;
        long double rho = dd;
        for (int j = 0; j < steps; j++) {
            const long double rn = 1.0L / (2.0L * sig - rho);
            c1[k * CHEB_KMAX + j] = (double)(rn * rho);
            c2[k * CHEB_KMAX + j] = (double)(2.0L * rn / dd);
            rho = rn;
        }
    }
}

dd_status setup_3d(dd_ctx* c, const double* K, const double* mu_inv, const double* poles, const double* residues,
                   const double* c0, const dd_dist* dist) {
    Face3& f = c->f3;
    const int N = c->N, n = c->n;
    if (c->n_param != 1) return set_error(DD_EUNSUPPORTED, "3D handles take one parameter set");
    f.n = n;
    f.n2 = n * n;
    f.ldf = round_up(n, 16);
    f.NP = (long long)f.ldf * f.ldf;
    const long double h = 1.0L / N;
    const double hh12 = (double)(h * h / 12.0L);
    const int Srows = std::max(round_up(n, 64), f.ldf);
    const size_t slack = (size_t)64 * f.ldf;   // slab GEMM tiles may read up to 64 rows past a slab

    // --- sine matrix and Schur weights s_ab = h(1 + (σ_a+σ_b)/2 - Σ_m (2/N) sin^2(mπ/N)/(σ_m+σ_a+σ_b))
    std::vector<long double> sintab(2 * N), sig(n);
    for (int a = 0; a < 2 * N; a++) sintab[a] = sinl(PI_L * a / N);
    for (int a = 1; a <= n; a++) {
        const long double sh = sinl(PI_L * a / (2.0L * N));
        sig[a - 1] = 4.0L * sh * sh;
    }
    const long double sc = sqrtl(2.0L / N);
    std::vector<double> Sh((size_t)Srows * f.ldf, 0.0), swh(f.NP, 0.0);
    for (int q = 1; q <= n; q++)
        for (int r = 1; r <= n; r++) Sh[(size_t)(q - 1) * f.ldf + (r - 1)] = (double)(sc * sintab[((long long)q * r) % (2 * N)]);
    for (int a = 0; a < n; a++)
        for (int b = 0; b < n; b++) {
            long double g = 0.0L;
            for (int m = 0; m < n; m++) {
                const long double s1 = sintab[m + 1];
                g += (2.0L / N) * s1 * s1 / (sig[m] + sig[a] + sig[b]);
            }
            swh[(size_t)a * f.ldf + b] = (double)(h * (1.0L + 0.5L * (sig[a] + sig[b]) - g));
        }
    DD_CK(dalloc(c, &f.S, Sh.size()));
    DD_CK(cudaMemcpyAsync(f.S, Sh.data(), Sh.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    DD_CK(dalloc(c, &f.sw, (size_t)f.NP));
    DD_CK(cudaMemcpyAsync(f.sw, swh.data(), swh.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));

    // parity order of the sine index (dd_ctx.h: Face3::Sp): 0-based a = 0, 2, 4, .. then 1, 3, ..
    std::vector<int> perm, ipos(n);
    for (int a = 0; a < n; a += 2) perm.push_back(a);
    const int ne = (int)perm.size();
    for (int a = 1; a < n; a += 2) perm.push_back(a);
    for (int i = 0; i < n; i++) ipos[perm[i]] = i;
    {
        const char* nk = std::getenv("DD_NO_KPAR");
        f.kpar = (ne % 64 == 0 && ne < f.ldf && !(nk && nk[0] == '1')) ? ne : 0;
        std::vector<double> Sp((size_t)Srows * f.ldf, 0.0), SpT((size_t)Srows * f.ldf, 0.0);
        for (int i = 0; i < n; i++)
            for (int col = 0; col < n; col++) {
                Sp[(size_t)i * f.ldf + col] = Sh[(size_t)perm[i] * f.ldf + col];
                SpT[(size_t)col * f.ldf + i] = Sh[(size_t)perm[i] * f.ldf + col];
            }
        DD_CK(dalloc(c, &f.Sp, Sp.size()));
        DD_CK(dalloc(c, &f.SpT, SpT.size()));
        DD_CK(cudaMemcpyAsync(f.Sp, Sp.data(), Sp.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        DD_CK(cudaMemcpyAsync(f.SpT, SpT.data(), SpT.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        DD_CK(cudaStreamSynchronize(c->stream));
    }

    // --- dense fractional term via the generalised eigenproblem A_Γ U = M_Γ U Λ, U^T M U = I
    //     (RA mode, Remark 1: no dense F and no eigensolve; the interval only steers the pole split)
    if (c->frac_mode != DD_FRAC_DENSE) {
        f.lam_min = (double)(2.0L * PI_L * PI_L);
        f.lam_max = (double)(25.85L / (h * h));
    } else {
        const int n2 = f.n2;
        const int kp = round_up(n2, 16);
        const size_t big = (size_t)round_up(n2, 64) * kp + 1024;
        double *dA = nullptr, *dM = nullptr, *dW = nullptr, *work = nullptr;
        int* info = nullptr;
        DD_CK(cudaMalloc(&dA, big * sizeof(double)));
        DD_CK(cudaMalloc(&dM, big * sizeof(double)));
        DD_CK(cudaMalloc(&dW, (size_t)n2 * sizeof(double)));
        DD_CK(cudaMalloc(&info, sizeof(int)));
        DD_CK(cudaMemsetAsync(dA, 0, big * sizeof(double), c->stream));
        DD_CK(cudaMemsetAsync(dM, 0, big * sizeof(double), c->stream));
        DD_CK(face_dense_pair(n, hh12, dA, dM, c->stream));
        cusolverDnHandle_t hs = nullptr;
        SK(cusolverDnCreate(&hs));
        SK(cusolverDnSetStream(hs, c->stream));
        int lwork = 0;
        SK(cusolverDnDsygvd_bufferSize(hs, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n2, dA,
                                       n2, dM, n2, dW, &lwork));
        DD_CK(cudaMalloc(&work, (size_t)lwork * sizeof(double)));
        SK(cusolverDnDsygvd(hs, CUSOLVER_EIG_TYPE_1, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, n2, dA, n2, dM, n2,
                            dW, work, lwork, info));
        int hinfo = 0;
        std::vector<double> lam(n2);
        DD_CK(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        DD_CK(cudaMemcpyAsync(lam.data(), dW, n2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        DD_CK(cudaStreamSynchronize(c->stream));
        cusolverDnDestroy(hs);
        cudaFree(work);
        if (hinfo != 0) return set_error(DD_ECUDA, "cusolverDnDsygvd info != 0");
        f.lam_min = lam.front();
        f.lam_max = lam.back();
        std::vector<double> w4(n2);
        // F = (M U)(Λ + σ)^t (M U)^T = B B^T with B = M U (Λ + σ)^{t/2}  (Eq.(7); dd_frac)
        for (int j = 0; j < n2; j++)
            w4[j] = (double)powl((long double)lam[j] + (long double)c->frac_sigma, 0.5L * (long double)c->frac_t);
        DD_CK(cudaMemcpyAsync(dW, w4.data(), n2 * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        // B = M U Λ^{-1/4} (column-major in dM), then row-major in dA; F = B B^T into the padded layout
        DD_CK(face_mass_cols(n, hh12, dA, dM, n2, n2, c->stream));
        DD_CK(cudaMemsetAsync(dA, 0, big * sizeof(double), c->stream));
        DD_CK(scale_transpose(dM, dW, n2, dA, kp, c->stream));
        const size_t frows = (size_t)round_up((int)f.NP, 256);
        // row-sharded F under a multi-rank pole split (SURVEY §8(e) option): rank ρ keeps rows
        // [r0(ρ), r0(ρ+1)) in whole 256-row tiles of the F stream; DD_FX_ROWSHARD=0 keeps all rows
        const char* rsh = std::getenv("DD_FX_ROWSHARD");
        const bool shardF = dist && dist->world > 1 && dist->mode == DD_SHARD_POLES && !(rsh && rsh[0] == '0');
        // otherwise the packed-symmetric F (row a-3: upper blocks only, half the bytes and half the
        // memory; config 4: 214 + 24 µs per apply vs 386 µs for the full-F stream);
        // DD_FX_PACKED=0 keeps the full row-major F
        const char* fp = std::getenv("DD_FX_PACKED");
        const bool packed = !shardF && fx_sym_supported(f.NP) && !(fp && fp[0] == '0');
        // fold the interior solve into the dense operator: rows pad(j) of F <- γ F + K S_unit e_j
        // (one parameter set per 3D handle; S_unit applied to the identity columns by the same slab
        // passes the per-apply path runs; symmetric), DD_FX_FOLD=0 keeps the per-apply transforms
        const char* fo = std::getenv("DD_FX_FOLD");
        const bool fold = !(fo && fo[0] == '0');
        auto fold_into = [&](double* Fd) -> dd_status {
            const int BC = 256;
            const size_t len = (size_t)BC * f.NP + (size_t)64 * f.ldf;   // slab passes read up to 64 rows past a slab
            struct Bufs {                                                 // freed on every exit path
                double *X = nullptr, *Y1 = nullptr, *Y2 = nullptr, *Kc = nullptr;
                ~Bufs() { cudaFree(X); cudaFree(Y1); cudaFree(Y2); cudaFree(Kc); }
            } b;
            DD_CK(cudaMalloc(&b.X, len * sizeof(double)));
            DD_CK(cudaMalloc(&b.Y1, len * sizeof(double)));
            DD_CK(cudaMalloc(&b.Y2, len * sizeof(double)));
            DD_CK(cudaMalloc(&b.Kc, BC * sizeof(double)));
            DD_CK(cudaMemsetAsync(b.Y1, 0, len * sizeof(double), c->stream));
            DD_CK(cudaMemsetAsync(b.Y2, 0, len * sizeof(double), c->stream));
            DD_CK(cudaMemsetAsync(b.X, 0, len * sizeof(double), c->stream));
            const std::vector<double> kh(BC, K[0]);
            DD_CK(cudaMemcpyAsync(b.Kc, kh.data(), BC * sizeof(double), cudaMemcpyHostToDevice, c->stream));
            for (int j0 = 0; j0 < n2; j0 += BC) {
                const int nb = std::min(BC, n2 - j0);
                DD_CK(face_identity_cols(n, f.ldf, f.NP, j0, nb, b.X, c->stream));
                DD_CK(face_slab_pass(b.X, b.Y1, nb, n, f.ldf, f.S, c->stream));
                DD_CK(face_slab_pass_scaled(b.Y1, b.Y2, nb, n, f.ldf, f.S, f.sw, 0, 1, b.Kc, c->stream));
                DD_CK(face_slab_pass(b.Y2, b.Y1, nb, n, f.ldf, f.S, c->stream));
                DD_CK(face_slab_pass(b.Y1, b.Y2, nb, n, f.ldf, f.S, c->stream));
                DD_CK(face_fold_rows(Fd, f.NP, n, f.ldf, j0, nb, mu_inv[0], b.Y2, c->stream));
            }
            DD_CK(cudaStreamSynchronize(c->stream));   // kh and the buffers outlive the queued work
            return DD_OK;
        };
        // B̃ = T B column by column: eigen columns of B (row-major n2 x kp in Bd) gathered into padded
        // face vectors, two slab passes with Sp, scattered back
        auto transform_columns = [&](double* Bd, int n2c, int ldb) -> dd_status {
            const int BC = 256;
            const size_t len = (size_t)BC * f.NP + (size_t)64 * f.ldf;
            struct Bufs {
                double *X = nullptr, *Y = nullptr;
                ~Bufs() { cudaFree(X); cudaFree(Y); }
            } b;
            DD_CK(cudaMalloc(&b.X, len * sizeof(double)));
            DD_CK(cudaMalloc(&b.Y, len * sizeof(double)));
            DD_CK(cudaMemsetAsync(b.X, 0, len * sizeof(double), c->stream));
            DD_CK(cudaMemsetAsync(b.Y, 0, len * sizeof(double), c->stream));
            for (int j0 = 0; j0 < n2c; j0 += BC) {
                const int nb = std::min(BC, n2c - j0);
                DD_CK(face_gather_cols(Bd, n2c, ldb, j0, nb, n, f.ldf, f.NP, b.X, c->stream));
                DD_CK(face_slab_pass(b.X, b.Y, nb, n, f.ldf, f.Sp, c->stream));
                DD_CK(face_slab_pass(b.Y, b.X, nb, n, f.ldf, f.Sp, c->stream));
                DD_CK(face_scatter_cols(b.X, n2c, ldb, j0, nb, n, f.ldf, f.NP, Bd, c->stream));
            }
            DD_CK(cudaStreamSynchronize(c->stream));
            return DD_OK;
        };
        {   // Schur weights in the parity-ordered sine domain: the diagonal of T S_unit T^T
            std::vector<double> swp(f.NP, 0.0);
            for (int a2 = 0; a2 < n; a2++)
                for (int b2 = 0; b2 < n; b2++) swp[(size_t)ipos[a2] * f.ldf + ipos[b2]] = swh[(size_t)a2 * f.ldf + b2];
            DD_CK(dalloc(c, &f.sw_hat, (size_t)f.NP));
            DD_CK(cudaMemcpyAsync(f.sw_hat, swp.data(), swp.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
            DD_CK(cudaStreamSynchronize(c->stream));
        }
        double* Ffull = nullptr;
        f.fx_r0 = 0;
        f.fx_r1 = (int)f.NP;
        if (packed || shardF) {
            DD_CK(cudaMalloc(&Ffull, frows * (size_t)f.NP * sizeof(double)));
            DD_CK(cudaMemsetAsync(Ffull, 0, frows * (size_t)f.NP * sizeof(double), c->stream));
        } else {
            DD_CK(dalloc(c, &f.F, frows * (size_t)f.NP));
            Ffull = f.F;
        }
        DD_CK(face_gram_scatter(dA, n2, kp, Ffull, n, f.ldf, f.NP, c->num_sms, c->stream));
        if (shardF) {
            const int W = dist->world, ntile = (int)((f.NP + 255) / 256);
            std::vector<int> r0s(W + 1);
            for (int q = 0; q <= W; q++) r0s[q] = std::min((int)f.NP, (int)((long long)q * ntile / W) * 256);
            f.fx_r0 = r0s[dist->rank];
            f.fx_r1 = r0s[dist->rank + 1];
            for (int q = 0; q < W; q++) f.fx_rows_max = std::max(f.fx_rows_max, r0s[q + 1] - r0s[q]);
            const size_t rows = (size_t)std::max(1, f.fx_r1 - f.fx_r0);
            DD_CK(dalloc(c, &f.F, (size_t)round_up((int)rows, 256) * (size_t)f.NP));
            DD_CK(cudaMemcpyAsync(f.F, Ffull + (size_t)f.fx_r0 * f.NP, (size_t)(f.fx_r1 - f.fx_r0) * f.NP * sizeof(double),
                                  cudaMemcpyDeviceToDevice, c->stream));
            if (fold) {                    // the Schur apply streams this rank's rows of H; F rows stay for bulk
                dd_status fs = fold_into(Ffull);
                if (fs != DD_OK) return fs;
                DD_CK(dalloc(c, &f.Hrows, (size_t)round_up((int)rows, 256) * (size_t)f.NP));
                DD_CK(cudaMemcpyAsync(f.Hrows, Ffull + (size_t)f.fx_r0 * f.NP,
                                      (size_t)(f.fx_r1 - f.fx_r0) * f.NP * sizeof(double), cudaMemcpyDeviceToDevice,
                                      c->stream));
            }
            DD_CK(dalloc(c, &f.fx_r0s, (size_t)W + 1));
            DD_CK(cudaMemcpyAsync(f.fx_r0s, r0s.data(), sizeof(int) * (W + 1), cudaMemcpyHostToDevice, c->stream));
            DD_CK(dalloc(c, &f.fx_send, (size_t)c->max_cols * f.fx_rows_max));
            DD_CK(dalloc(c, &f.fx_recv, (size_t)W * c->max_cols * f.fx_rows_max));
            DD_CK(cudaStreamSynchronize(c->stream));
            cudaFree(Ffull);
            Ffull = nullptr;
        }
        if (packed) {
            // F is symmetric (B B^T): keep the upper 128 x 128 blocks only (row a-3, half the bytes)
            std::vector<int> ij;
            fx_sym_block_table(f.NP, ij);
            DD_CK(dalloc(c, &f.fblk, ij.size()));
            DD_CK(cudaMemcpyAsync(f.fblk, ij.data(), ij.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
            DD_CK(dalloc(c, &f.Fp, fx_sym_packed_doubles(f.NP)));
            DD_CK(fx_sym_pack(Ffull, f.NP, f.fblk, f.Fp, c->stream));
            DD_CK(dalloc(c, &f.fxD, fx_sym_partial_doubles(f.NP, c->max_cols)));
            DD_CK(dalloc(c, &f.fxT, fx_sym_partial_doubles(f.NP, c->max_cols)));
            if (fold) {
                // the PCG runs in the parity-ordered sine domain (T = Sp ⊗ Sp, orthogonal): there
                // K S_unit is the diagonal K s (permuted) and γ F is B̃ B̃^T with B̃ = T B, so
                // H̃ = T (γ F + K S_unit) T^T = γ B̃ B̃^T + K diag(s_perm) — the columns of B are
                // transformed by the slab passes, the Gram product reruns, the diagonal is added
                dd_status fs = transform_columns(dA, n2, kp);
                if (fs != DD_OK) return fs;
                DD_CK(cudaMemsetAsync(Ffull, 0, frows * (size_t)f.NP * sizeof(double), c->stream));
                DD_CK(face_gram_scatter(dA, n2, kp, Ffull, n, f.ldf, f.NP, c->num_sms, c->stream));
                DD_CK(face_hat_diag(Ffull, f.NP, n, f.ldf, mu_inv[0], K[0], f.sw_hat, c->stream));
                // the face pencil keeps the parity classes c(a,b) = par(a) xor par(b) of the sine modes
                // (A is sine-diagonal, M - M̃ couples opposite parities in both indices), so H̃ is
                // block-diagonal in them: at ldf = 128 each 64-row half of a 128 x 128 block has one
                // nonzero 64-column quadrant (the others are rounding, ~1e-15 relative: dropped)
                const char* csenv = std::getenv("DD_FX_CLASS_SPARSE");
                f.hat_cs = cheb_fused_ok(n, f.ldf) && !(csenv && csenv[0] == '0');
                DD_CK(dalloc(c, &f.Hp, fx_sym_packed_doubles(f.NP, f.hat_cs)));
                DD_CK(fx_sym_pack(Ffull, f.NP, f.fblk, f.Hp, c->stream, f.hat_cs));
                f.hat = true;
            }
        }
        DD_CK(cudaStreamSynchronize(c->stream));
        if (packed) cudaFree(Ffull);
        cudaFree(dA); cudaFree(dM); cudaFree(dW); cudaFree(info);
    }

    // --- pole systems: [M term if c0 != 0] + [poles with non-zero residue];  (a, b, w): a A + b M
    struct Sys { double a, b, w, cost; };
    std::vector<Sys> sys;
    // cost: the inner CG is preconditioned by the sine-diagonal part of each system (κ <= 3 for
    // every shift, ~20 iterations whatever the pole) and batched over (system, column) pairs, so a
    // rank's share of the pole sum costs in proportion to the NUMBER of its systems — not √κ of
    // the unpreconditioned system (which would put 1 system on most ranks and 5-6 on the rest)
    if (c0[0] != 0.0) sys.push_back({0.0, 1.0, c0[0], 1.0});
    for (int k = 0; k < c->n_poles; k++) {
        const double p = poles[k], r = residues[k];
        if (r == 0.0) continue;
        sys.push_back({1.0, -p, r, 1.0});
    }
    f.nsys_total = (int)sys.size();
    f.rank = dist ? dist->rank : 0;
    f.world = dist ? dist->world : 1;
    std::vector<int> mine;
    if (f.world > 1 && dist->mode == DD_SHARD_POLES) {
        // balanced by predicted inner-CG cost (longest-processing-time greedy):
        // equal costs give contiguous-by-order round robin, e.g. 21 systems on 8 ranks -> 3,3,3,3,3,2,2,2
        std::vector<int> order(sys.size());
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return sys[x].cost > sys[y].cost; });
        std::vector<double> load(f.world, 0.0);
        std::vector<int> owner(sys.size(), 0);
        for (int i : order) {
            int r = 0;
            for (int q = 1; q < f.world; q++)
                if (load[q] < load[r]) r = q;
            owner[i] = r;
            load[r] += sys[i].cost;
        }
        for (int i = 0; i < (int)sys.size(); i++)
            if (owner[i] == f.rank) mine.push_back(i);
    } else {
        for (int i = 0; i < (int)sys.size(); i++) mine.push_back(i);
    }
    f.sys_ids = mine;
    f.nsys = (int)mine.size();
    // Sine-domain form of every system a A + b M (exact algebra of the Kuhn face pair):
    //   Q (a A + b M) Q = diag(a α_ab + b μ̃_ab) + (b h^2/24) D̂ ⊗ D̂,
    //   α_ab = σ_a + σ_b,  μ̃_ab = (h^2/12)(6 + 2c_a + 2c_b + 2 c_a c_b),  D̂ = S D S,  (D v)_j = v_{j+1} - v_{j-1},
    // since M - M̃ = (h^2/24) D⊗D collects the (1,1)/(-1,-1) couplings minus their symmetrised part.
    const int ns = std::max(1, f.nsys);
    std::vector<double> sa(ns, 0.0), sb(ns, 1.0), swt(ns, 0.0), cs(ns, 0.0), dg((size_t)ns * f.NP, 0.0),
        idg((size_t)ns * f.NP, 0.0);
    for (int i = 0; i < f.nsys; i++) {
        const Sys& s = sys[mine[i]];
        sa[i] = s.a; sb[i] = s.b; swt[i] = s.w;
        cs[i] = (double)((long double)s.b * h * h / 24.0L);
        for (int a = 0; a < n; a++)
            for (int b = 0; b < n; b++) {
                const long double ca = 1.0L - 0.5L * sig[a], cb = 1.0L - 0.5L * sig[b];
                const long double alpha = sig[a] + sig[b];
                const long double mut = (long double)hh12 * (6.0L + 2.0L * ca + 2.0L * cb + 2.0L * ca * cb);
                const long double d = (long double)s.a * alpha + (long double)s.b * mut;
                const size_t e = (size_t)ipos[a] * f.ldf + ipos[b];
                dg[(size_t)i * f.NP + e] = (double)d;
                idg[(size_t)i * f.NP + e] = (double)(1.0L / d);
            }
    }
    std::vector<double> Dh((size_t)Srows * f.ldf, 0.0);
    {
        std::vector<long double> SL((size_t)n * n);
        for (int q = 0; q < n; q++)
            for (int r = 0; r < n; r++) SL[(size_t)q * n + r] = sc * sintab[((long long)(q + 1) * (r + 1)) % (2 * N)];
        for (int a = 0; a < n; a++)
            for (int b = 0; b < n; b++) {
                long double acc = 0.0L;
                for (int j = 0; j < n; j++) {
                    const long double dj = (j + 1 < n ? SL[(size_t)(j + 1) * n + b] : 0.0L) - (j >= 1 ? SL[(size_t)(j - 1) * n + b] : 0.0L);
                    acc += SL[(size_t)a * n + j] * dj;
                }
                // parity order; D̂_ab = 0 exactly when a + b is even (Σ_j sin(j a θ) cos(j b θ) over
                // a sum of even frequencies vanishes), stored as an exact zero
                Dh[(size_t)ipos[a] * f.ldf + ipos[b]] = (a + b) % 2 == 0 ? 0.0 : (double)acc;
            }
    }
    // D̂ = S D S is antisymmetric (S symmetric, D antisymmetric): make the table exactly so, so that
    // the fused Chebyshev step may use E = D̂[o][e] for both off-diagonal blocks (D̂[e][o] = -E^T)
    for (int i = 0; i < n; i++)
        for (int j2 = 0; j2 < i; j2++) Dh[(size_t)i * f.ldf + j2] = -Dh[(size_t)j2 * f.ldf + i];
    {
        const char* fz = std::getenv("DD_CHEB_FUSED");
        f.cheb_fused = cheb_fused_ok(n, f.ldf) && !(fz && fz[0] == '0');
    }
    DD_CK(dalloc(c, &f.Dh, Dh.size()));
    DD_CK(cudaMemcpyAsync(f.Dh, Dh.data(), Dh.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    DD_CK(dalloc(c, &f.sys_a, ns));
    DD_CK(dalloc(c, &f.sys_b, ns));
    DD_CK(dalloc(c, &f.sys_w, ns));
    DD_CK(dalloc(c, &f.cs, ns));
    DD_CK(dalloc(c, &f.dg, dg.size()));
    DD_CK(dalloc(c, &f.idg, idg.size()));
    DD_CK(cudaMemcpyAsync(f.sys_a, sa.data(), ns * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    DD_CK(cudaMemcpyAsync(f.sys_b, sb.data(), ns * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    DD_CK(cudaMemcpyAsync(f.sys_w, swt.data(), ns * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    DD_CK(cudaMemcpyAsync(f.cs, cs.data(), ns * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    DD_CK(cudaMemcpyAsync(f.dg, dg.data(), dg.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    DD_CK(cudaMemcpyAsync(f.idg, idg.data(), idg.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    {
        const char* icg = std::getenv("DD_INNER_CG");
        f.inner_cheb = !(icg && icg[0] == '1');
        std::vector<std::pair<double, double>> ab;
        for (int i = 0; i < f.nsys; i++) ab.emplace_back(sa[i], sb[i]);
        std::vector<double> c1, c2;
        std::vector<int> K;
        build_cheb(ab, hh12, f.inner_rtol, c1, c2, K, f.kmax_all);
        DD_CK(dalloc(c, &f.cc1, c1.size()));
        DD_CK(dalloc(c, &f.cc2, c2.size()));
        DD_CK(dalloc(c, &f.kmax, K.size()));
        DD_CK(cudaMemcpyAsync(f.cc1, c1.data(), c1.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        DD_CK(cudaMemcpyAsync(f.cc2, c2.data(), c2.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        DD_CK(cudaMemcpyAsync(f.kmax, K.data(), K.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
        DD_CK(cudaStreamSynchronize(c->stream));
    }

    // --- RA mode: the r_F systems (fc0 M + Σ_k fc_k (A - fp_k M)^-1 ≈ L^t) in the same sine-domain form
    if (c->frac_mode == DD_FRAC_RA) {
        std::vector<Sys> fsys;
        if (c->fra_c0 != 0.0) fsys.push_back({0.0, 1.0, c->fra_c0, 1.0});
        for (size_t k = 0; k < c->fra_poles.size(); k++)
            if (c->fra_res[k] != 0.0) fsys.push_back({1.0, -c->fra_poles[k], c->fra_res[k], 1.0});
        FSet& F = f.fs;
        F.nsys = (int)fsys.size();
        const int nf = std::max(1, F.nsys);
        std::vector<double> fa(nf, 0.0), fb(nf, 1.0), fw(nf, 0.0), fcs(nf, 0.0), fdg((size_t)nf * f.NP, 0.0),
            fidg((size_t)nf * f.NP, 0.0);
        for (int i = 0; i < F.nsys; i++) {
            const Sys& sy = fsys[i];
            fa[i] = sy.a; fb[i] = sy.b; fw[i] = sy.w;
            fcs[i] = (double)((long double)sy.b * h * h / 24.0L);
            for (int a = 0; a < n; a++)
                for (int b = 0; b < n; b++) {
                    const long double ca = 1.0L - 0.5L * sig[a], cb = 1.0L - 0.5L * sig[b];
                    const long double alpha = sig[a] + sig[b];
                    const long double mut = (long double)hh12 * (6.0L + 2.0L * ca + 2.0L * cb + 2.0L * ca * cb);
                    const long double d = (long double)sy.a * alpha + (long double)sy.b * mut;
                    const size_t e = (size_t)ipos[a] * f.ldf + ipos[b];
                    fdg[(size_t)i * f.NP + e] = (double)d;
                    fidg[(size_t)i * f.NP + e] = (double)(1.0L / d);
                }
        }
        for (double** v : {&F.sys_a, &F.sys_b, &F.sys_w, &F.cs}) DD_CK(dalloc(c, v, nf));
        DD_CK(dalloc(c, &F.dg, fdg.size()));
        DD_CK(dalloc(c, &F.idg, fidg.size()));
        DD_CK(cudaMemcpyAsync(F.sys_a, fa.data(), nf * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        DD_CK(cudaMemcpyAsync(F.sys_b, fb.data(), nf * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        DD_CK(cudaMemcpyAsync(F.sys_w, fw.data(), nf * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        DD_CK(cudaMemcpyAsync(F.cs, fcs.data(), nf * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        DD_CK(cudaMemcpyAsync(F.dg, fdg.data(), fdg.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        DD_CK(cudaMemcpyAsync(F.idg, fidg.data(), fidg.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        std::vector<std::pair<double, double>> fab;
        for (int i = 0; i < F.nsys; i++) fab.emplace_back(fa[i], fb[i]);
        std::vector<double> c1, c2;
        std::vector<int> K;
        build_cheb(fab, hh12, f.inner_rtol, c1, c2, K, F.kmax_all);
        DD_CK(dalloc(c, &F.cc1, c1.size()));
        DD_CK(dalloc(c, &F.cc2, c2.size()));
        DD_CK(dalloc(c, &F.kmax, K.size()));
        DD_CK(cudaMemcpyAsync(F.cc1, c1.data(), c1.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        DD_CK(cudaMemcpyAsync(F.cc2, c2.data(), c2.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        DD_CK(cudaMemcpyAsync(F.kmax, K.data(), K.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
        DD_CK(cudaStreamSynchronize(c->stream));
    }

    // --- per-parameter K, γ and workspaces
    DD_CK(dalloc(c, &c->Kp, c->n_param));
    DD_CK(dalloc(c, &c->gp, c->n_param));
    DD_CK(cudaMemcpyAsync(c->Kp, K, c->n_param * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    DD_CK(cudaMemcpyAsync(c->gp, mu_inv, c->n_param * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    const int cp8 = round_up(c->max_cols, 8);
    const size_t vec = (size_t)f.NP * cp8 + slack;
    for (double** v : {&f.x, &f.r, &f.p, &f.q, &f.z, &f.U1, &f.U2}) DD_CK(dalloc(c, v, vec));
    const size_t pairs = (size_t)ns * c->max_cols;
    const size_t pv = (size_t)f.NP * pairs + slack;
    for (double** v : {&f.ix, &f.ir, &f.ip, &f.iq, &f.iz, &f.T1, &f.T2}) DD_CK(dalloc(c, v, pv));
    if (c->frac_mode == DD_FRAC_RA) {
        FSet& F = f.fs;
        const size_t fpv = (size_t)f.NP * std::max(1, F.nsys) * c->max_cols + slack;
        for (double** v : {&F.ix, &F.ir, &F.ip, &F.iq, &F.iz, &F.T1}) DD_CK(dalloc(c, v, fpv));
        DD_CK(dalloc(c, &F.irho, (size_t)std::max(1, F.nsys) * c->max_cols));
        DD_CK(dalloc(c, &F.irho0, (size_t)std::max(1, F.nsys) * c->max_cols));
        DD_CK(dalloc(c, &F.iactive, (size_t)std::max(1, F.nsys) * c->max_cols));
        for (double** v : {&F.V1, &F.V2, &F.W1, &F.W2}) DD_CK(dalloc(c, v, vec));
        DD_CK(dalloc(c, &F.gcol, cp8));
    }
    DD_CK(dalloc(c, &f.irho, pairs));
    DD_CK(dalloc(c, &f.irho0, pairs));
    DD_CK(dalloc(c, &f.iactive, pairs));
    DD_CK(dalloc(c, &f.Kcol, cp8));
    DD_CK(dalloc(c, &f.fx_ws, face_fx_ws_doubles(f.NP, cp8, c->num_sms)));
    DD_CK(dalloc(c, &f.fx_cnt, face_fx_tiles(f.NP, cp8) + 1));
    DD_CK(dalloc(c, &c->bst, (size_t)f.n2 * c->max_cols));
    DD_CK(dalloc(c, &c->xst, (size_t)f.n2 * c->max_cols));
    DD_CK(dalloc(c, &c->colp_st, c->max_cols));
    if (const char* it = std::getenv("DD_INNER_MAXIT")) f.inner_maxit = std::max(1, atoi(it));

    // --- NCCL communicator for the pole split (bootstrapped by the caller's unique id)
    if (f.world > 1 && dist->mode == DD_SHARD_POLES && dist->nccl_unique_id) {
        ncclUniqueId id;
        std::memcpy(&id, dist->nccl_unique_id, sizeof(id));
        ncclComm_t comm = nullptr;
        NK(ncclCommInitRank(&comm, f.world, id, f.rank));
        f.nccl = comm;
    }
    DD_CK(cudaStreamSynchronize(c->stream));
    return DD_OK;
}

void destroy_3d(dd_ctx* c) {
    if (c->f3.fs.exec) {
        cudaGraphExecDestroy(c->f3.fs.exec);
        c->f3.fs.exec = nullptr;
    }
    if (c->f3.inner_exec) {
        cudaGraphExecDestroy(c->f3.inner_exec);
        c->f3.inner_exec = nullptr;
    }
    if (c->f3.nccl) {
        ncclCommDestroy(static_cast<ncclComm_t>(c->f3.nccl));
        c->f3.nccl = nullptr;
    }
}

// One set of shifted face systems Σ_s w_s (a_s A + b_s M)^-1 applied by the batched sine-domain CG:
// the preconditioner's RA systems (Eq.(8)) or, in RA mode, the fractional term's r_F systems
// (Remark 1).  W1, W2: NP x ncols scratch for the transforms.
struct InnerView {
    int nsys;
    double *sys_a, *sys_b, *sys_w, *cs, *dg, *idg;
    double *ix, *ir, *ip, *iq, *iz, *T1, *irho, *irho0;
    int* iactive;
    cudaGraphExec_t* exec;
    int* key;
    bool* on_dev;
    int* last_iters;
    int slot_act, slot_cnt;        // ints[] slots: active-pair counter, iteration counter (+2: total)
    int slot_done;                 // ints[] slot: CTA arrival counter of the fused Chebyshev step
    long long* iter_launches;
    const double *cc1, *cc2;       // Chebyshev tables (reading A12')
    const int* kmax;
    int kmax_all;
};

static InnerView view_P(Face3& f, dd_ctx* c) {
    return InnerView{f.nsys, f.sys_a, f.sys_b, f.sys_w, f.cs, f.dg, f.idg, f.ix, f.ir, f.ip, f.iq, f.iz, f.T1,
                     f.irho, f.irho0, f.iactive, &f.inner_exec, &f.inner_key, &f.inner_iters_on_device,
                     &f.last_inner_iters, 1, 6, 9, &c->inner_iter_launches, f.cc1, f.cc2, f.kmax, f.kmax_all};
}
static InnerView view_F(Face3& f, dd_ctx* c) {
    FSet& s = f.fs;
    return InnerView{s.nsys, s.sys_a, s.sys_b, s.sys_w, s.cs, s.dg, s.idg, s.ix, s.ir, s.ip, s.iq, s.iz, s.T1,
                     s.irho, s.irho0, s.iactive, &s.exec, &s.key, &s.on_dev, &s.last_iters, 11, 12, 10,
                     &c->f_inner_iter_launches, s.cc1, s.cc2, s.kmax, s.kmax_all};
}

// hat_io: r and z already live in the parity-ordered sine domain (the 3D PCG with H̃): no transforms
static dd_status inner_apply(dd_ctx* c, const InnerView& v, int ncols, const double* r, double* z, double* W1,
                             double* W2, bool hat_io = false) {
    Face3& f = c->f3;
    InnerArgs a{};
    a.n = f.n; a.ldf = f.ldf; a.NP = f.NP;
    a.npair = v.nsys * ncols; a.C = ncols;
    a.hh12 = (double)(1.0L / ((long double)c->N * c->N * 12.0L));
    a.sys_a = v.sys_a; a.sys_b = v.sys_b;
    a.x = v.ix; a.r = v.ir; a.p = v.ip; a.q = v.iq; a.z = v.iz;
    a.rho = v.irho; a.rho0 = v.irho0; a.active = v.iactive; a.rtol = f.inner_rtol;
    a.dg = v.dg; a.idg = v.idg; a.cs = v.cs;
    int* n_act_slot = c->ints + v.slot_act;
    int* cnt_slot = c->ints + v.slot_cnt;
    // r̂_c = Q r_c once per column (2 slab passes, into the parity-ordered sine domain); hat_io: r̂ given —
    // read in place by the cooperative multi-step path, else copied into W2 (the b̂ slot a captured
    // WHILE loop has baked in)
    static const bool multi_env = !(std::getenv("DD_CHEB_MULTI") && std::getenv("DD_CHEB_MULTI")[0] == '0');
    const bool multi = f.inner_cheb && v.cc1 && f.cheb_fused && multi_env;
    const double* bh = W2;
    if (hat_io && multi) {
        bh = r;
    } else if (hat_io) {
        DD_CK(cudaMemcpyAsync(W2, r, sizeof(double) * (size_t)f.NP * ncols, cudaMemcpyDeviceToDevice, c->stream));
    } else {
        DD_TIMED(DD_KCLASS_POLESUM, face_slab_pass(r, W1, ncols, f.n, f.ldf, f.Sp, c->stream));
        DD_TIMED(DD_KCLASS_POLESUM, face_slab_pass(W1, W2, ncols, f.n, f.ldf, f.Sp, c->stream));
    }
    const bool cheb = f.inner_cheb && v.cc1;
    a.cc1 = v.cc1; a.cc2 = v.cc2; a.kmax = v.kmax; a.kstride = CHEB_KMAX; a.kiter = cnt_slot;
    // Chebyshev: step 1 is the init (x̂_1 = P^-1 b̂), the loop runs the other K_s - 1
    const int loop_max = cheb ? std::min(f.inner_maxit, v.kmax_all - 1) : f.inner_maxit;
    if (cheb) DD_TIMED(DD_KCLASS_POLESUM, inner_init_cheb(a, bh, c->stream));
    else DD_TIMED(DD_KCLASS_POLESUM, inner_init_hat(a, W2, c->stream));
    // fused Chebyshev step (n_e = 64): one persistent kernel per step that also evaluates the loop
    // condition, so it stands in the condition slot and the body is empty
    const bool fused = cheb && f.cheb_fused;
    if (fused) a.x1 = v.iz;
    auto body = [&](cudaStream_t st, int* n_act) -> dd_status {
        if (fused) return DD_OK;
        if (cheb) {
            // T = D̂ x̂ (active pairs), then r, d and x̂ in the second pass's epilogue
            DD_TIMED(DD_KCLASS_POLESUM, face_slab_pass_active(v.ix, v.T1, a.npair, f.n, f.ldf, f.Dh, v.iactive, f.kpar,
                                                              st));
            DD_TIMED(DD_KCLASS_POLESUM, face_inner_cheb_pass(v.T1, a, W2, f.Dh, f.kpar, st));
            return DD_OK;
        }
        // q̂ = dg ∘ p̂ + cs D̂ p̂ D̂^T on the active pairs, then the fused CG update
        DD_TIMED(DD_KCLASS_POLESUM, face_slab_pass_active(v.ip, v.T1, a.npair, f.n, f.ldf, f.Dh, v.iactive, f.kpar, st));
        DD_TIMED(DD_KCLASS_POLESUM, face_inner_op_pass(v.T1, v.iq, v.ip, a.npair, ncols, f.n, f.ldf, f.Dh, v.dg, v.cs,
                                                       v.iactive, f.kpar, st));
        DD_TIMED(DD_KCLASS_POLESUM, inner_update_hat(a, n_act, st));
        return DD_OK;
    };
    auto cond = [&](cudaStream_t st, unsigned long long h) -> cudaError_t {
        if (fused)
            return cheb_step_fused(a, W2, f.Dh, n_act_slot, cnt_slot, c->ints + v.slot_done, loop_max, h, c->num_sms, st);
        return cheb ? inner_cond_cheb(a, n_act_slot, cnt_slot, loop_max, h, st)
                    : inner_cond(n_act_slot, cnt_slot, loop_max, h, st);
    };
    // fused steps all in one cooperative launch (grid barrier between steps; DD_CHEB_MULTI=0: one launch
    // per step inside the WHILE graph)
    if (cheb && loop_max <= 0) {
        // every system is done after the init step
        DD_CK(cudaMemsetAsync(cnt_slot, 0, sizeof(int), c->stream));
        *v.last_iters = 0;
        *v.on_dev = false;
    } else if (multi) {
        DD_CK(cudaMemsetAsync(cnt_slot, 0, sizeof(int), c->stream));
        DD_TIMED(DD_KCLASS_POLESUM, cheb_step_fused(a, bh, f.Dh, n_act_slot, cnt_slot, c->ints + v.slot_done, loop_max,
                                                    0ull, c->num_sms, c->stream, loop_max));
        *v.last_iters = loop_max;
        *v.on_dev = false;
    } else if (c->graph_ok && !c->prof) {
        // the whole inner loop as one conditional WHILE graph (no host round trips)
        if (!*v.exec || *v.key != ncols) {
            if (*v.exec) cudaGraphExecDestroy(*v.exec);
            *v.exec = nullptr;
            cudaGraph_t g = nullptr;
            DD_CK(cudaGraphCreate(&g, 0));
            cudaGraphConditionalHandle h;
            DD_CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
            cudaGraphNodeParams cp = {};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = h;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            cudaGraphNode_t node;
            DD_CK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
            cudaStream_t cap = nullptr;
            DD_CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
            DD_CK(cudaStreamBeginCaptureToGraph(cap, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                cudaStreamCaptureModeRelaxed));
            const bool prof = c->prof;
            c->prof = false;
            const long long l0 = c->launches;
            dd_status bs = body(cap, n_act_slot);
            cudaError_t ce = cond(cap, (unsigned long long)h);
            *v.iter_launches = c->launches - l0 + 1;
            c->launches = l0;
            c->prof = prof;
            cudaGraph_t captured = nullptr;
            cudaError_t ee = cudaStreamEndCapture(cap, &captured);
            cudaStreamDestroy(cap);
            if (bs != DD_OK || ce != cudaSuccess || ee != cudaSuccess) {
                cudaGraphDestroy(g);
                return bs != DD_OK ? bs : set_error(DD_ECUDA, "inner-loop graph capture");
            }
            DD_CK(cudaGraphInstantiate(v.exec, g, 0));
            cudaGraphDestroy(g);
            *v.key = ncols;
        }
        DD_CK(cudaMemsetAsync(cnt_slot, 0, sizeof(int), c->stream));
        DD_CK(cudaMemsetAsync(n_act_slot, 0, sizeof(int), c->stream));
        DD_CK(cudaGraphLaunch(*v.exec, c->stream));
        *v.on_dev = true;
    } else {
        int it = 0;
        DD_CK(cudaMemsetAsync(cnt_slot, 0, sizeof(int), c->stream));
        for (it = 1; it <= loop_max; it++) {
            if (!cheb) DD_CK(cudaMemsetAsync(n_act_slot, 0, sizeof(int), c->stream));
            dd_status bs = body(c->stream, n_act_slot);
            if (bs != DD_OK) return bs;
            if (cheb) DD_TIMED(DD_KCLASS_POLESUM, cond(c->stream, 0ull));   // (fused step +) counter, flags, *n_active
            if (it % 4 == 0 || it == loop_max) {
                DD_CK(cudaMemcpyAsync(c->h_ints + v.slot_act, n_act_slot, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
                DD_CK(cudaStreamSynchronize(c->stream));
                if (c->h_ints[v.slot_act] == 0) break;
            }
        }
        *v.last_iters = std::min(it, loop_max);
        *v.on_dev = false;
    }
    // ẑ_c = Σ_s w_s x̂_{s,c} (fixed system order), z_c = Q ẑ_c
    if (hat_io) {
        DD_TIMED(DD_KCLASS_POLESUM, inner_combine(a, v.sys_w, v.nsys, z, c->stream));
        return DD_OK;
    }
    DD_TIMED(DD_KCLASS_POLESUM, inner_combine(a, v.sys_w, v.nsys, W1, c->stream));
    DD_TIMED(DD_KCLASS_POLESUM, face_slab_pass(W1, W2, ncols, f.n, f.ldf, f.SpT, c->stream));
    DD_TIMED(DD_KCLASS_POLESUM, face_slab_pass(W2, z, ncols, f.n, f.ldf, f.SpT, c->stream));
    return DD_OK;
}

// z = P_RA r on padded face vectors (rank-local systems, then the allreduce of the pole split)
static dd_status precond_core(dd_ctx* c, int ncols, const double* r, double* z, bool hat_io = false) {
    Face3& f = c->f3;
    if (f.nsys == 0) {
        DD_CK(cudaMemsetAsync(z, 0, sizeof(double) * (size_t)f.NP * ncols, c->stream));
    } else {
        dd_status s = inner_apply(c, view_P(f, c), ncols, r, z, f.U1, f.U2, hat_io);
        if (s != DD_OK) return s;
    }
    if (f.nccl) {
        NK(ncclAllReduce(z, z, (size_t)f.NP * ncols, ncclDouble, ncclSum, static_cast<ncclComm_t>(f.nccl), c->stream));
    }
    return DD_OK;
}

// y = S x on padded face vectors p -> q
// q = γ F p + D with the dense F stream (row a-3); a row-sharded F (pole split, §8(e)) computes this
// rank's rows and gathers the others with one ncclAllGather (without a communicator — ranks emulated
// in one process — the other rows are zero, so the ranks' outputs add up to the full product)
// Mat = F (γ per column, + D) or the folded H rows (Mat = f.Hrows, gp = D = NULL)
static dd_status fx_apply(dd_ctx* c, int ncols, const int* colp, const double* p, double* q, const double* D,
                          const double* Mat, const double* gp) {
    Face3& f = c->f3;
    const int rows = f.fx_r1 - f.fx_r0;
    if (rows >= f.NP) {
        DD_TIMED(DD_KCLASS_GEMM_SCHUR, face_fx(Mat, f.NP, p, q, D, ncols, colp, c->n_param, gp, f.fx_ws, f.fx_cnt,
                                               c->num_sms, c->stream));
        return DD_OK;
    }
    if (rows > 0)
        DD_TIMED(DD_KCLASS_GEMM_SCHUR, face_fx(Mat, f.NP, p, q, D, ncols, colp, c->n_param, gp, f.fx_ws, f.fx_cnt,
                                               c->num_sms, c->stream, f.fx_r0, rows));
    if (f.nccl) {
        DD_TIMED(DD_KCLASS_OTHER, fx_pack(q, f.NP, ncols, f.fx_r0, rows, f.fx_rows_max, f.fx_send, c->stream));
        NK(ncclAllGather(f.fx_send, f.fx_recv, (size_t)ncols * f.fx_rows_max, ncclDouble,
                         static_cast<ncclComm_t>(f.nccl), c->stream));
        DD_TIMED(DD_KCLASS_OTHER, fx_unpack(f.fx_recv, f.NP, ncols, f.world, f.fx_rows_max, f.fx_r0s, q, c->stream));
    } else {
        DD_TIMED(DD_KCLASS_OTHER, fx_zero_outside(f.NP, ncols, f.fx_r0, f.fx_r1, q, c->stream));
    }
    return DD_OK;
}

// q̂ = H̃ p̂ in the parity-ordered sine domain (the 3D PCG's Schur apply when f.hat)
static dd_status schur_core_hat(dd_ctx* c, int ncols, const int* colp, const double* p, double* q) {
    Face3& f = c->f3;
    DD_TIMED(DD_KCLASS_GEMM_SCHUR, fx_sym_apply(f.Hp, f.fblk, f.NP, p, q, nullptr, ncols, colp, c->n_param, nullptr,
                                                f.fxD, f.fxT, c->num_sms, c->stream, f.hat && f.hat_cs));
    return DD_OK;
}

static dd_status schur_core(dd_ctx* c, int ncols, const int* colp, const double* p, double* q) {
    Face3& f = c->f3;
    if (f.Hp) {
        // S = K S_unit + γ F folded at setup into one packed-symmetric stream; with f.hat that
        // operator is T S T^T, so a physical-domain apply transforms in and out
        if (!f.hat) return schur_core_hat(c, ncols, colp, p, q);
        DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass(p, f.U1, ncols, f.n, f.ldf, f.Sp, c->stream));
        DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass(f.U1, f.U2, ncols, f.n, f.ldf, f.Sp, c->stream));
        dd_status st = schur_core_hat(c, ncols, colp, f.U2, f.U1);
        if (st != DD_OK) return st;
        DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass(f.U1, f.U2, ncols, f.n, f.ldf, f.SpT, c->stream));
        DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass(f.U2, q, ncols, f.n, f.ldf, f.SpT, c->stream));
        return DD_OK;
    }
    if (f.Hrows) return fx_apply(c, ncols, colp, p, q, nullptr, f.Hrows, nullptr);   // this rank's rows of H
    DD_TIMED(DD_KCLASS_OTHER, gather_param(ncols, colp, c->n_param, c->Kp, f.Kcol, c->stream));
    DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass(p, f.U1, ncols, f.n, f.ldf, f.S, c->stream));
    DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass_scaled(f.U1, f.U2, ncols, f.n, f.ldf, f.S, f.sw, 0, 1, f.Kcol, c->stream));
    DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass(f.U2, f.U1, ncols, f.n, f.ldf, f.S, c->stream));
    DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass(f.U1, f.U2, ncols, f.n, f.ldf, f.S, c->stream));
    if (c->frac_mode == DD_FRAC_RA) {
        // Remark 1: γ F p ≈ γ M r_F(L) M p — the face pole sum of the r_F systems
        // between two consistent-mass products, no dense F
        const double hh12 = (double)(1.0L / ((long double)c->N * c->N * 12.0L));
        DD_TIMED(DD_KCLASS_OTHER, gather_param(ncols, colp, c->n_param, c->gp, f.fs.gcol, c->stream));
        DD_TIMED(DD_KCLASS_GEMM_SCHUR, face_mass_axpy(f.n, f.ldf, f.NP, ncols, hh12, p, nullptr, nullptr, f.fs.V1,
                                                      c->stream));
        dd_status s = inner_apply(c, view_F(f, c), ncols, f.fs.V1, f.fs.V2, f.fs.W1, f.fs.W2);
        if (s != DD_OK) return s;
        DD_TIMED(DD_KCLASS_GEMM_SCHUR, face_mass_axpy(f.n, f.ldf, f.NP, ncols, hh12, f.fs.V2, f.fs.gcol, f.U2, q,
                                                      c->stream));
        return DD_OK;
    }
    if (f.Fp) {
        DD_TIMED(DD_KCLASS_GEMM_SCHUR, fx_sym_apply(f.Fp, f.fblk, f.NP, p, q, f.U2, ncols, colp, c->n_param, c->gp,
                                                    f.fxD, f.fxT, c->num_sms, c->stream));
        return DD_OK;
    }
    return fx_apply(c, ncols, colp, p, q, f.U2, f.F, c->gp);
}

dd_status schur_3d(dd_ctx* c, int ncols, const int* colp, const double* xin, double* yout, bool user_layout) {
    Face3& f = c->f3;
    if (!user_layout) return schur_core(c, ncols, colp, xin, yout);
    DD_TIMED(DD_KCLASS_OTHER, face_copy_in(f.n, f.ldf, f.NP, ncols, xin, f.n2, f.p, c->stream));
    dd_status s = schur_core(c, ncols, colp, f.p, f.q);
    if (s != DD_OK) return s;
    DD_TIMED(DD_KCLASS_OTHER, face_copy_out(f.n, f.ldf, f.NP, ncols, f.q, yout, f.n2, c->stream));
    return DD_OK;
}

dd_status precond_3d(dd_ctx* c, int ncols, const int* colp, const double* rin, double* zout, bool user_layout) {
    (void)colp;
    Face3& f = c->f3;
    if (!user_layout) return precond_core(c, ncols, rin, zout);
    DD_TIMED(DD_KCLASS_OTHER, face_copy_in(f.n, f.ldf, f.NP, ncols, rin, f.n2, f.r, c->stream));
    dd_status s = precond_core(c, ncols, f.r, f.z);
    if (s != DD_OK) return s;
    DD_TIMED(DD_KCLASS_OTHER, face_copy_out(f.n, f.ldf, f.NP, ncols, f.z, zout, f.n2, c->stream));
    return DD_OK;
}

dd_status pcg_3d(dd_ctx* c, int ncols, const int* colp, const double* b, double* x, double rtol, int maxit,
                 int norm_kind) {
    Face3& f = c->f3;
    // f.hat: the whole PCG in the parity-ordered sine domain (T orthogonal: the same iteration, the
    // inner products invariant) — b transformed once, x transformed back once, no transforms inside
    const bool hat = f.hat;
    DD_TIMED(DD_KCLASS_OTHER, face_copy_in(f.n, f.ldf, f.NP, ncols, b, f.n2, f.r, c->stream));
    if (hat) {
        DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass(f.r, f.U1, ncols, f.n, f.ldf, f.Sp, c->stream));
        DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass(f.U1, f.r, ncols, f.n, f.ldf, f.Sp, c->stream));
    }
    dd_status s = precond_core(c, ncols, f.r, f.z, hat);
    if (s != DD_OK) return s;
    Pcg3 st{};
    st.NP = f.NP; st.ncols = ncols;
    st.x = f.x; st.r = f.r; st.p = f.p; st.q = f.q; st.z = f.z;
    st.rho = c->rho; st.eta0 = c->eta0; st.relres = c->relres; st.active = c->active; st.iters = c->iters;
    st.hist = c->hist_on ? c->hist : nullptr; st.rtol = rtol; st.norm_kind = norm_kind; st.status = c->ints + 4;
    DD_TIMED(DD_KCLASS_OTHER, pcg3_start(st, c->stream));
    int k = 0;
    for (k = 1; k <= maxit; k++) {
        s = hat ? schur_core_hat(c, ncols, colp, f.p, f.q) : schur_core(c, ncols, colp, f.p, f.q);
        if (s != DD_OK) return s;
        DD_TIMED(DD_KCLASS_OTHER, pcg3_alpha(st, c->stream));
        s = precond_core(c, ncols, f.r, f.z, hat);
        if (s != DD_OK) return s;
        DD_CK(cudaMemsetAsync(c->ints + 2, 0, sizeof(int), c->stream));
        DD_TIMED(DD_KCLASS_OTHER, pcg3_beta(st, k, maxit, c->ints + 2, c->stream));
        DD_CK(cudaMemcpyAsync(c->h_ints + 2, c->ints + 2, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
        DD_CK(cudaStreamSynchronize(c->stream));
        if (c->h_ints[2] == 0) break;
    }
    c->h_ints[0] = std::min(k, maxit);
    DD_CK(cudaMemcpyAsync(c->ints, c->h_ints, sizeof(int), cudaMemcpyHostToDevice, c->stream));
    DD_CK(cudaStreamSynchronize(c->stream));
    if (hat) {
        DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass(f.x, f.U1, ncols, f.n, f.ldf, f.SpT, c->stream));
        DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass(f.U1, f.x, ncols, f.n, f.ldf, f.SpT, c->stream));
    }
    DD_TIMED(DD_KCLASS_OTHER, face_copy_out(f.n, f.ldf, f.NP, ncols, f.x, x, f.n2, c->stream));
    return DD_OK;
}

// Full DD solve on bulk right-hand sides (3D; bulk3d.cu has the algebra)
// exact: x_Γ by the interface PCG (the bulk solve); else the Eq.(5) DD preconditioner 𝓑 with
// S_Γ^-1 realised by the handle's RA (the bulk PCG's preconditioner)
static dd_status bulk_eliminate_3d(dd_ctx* c, int ncols, const int* colp, const double* b, double* x, bool exact,
                                   double rtol, int maxit, int norm_kind, int* iters, double* rel_res);

dd_status bulk_solve_3d(dd_ctx* c, int ncols, const int* colp, const double* b, double* x, double rtol, int maxit,
                        int norm_kind, int* iters, double* rel_res) {
    return bulk_eliminate_3d(c, ncols, colp, b, x, true, rtol, maxit, norm_kind, iters, rel_res);
}

static dd_status bulk_eliminate_3d(dd_ctx* c, int ncols, const int* colp, const double* b, double* x, bool exact,
                                   double rtol, int maxit, int norm_kind, int* iters, double* rel_res) {
    Face3& f = c->f3;
    const int n = f.n, ldf = f.ldf, lk = f.ldf;
    const long long NP = f.NP;
    const size_t slack = (size_t)64 * ldf;
    const size_t field = (size_t)c->max_cols * n * NP + slack, faces = (size_t)c->max_cols * NP + slack;
    if (!f.b3X) {
        for (double** v : {&f.b3X, &f.b3T, &f.b3Y}) DD_CK(dalloc(c, v, field));
        DD_CK(dalloc(c, &f.b3L, (size_t)c->max_cols * NP * lk + slack));
        for (double** v : {&f.b3G, &f.b3W, &f.b3W2}) DD_CK(dalloc(c, v, faces));
        DD_CK(dalloc(c, &f.b3g, (size_t)c->max_cols * f.n2));
        DD_CK(dalloc(c, &f.b3xg, (size_t)c->max_cols * f.n2));
        std::vector<double> sig(n);
        const long double PI = 3.141592653589793238462643383279502884L;
        for (int a = 0; a < n; a++) {
            const long double sh = sinl(PI * (a + 1) / (2.0L * c->N));
            sig[a] = (double)(4.0L * sh * sh);
        }
        DD_CK(dalloc(c, &f.b3sig, (size_t)n));
        DD_CK(cudaMemcpyAsync(f.b3sig, sig.data(), sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
        DD_CK(cudaStreamSynchronize(c->stream));
    }
    const long long nb = (long long)n * n * n + (long long)n * n;
    const double* s1 = f.S;                  // row 1 of Q (the first interior layer)
    // Ŷ = (Q⊗Q⊗Q b_0) / Σ;  b_Γ -> G
    DD_TIMED(DD_KCLASS_OTHER, bulk3_in(n, ldf, NP, ncols, b, nb, f.b3X, f.b3G, c->stream));
    DD_TIMED(DD_KCLASS_GEMM_DST, bulk3_forward(n, ldf, lk, NP, ncols, f.S, f.b3sig, f.b3X, f.b3T, f.b3L, f.b3Y,
                                               c->stream));
    // g = b_Γ + (L^-1 b_0)|_{i=1} = b_Γ + (Q⊗Q) Σ_a s1_a Ŷ_a
    DD_TIMED(DD_KCLASS_OTHER, bulk3_layer1(n, NP, ncols, f.b3Y, s1, f.b3W, c->stream));
    DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass(f.b3W, f.b3W2, ncols, n, ldf, f.S, c->stream));
    DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass(f.b3W2, f.b3W, ncols, n, ldf, f.S, c->stream));
    DD_TIMED(DD_KCLASS_OTHER, bulk3_g(n, ldf, NP, ncols, f.b3G, f.b3W, f.b3g, c->stream));
    dd_status ps = DD_OK;
    if (exact) {
        // x_Γ = S^-1 g  (the interface PCG of this handle)
        ps = dd_pcg_solve(c, ncols, colp, f.b3g, f.b3xg, rtol, maxit, norm_kind, iters, rel_res, nullptr);
        if (ps != DD_OK && ps != DD_ENOCONV) return ps;
    } else {
        // z_Γ = P g  (Eq.(5)'s S_Γ^-1 by the RA preconditioner, Eq.(8))
        ps = precond_3d(c, ncols, colp, f.b3g, f.b3xg, true);
        if (ps != DD_OK) return ps;
    }
    // x̂_0 = Ŷ / (K h) + s1 ⊗ (Q⊗Q x_Γ) / Σ;  x_0 = Q⊗Q⊗Q x̂_0
    DD_TIMED(DD_KCLASS_OTHER, bulk3_pad(n, ldf, NP, ncols, f.b3xg, f.n2, f.b3W2, c->stream));
    DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass(f.b3W2, f.b3W, ncols, n, ldf, f.S, c->stream));
    DD_TIMED(DD_KCLASS_GEMM_DST, face_slab_pass(f.b3W, f.b3W2, ncols, n, ldf, f.S, c->stream));
    DD_TIMED(DD_KCLASS_OTHER, bulk3_combine(n, ldf, NP, ncols, f.b3Y, f.b3W2, s1, f.b3sig, colp, c->n_param, c->Kp,
                                            1.0 / c->N, c->stream));
    DD_TIMED(DD_KCLASS_GEMM_DST, bulk3_inverse(n, ldf, lk, NP, ncols, f.S, f.b3Y, f.b3T, f.b3L, f.b3X, c->stream));
    DD_TIMED(DD_KCLASS_OTHER, bulk3_out(n, ldf, NP, ncols, f.b3X, f.b3xg, x, nb, c->stream));
    return ps;
}

// PCG on the 3D bulk system 𝒜 x = b preconditioned by 𝓑 (Eq.(5)), x0 = 0, stopping on
// sqrt(r·𝓑r) <= rtol sqrt(r0·𝓑r0) (reading A1) — the 2D loop of dd_api.cpp
dd_status bulk_pcg_3d(dd_ctx* c, int ncols, const int* colp, const double* b, double* x, double rtol, int maxit,
                      int* iters, double* rel_res) {
    Face3& f = c->f3;
    const int n = f.n, ldf = f.ldf;
    const long long NP = f.NP;
    const long long nb = (long long)n * n * n + (long long)n * n;
    if (!c->bpcg_r) {
        for (double** v : {&c->bpcg_r, &c->bpcg_p, &c->bpcg_q, &c->bpcg_z}) DD_CK(dalloc(c, v, (size_t)nb * c->max_cols));
    }
    if (!f.b3Z) {
        DD_CK(dalloc(c, &f.b3Z, (size_t)c->max_cols * NP + (size_t)64 * ldf));    // zero faces (F-stream D)
        DD_CK(dalloc(c, &f.b3F, (size_t)c->max_cols * NP + (size_t)64 * ldf));
        DD_CK(dalloc(c, &f.b3P, (size_t)c->max_cols * NP + (size_t)64 * ldf));
    }
    DD_CK(cudaMemsetAsync(c->ints, 0, sizeof(int) * 8, c->stream));
    DD_TIMED(DD_KCLASS_OTHER, launch_check_params(ncols, colp, c->n_param, c->ints + 5, c->stream));
    DD_CK(cudaMemsetAsync(x, 0, sizeof(double) * (size_t)nb * ncols, c->stream));
    DD_CK(cudaMemcpyAsync(c->bpcg_r, b, sizeof(double) * (size_t)nb * ncols, cudaMemcpyDeviceToDevice, c->stream));
    auto apply = [&](const double* in, double* out) -> dd_status {
        DD_TIMED(DD_KCLASS_OTHER, bulk3_pad(n, ldf, NP, ncols, in + (size_t)n * n * n, nb, f.b3P, c->stream));
        if (c->frac_mode == DD_FRAC_RA) {
            // Remark 1: γ F x_Γ ≈ γ M r_F(L) M x_Γ — the operator evaluated by RA too
            const double hh12 = (double)(1.0L / ((long double)c->N * c->N * 12.0L));
            DD_TIMED(DD_KCLASS_OTHER, gather_param(ncols, colp, c->n_param, c->gp, f.fs.gcol, c->stream));
            DD_TIMED(DD_KCLASS_GEMM_SCHUR, face_mass_axpy(f.n, f.ldf, f.NP, ncols, hh12, f.b3P, nullptr, nullptr,
                                                          f.fs.V1, c->stream));
            dd_status s = inner_apply(c, view_F(f, c), ncols, f.fs.V1, f.fs.V2, f.fs.W1, f.fs.W2);
            if (s != DD_OK) return s;
            DD_TIMED(DD_KCLASS_GEMM_SCHUR, face_mass_axpy(f.n, f.ldf, f.NP, ncols, hh12, f.fs.V2, f.fs.gcol, f.b3Z,
                                                          f.b3F, c->stream));
        } else if (f.Fp) {
            DD_TIMED(DD_KCLASS_GEMM_SCHUR, fx_sym_apply(f.Fp, f.fblk, NP, f.b3P, f.b3F, f.b3Z, ncols, colp, c->n_param,
                                                        c->gp, f.fxD, f.fxT, c->num_sms, c->stream));
        } else {
            dd_status fs = fx_apply(c, ncols, colp, f.b3P, f.b3F, f.b3Z, f.F, c->gp);
            if (fs != DD_OK) return fs;
        }
        DD_TIMED(DD_KCLASS_OTHER, bulk3_apply(n, ldf, NP, ncols, in, nb, f.b3F, colp, c->n_param, c->Kp, 1.0 / c->N, out,
                                              c->stream));
        return DD_OK;
    };
    dd_status st;
    if ((st = bulk_eliminate_3d(c, ncols, colp, c->bpcg_r, c->bpcg_z, false, 0, 0, 0, nullptr, nullptr)) != DD_OK)
        return st;
    DD_TIMED(DD_KCLASS_OTHER, bpcg_b(ncols, nb, c->bpcg_r, c->bpcg_z, c->bpcg_p, c->rho, c->eta0, c->relres, c->active,
                                     c->iters, 0, rtol, maxit, 1, c->ints + 1, c->ints + 4, c->stream));
    int k = 0;
    for (k = 1; k <= maxit; k++) {
        if ((st = apply(c->bpcg_p, c->bpcg_q)) != DD_OK) return st;
        DD_TIMED(DD_KCLASS_OTHER, bpcg_a(ncols, nb, x, c->bpcg_r, c->bpcg_p, c->bpcg_q, c->rho, c->active, c->ints + 4,
                                         c->stream));
        if ((st = bulk_eliminate_3d(c, ncols, colp, c->bpcg_r, c->bpcg_z, false, 0, 0, 0, nullptr, nullptr)) != DD_OK)
            return st;
        DD_CK(cudaMemsetAsync(c->ints + 1, 0, sizeof(int), c->stream));
        DD_TIMED(DD_KCLASS_OTHER, bpcg_b(ncols, nb, c->bpcg_r, c->bpcg_z, c->bpcg_p, c->rho, c->eta0, c->relres,
                                         c->active, c->iters, k, rtol, maxit, 0, c->ints + 1, c->ints + 4, c->stream));
        DD_CK(cudaMemcpyAsync(c->h_ints, c->ints, sizeof(int) * 8, cudaMemcpyDeviceToHost, c->stream));
        DD_CK(cudaStreamSynchronize(c->stream));
        if (c->h_ints[1] == 0 || c->h_ints[4] != 0) break;
    }
    if (iters) DD_CK(cudaMemcpyAsync(iters, c->iters, sizeof(int) * ncols, cudaMemcpyDeviceToHost, c->stream));
    if (rel_res) DD_CK(cudaMemcpyAsync(rel_res, c->relres, sizeof(double) * ncols, cudaMemcpyDeviceToHost, c->stream));
    DD_CK(cudaMemcpyAsync(c->h_ints, c->ints, sizeof(int) * 8, cudaMemcpyDeviceToHost, c->stream));
    DD_CK(cudaStreamSynchronize(c->stream));
    if (c->h_ints[5]) return set_error(DD_EINVAL, "col_param entry out of range (clamped; outputs undefined)");
    if (c->h_ints[4] == DD_ENOTSPD) return set_error(DD_ENOTSPD, "p.Ap <= 0 or r.Br < 0 in the bulk PCG");
    std::vector<int> itv(ncols);
    std::vector<double> rr(ncols);
    DD_CK(cudaMemcpy(itv.data(), c->iters, sizeof(int) * ncols, cudaMemcpyDeviceToHost));
    DD_CK(cudaMemcpy(rr.data(), c->relres, sizeof(double) * ncols, cudaMemcpyDeviceToHost));
    for (int i = 0; i < ncols; i++)
        if (itv[i] >= maxit && !(rr[i] <= rtol)) return set_error(DD_ENOCONV, "maxit reached");
    return DD_OK;
}

}  // namespace dd

extern "C" dd_status dd_nccl_unique_id(void* out128) {
    if (!out128) return dd::set_error(DD_EINVAL, "NULL buffer");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return dd::set_error(DD_ENCCL, ncclGetErrorString(r));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
    return DD_OK;
}

extern "C" dd_status dd_inner_iterations(const dd_ctx* c, int* iters) {
    if (!c || !iters) return dd::set_error(DD_EINVAL, "NULL argument");
    if (c->f3.inner_iters_on_device) {
        // the WHILE graph counts its iterations on the device (ints[6]); read it synchronously
        int v = 0;
        if (cudaSetDevice(c->device) != cudaSuccess || cudaStreamSynchronize(c->stream) != cudaSuccess ||
            cudaMemcpy(&v, c->ints + 6, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
            return dd::set_error(DD_ECUDA, "reading the inner iteration count");
        *iters = v;
        return DD_OK;
    }
    *iters = c->f3.last_inner_iters;
    return DD_OK;
}
