"""Shared test helpers: RA fits for a parameter list, tolerances.  No method arithmetic."""
import numpy as np

from paper_2211_15308_b200 import rafit


def fit_all(N, params, m):
    lo, hi = rafit.interval_1d(N)
    return [rafit.fit_ra(K, g, lo, hi, m) for K, g in params]


def rel_l2_cols(a, b):
    """max over columns of ||a_c - b_c|| / ||b_c||  (arrays shaped (ncols, n))."""
    a = np.asarray(a); b = np.asarray(b)
    num = np.linalg.norm(a - b, axis=1)
    den = np.linalg.norm(b, axis=1)
    den = np.where(den == 0, 1.0, den)
    return float(np.max(num / den))


def kappa_c(r) -> float:
    """The cancellation factor κ_c of reading A11 computed by the ORACLE (oracle.ra.cancellation_factor)
    for an RA fit r (its c0/poles/residues, target f(K, γ, t, σ) and spectral interval), on the same
    2e4-point geometric grid of [λ_min, λ_max] the fit reports on."""
    from oracle import ra as ora
    xs = np.geomspace(r.lam_min, r.lam_max, 20000)
    return ora.cancellation_factor(r.c0, r.poles, r.residues, r.K, r.gamma, xs, t=getattr(r, "t", -0.5),
                                   sigma=getattr(r, "sigma", 0.0))


def precond_tol(ras):
    # max(1e-10, 1e-15 κ_c) relative ℓ2 (κ_c = cancellation factor, reading A11, from the oracle)
    return max(1e-10, 1e-15 * max(kappa_c(r) for r in ras))


def check_precond(z_gpu, z_banded, z_eigen, ras):
    """Preconditioner parity (reading A11'): the GPU result must match the oracle's
    eigen form U diag(r(λ)) U^T within max(1e-10, 1e-15 κ_c), and the oracle's parity form
    (LAPACK banded Cholesky per pole) within that bar plus the oracle's own measured
    parity-vs-eigen discrepancy (the banded solves of the least-shifted pole carry
    ~eps·cond(A_Γ - p M_Γ) ≈ 1e-10 at n = 4095)."""
    tol = precond_tol(ras)
    e_eig = rel_l2_cols(z_gpu, z_eigen)
    self_err = rel_l2_cols(z_banded, z_eigen)
    e_band = rel_l2_cols(z_gpu, z_banded)
    assert e_eig <= tol, (e_eig, tol)
    assert e_band <= tol + self_err, (e_band, tol, self_err)
    return e_eig, e_band, self_err
