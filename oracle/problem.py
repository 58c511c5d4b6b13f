"""Assembled Schur-system problem per parameter set (oracle; test infra only).

The system of the north star (Eq.(2)) on Γ after eliminating the bulk:
    S = K S_unit + γ F,   S_unit = A^ii - A^i0 (A^00)^-1 A^0i,   F = L_h^{-1/2}
(PAPER.md:107-122, 146-148, 178-180, 219-221), preconditioned by the RA of
S_Γ^-1 = (K L^{1/2} + γ L^{-1/2})^-1.

Two tiers:
  DenseProblem  — dense S_unit by elimination of the assembled stiffness, dense F by the
                  generalised eigendecomposition; any dim, small/moderate N.
  ModeProblem2D — 2D only, full config sizes: the same operators applied in the
                  orthonormal sine basis of Γ (scipy.fft DST-I), with S_unit's mode values
                  from the mode-wise layer elimination and the pair's mode values from the
                  assembled tridiagonal entries; pinned to DenseProblem in tests.
"""
from __future__ import annotations

import numpy as np

from . import fem, ra, schur, spectral


class DenseProblem:
    """t, sigma: the perturbation γ L^t with L = -Δ_Γ + σ I_Γ (Eq.(2): t = -1/2, σ = 0;
    Eq.(9): general -1 < t < 1 and σ = 1)."""

    def __init__(self, dim: int, N: int, method: str = "layers", t: float = -0.5, sigma: float = 0.0,
                 frac_ra=None):
        """frac_ra = (c0, poles, residues): the fractional term evaluated by RA (Remark 1,
        PAPER.md:274-288): F = M (c0 M^-1 + Σ c_k (A - p_k M)^-1) M instead of Eq.(7)."""
        self.dim, self.N, self.t, self.sigma = dim, N, t, sigma
        self.S_unit = schur.schur_layers(dim, N) if method == "layers" else schur.schur_bruteforce(dim, N)
        self.A_g, self.M_g = fem.trace_pair(dim, N)
        self.gevp = spectral.GEVP(self.A_g, self.M_g)
        if frac_ra is None:
            self.F = self.gevp.power(t, sigma)
        else:
            c0, poles, res = frac_ra
            self.F = self.M_g @ ra.apply_ra(self.A_g, self.M_g, c0, poles, res, self.M_g)
        self.n_gamma = self.S_unit.shape[0]

    def S(self, K, gamma):
        return K * self.S_unit + gamma * self.F

    def apply_S(self, K, gamma, X):
        return K * (self.S_unit @ X) + gamma * (self.F @ X)

    def apply_P_ra(self, c0, poles, residues, X):
        return ra.apply_ra(self.A_g, self.M_g, c0, poles, residues, X)

    def apply_P_exact(self, K, gamma, X):
        return ra.apply_exact_precond(self.gevp, K, gamma, X, self.t, self.sigma)

    def apply_P_ra_eigen(self, c0, poles, residues, X):
        return ra.apply_ra_eigen(self.gevp, c0, poles, residues, X)

    def spectrum(self):
        return self.gevp.lam


class ModeProblem2D:
    def __init__(self, N: int, t: float = -0.5, sigma: float = 0.0, frac_ra=None):
        self.dim, self.N, self.t, self.sigma = 2, N, t, sigma
        n = N - 1
        self.n_gamma = n
        a_d, a_o, m_d, m_o = fem.trace_pair_1d(N)
        # uniform mesh: constant Toeplitz entries; mode value = diag + 2 off cos θ_b
        assert np.allclose(a_d, a_d[0]) and np.allclose(m_d, m_d[0])
        k = np.arange(1, n + 1)
        cm1 = -2.0 * np.sin(0.5 * np.pi * k / (n + 1)) ** 2     # cos θ_b - 1 without cancellation (A18)
        ao = a_o[0] if n > 1 else 0.0
        mo = m_o[0] if n > 1 else 0.0
        # mode value diag + 2 off cos θ written as (diag + 2 off) + 2 off (cos θ - 1): for A_Γ the first
        # bracket vanishes and the low modes keep full relative precision (reading A26)
        self.alpha = (a_d[0] + 2.0 * ao) + 2.0 * ao * cm1   # A_Γ mode values
        self.mu = (m_d[0] + 2.0 * mo) + 2.0 * mo * cm1      # M_Γ mode values
        self.lam = self.alpha / self.mu             # generalised eigenvalues of (A_Γ, M_Γ)
        self.s = schur.schur_modes_2d(N)            # S_unit mode values
        self.f = self.mu * (self.lam + sigma) ** t  # F mode values: (MU) (Λ+σ)^t (MU)^T
        if frac_ra is not None:                     # Remark 1: (MU) r_F(Λ) (MU)^T
            self.f = self.mu * ra.r_eval(self.lam, *frac_ra)
        self.band = (a_d, a_o, m_d, m_o)

    def apply_S(self, K, gamma, X):
        Xh = schur.dst_ortho(X, axis=0)
        w = (K * self.s + gamma * self.f)
        return schur.dst_ortho(w[:, None] * Xh if X.ndim == 2 else w * Xh, axis=0)

    def apply_P_ra(self, c0, poles, residues, X):
        """Parity form: banded Cholesky solves of the assembled tridiagonal pair."""
        a_d, a_o, m_d, m_o = self.band
        return ra.apply_ra_banded_tri(a_d, a_o, m_d, m_o, c0, poles, residues, X)

    def apply_P_ra_eigen(self, c0, poles, residues, X):
        """Eigen form U diag(r(λ)) U^T X of the same RA operator (fixed point (ii) of SURVEY §8c):
        (A - pM)^-1 = U diag(1/(λ-p)) U^T with U = S_dst diag(μ^-1/2)."""
        Xh = schur.dst_ortho(X, axis=0)
        w = ra.r_eval(self.lam, c0, poles, residues) / self.mu
        return schur.dst_ortho(w[:, None] * Xh if X.ndim == 2 else w * Xh, axis=0)

    def apply_P_exact(self, K, gamma, X):
        Xh = schur.dst_ortho(X, axis=0)
        x = self.lam + self.sigma
        w = 1.0 / (self.mu * (K * x ** 0.5 + gamma * x ** self.t))
        return schur.dst_ortho(w[:, None] * Xh if X.ndim == 2 else w * Xh, axis=0)

    def spectrum(self):
        return np.sort(self.lam)
