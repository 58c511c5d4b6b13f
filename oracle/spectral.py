"""Generalised eigen-factorisation and fractional powers (oracle; test infra only).

PAPER.md:172-180 (footnote, Eq.(7)): "the factorization L_h U_h = M_h U_h Λ_h,
U_h^T M_h U_h = Id holds ... We then define L^s_h = (M_h U_h) Λ^s_h (M_h U_h)^T."
PAPER.md:219-221: the fractional perturbation is γ T_h^T L^t_h T_h; for Eq.(2) t = -1/2
and T_h restricted to Γ is the identity on the Γ DOFs (reading A6), so the dense Γ×Γ
block of Fig. 1 is  F = L_h^{-1/2}.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla


def _scale_rows(w: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """diag(w) Y for a vector or a matrix Y."""
    return w * Y if Y.ndim == 1 else w[:, None] * Y


class GEVP:
    """Dense generalised eigenpairs of the SPD pair (L_h, M_h) via scipy.linalg.eigh
    (LAPACK: Cholesky reduction of M then a symmetric eigensolver)."""

    def __init__(self, L: np.ndarray, M: np.ndarray):
        lam, U = sla.eigh(L, M)
        self.lam, self.U, self.M, self.L = lam, U, M, L
        self.MU = M @ U

    def power(self, s: float, sigma: float = 0.0) -> np.ndarray:
        """L^s_h = (M U) Λ^s (M U)^T  (Eq.(7)); with sigma, of L + σM (same U, eigenvalues
        λ + σ) — Eq.(9)'s shifted L = -Δ_Γ + I_Γ for σ = 1."""
        return (self.MU * (self.lam + sigma) ** s) @ self.MU.T

    def apply_power(self, s: float, X: np.ndarray) -> np.ndarray:
        return self.MU @ _scale_rows(self.lam ** s, self.MU.T @ X)

    def apply_sum_inverse(self, terms, B: np.ndarray, sigma: float = 0.0) -> np.ndarray:
        """x = U diag(Σ_i α_i (λ+σ)^{s_i})^{-1} U^T b: the exact inverse of Σ_i α_i L^{s_i}
        in the Eq.(7) calculus (inverse of the Schur preconditioner Eq.(6), L = A + σM)."""
        w = np.zeros_like(self.lam)
        for alpha, s in terms:
            w = w + alpha * (self.lam + sigma) ** s
        return self.U @ _scale_rows(1.0 / w, self.U.T @ B)

    def apply_function(self, fvals: np.ndarray, B: np.ndarray) -> np.ndarray:
        """U diag(f(λ)) U^T b — the eigen form of any spectral function of the pair."""
        return self.U @ _scale_rows(fvals, self.U.T @ B)


def fractional_term(L: np.ndarray, M: np.ndarray, t: float = -0.5) -> np.ndarray:
    """Dense F = L_h^t (Eq.(7)); t = -1/2 for Eq.(2)."""
    return GEVP(L, M).power(t)
