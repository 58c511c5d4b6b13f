"""Rational-approximation solution operator and the exact Schur preconditioner (oracle).

PAPER.md:188-199 (footnote, Eq.(8)): the RA solution operator
    c_0 M_h^-1 + Σ_{k=1}^m c_k (L_h + p_k M_h)^-1
approximates the inverse of α L^s + β L^t via a rational approximation f_RA of
f(x) = (α x^s + β x^t)^-1 with ||f - f_RA|| <= ε_RA.
Here (Eq.(6)) S_Γ = K L^{1/2} + γ L^{-1/2}, so
f(x) = 1/(K x^{1/2} + γ x^{-1/2}).
Sign convention (reading A7): the poles passed around are the scalar poles of
r(x) = c0 + Σ c_k/(x - p_k), all p_k < 0; the shifted matrices are A_Γ - p_k M_Γ.

The fit itself (which poles) is an INPUT here: the paper defers the construction to its
references.  The oracle only evaluates and applies a given RA and
measures its error (the north-star fixed point "the rational-approximation error bound
on the spectral interval").
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def f_target(x, K: float, gamma: float, t: float = -0.5, sigma: float = 0.0):
    """f(x) = 1/(K x^{1/2} + γ x^{-1/2})  (with α=K, s=1/2, β=γ, t=-1/2);
    generally 1/(K (x+σ)^{1/2} + γ (x+σ)^t) — Eq.(9)'s S_Γ = K L^{1/2} + γ L^t with
    L = -Δ_Γ + σ I_Γ, as a function of the eigenvalue x of the pair (A_Γ, M_Γ)."""
    x = np.asarray(x, dtype=np.float64) + sigma
    return 1.0 / (K * np.sqrt(x) + gamma * x ** t)


def r_eval(x, c0: float, poles, residues):
    """r(x) = c0 + Σ_k c_k / (x - p_k)  — the scalar of Eq.(8) in the eigenbasis."""
    x = np.asarray(x, dtype=np.float64)
    out = np.full_like(x, c0)
    for p, c in zip(poles, residues):
        out = out + c / (x - p)
    return out


def ra_rel_error(c0, poles, residues, K, gamma, xs, t: float = -0.5, sigma: float = 0.0) -> float:
    """max_x |r(x)/f(x) - 1| over the points xs (pointwise relative error, reading A10)."""
    xs = np.asarray(xs, dtype=np.float64)
    return float(np.max(np.abs(r_eval(xs, c0, poles, residues) / f_target(xs, K, gamma, t, sigma) - 1.0)))


def cancellation_factor(c0, poles, residues, K, gamma, xs, t: float = -0.5, sigma: float = 0.0) -> float:
    """κ_c = max_x (|c0| + Σ|c_k/(x-p_k)|) / f(x)   (reading A11; f of `f_target`)."""
    xs = np.asarray(xs, dtype=np.float64)
    acc = np.full_like(xs, abs(c0))
    for p, c in zip(poles, residues):
        acc += np.abs(c / (xs - p))
    return float(np.max(acc / f_target(xs, K, gamma, t, sigma)))


def _to_band(T: np.ndarray) -> np.ndarray:
    """Upper-band storage of a symmetric tridiagonal matrix for solveh_banded."""
    n = T.shape[0]
    ab = np.zeros((2, n))
    ab[1] = np.diag(T)
    ab[0, 1:] = np.diag(T, 1)
    return ab


def apply_ra(A: np.ndarray, M: np.ndarray, c0, poles, residues, B: np.ndarray) -> np.ndarray:
    """Z = c0 M^-1 B + Σ_k c_k (A - p_k M)^-1 B, summed in the fixed order k = 0 (mass), 1..m.

    1D Γ (tridiagonal pair): LAPACK banded Cholesky (scipy.linalg.solveh_banded);
    2D Γ (face pair, dense or scipy.sparse): sparse direct LU (scipy.sparse.linalg.splu).
    B is (n_Γ, C).
    """
    B = np.asarray(B, dtype=np.float64)
    if sp.issparse(A) or sp.issparse(M):
        # sparse pair (the config-4 face, n_Γ = 16129): sparse direct LU per shifted matrix
        A, M = sp.csc_matrix(A), sp.csc_matrix(M)
        def solve(T, X):
            return spla.splu(sp.csc_matrix(T)).solve(X)
    else:
        tridiag = np.count_nonzero(np.triu(A, 2)) == 0 and np.count_nonzero(np.triu(M, 2)) == 0
        def solve(T, X):
            if tridiag:
                return sla.solveh_banded(_to_band(T), X, lower=False)
            return spla.splu(sp.csc_matrix(T)).solve(X)
    Z = np.zeros_like(B)
    if c0 != 0.0:
        Z = Z + c0 * solve(M, B)
    for p, c in zip(poles, residues):
        Z = Z + c * solve(A - p * M, B)
    return Z


def apply_ra_banded_tri(a_d, a_o, m_d, m_o, c0, poles, residues, B):
    """`apply_ra` for a tridiagonal pair given by its diagonals (no dense matrices)."""
    B = np.asarray(B, dtype=np.float64)
    def solve(d, o, X):
        ab = np.zeros((2, d.size)); ab[1] = d; ab[0, 1:] = o
        return sla.solveh_banded(ab, X, lower=False)
    Z = np.zeros_like(B)
    if c0 != 0.0:
        Z = Z + c0 * solve(m_d, m_o, B)
    for p, c in zip(poles, residues):
        Z = Z + c * solve(a_d - p * m_d, a_o - p * m_o, B)
    return Z


def apply_ra_eigen(gevp, c0, poles, residues, B: np.ndarray) -> np.ndarray:
    """Eigen form U diag(r(λ)) U^T B of the same operator: (A - pM)^-1 = U diag(1/(λ-p)) U^T."""
    return gevp.apply_function(r_eval(gevp.lam, c0, poles, residues), B)


def apply_exact_precond(gevp, K: float, gamma: float, B: np.ndarray, t: float = -0.5,
                        sigma: float = 0.0) -> np.ndarray:
    """Exact S_Γ^-1 B = U diag(1/(K λ^{1/2} + γ λ^{-1/2})) U^T B  (Eq.(6)/(7)); generally
    S_Γ = K L^{1/2} + γ L^t with L = A + σM (Eq.(9))."""
    return gevp.apply_sum_inverse([(K, 0.5), (gamma, t)], B, sigma)
