"""Steklov-Poincaré (Schur complement) operator of the bulk stiffness (oracle; test infra only).

PAPER.md:104-122 (Eq.(4)): with V = V0 ⊕ VΓ the operator has blocks
[A^00 A^0i; A^i0 A^ii]; S_Γ is "spectrally equivalent to the DD Schur
complement/Steklov-Poincaré operator"  S = A^ii - A^i0 (A^00)^-1 A^0i.
PAPER.md:229-230: "(A^00)^-1 ... computed exactly by LU factorization".

Three tiers, each the same plain definition:
  * `schur_bruteforce`  — dense Cholesky of A^00 on the element-assembled matrix.
  * `schur_layers`      — block elimination of the layer-tridiagonal A^00 from the far
                          layer (x = 1 - h) toward Γ: D <- A_ll - A_l,l+1 D^-1 A_l+1,l.
  * `schur_modes_2d` / `schur_modes_3d` — the same layer elimination done one sine mode at a
    time (each layer block is diagonal in the sine basis along Γ), i.e. the scalar
    continued fraction d <- (layer diagonal) - (coupling)^2 / d.  This is what lets the
    oracle reach full config sizes; it is pinned to the two dense tiers in tests.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

from .fem import BulkProblem


def schur_of(A: np.ndarray, gamma_idx) -> np.ndarray:
    """Plain definition on a dense SPD matrix: S = A_ΓΓ - A_ΓI A_II^-1 A_IΓ (Cholesky of A_II)."""
    A = np.asarray(A, dtype=np.float64)
    g = np.asarray(gamma_idx)
    I = np.setdiff1d(np.arange(A.shape[0]), g)
    Agg, AgI, AII = A[np.ix_(g, g)], A[np.ix_(g, I)], A[np.ix_(I, I)]
    if I.size == 0:
        return Agg.copy()
    X = sla.cho_solve(sla.cho_factor(AII), AgI.T)
    return Agg - AgI @ X


def schur_bruteforce(dim: int, N: int) -> np.ndarray:
    """Dense S_unit = A^ii - A^i0 (A^00)^-1 A^0i of the element-assembled P1 stiffness (K = 1)."""
    P = BulkProblem(dim, N)
    S = schur_of(P.A.toarray(), np.arange(P.n_gamma))
    return 0.5 * (S + S.T)


def schur_layers(dim: int, N: int) -> np.ndarray:
    """Dense layer-by-layer elimination of the assembled stiffness (K = 1).

    Free nodes are ordered layer-major (layer l = x-index), each layer holding n_Γ nodes
    in Γ order.  Asserts that the assembled matrix only couples adjacent layers.
    """
    P = BulkProblem(dim, N)
    A = P.A.tocsr()
    g = P.n_gamma
    L = N                     # layers 0 (Γ) .. N-1
    assert A.shape[0] == g * L
    def blk(a, b):
        return A[a * g:(a + 1) * g, b * g:(b + 1) * g]
    # the matrix must be block tridiagonal in layers
    coo = A.tocoo()
    assert np.all(np.abs(coo.row // g - coo.col // g) <= 1), "non-adjacent layer coupling"
    D = blk(L - 1, L - 1).toarray()
    for l in range(L - 2, -1, -1):
        C = blk(l, l + 1).toarray()                     # coupling layer l -> l+1
        Y = sla.cho_solve(sla.cho_factor(D), C.T)      # D^-1 A_l+1,l
        D = blk(l, l).toarray() - C @ Y
    return 0.5 * (D + D.T)


# ----------------------------------------------------------------- mode-by-mode (2D, 3D)
def _cos_theta(n: int) -> np.ndarray:
    """cos(k pi / (n+1)), k = 1..n, through sin^2 to avoid cancellation."""
    k = np.arange(1, n + 1)
    return 1.0 - 2.0 * np.sin(0.5 * np.pi * k / (n + 1)) ** 2


def schur_modes_2d(N: int) -> np.ndarray:
    """Eigenvalues s_b of S_unit in the orthonormal sine basis along Γ (2D, K = 1).

    Stiffness blocks of the Freudenthal P1 mesh in sine mode b (checked against element
    assembly in tests): interior layer diagonal 4 - 2cos θ_b = 2 + σ_b, inter-layer coupling -1,
    Γ-row diagonal 2 - cos θ_b = 1 + σ_b/2.  Layer elimination from the far layer:
    d <- (2 + σ_b) - 1/d, starting at d = 2 + σ_b, N-2 times; s_b = (1 + σ_b/2) - 1/d.
    The recursion is carried for e = d - 1 (e <- σ_b + e/(1+e), s_b = σ_b/2 + e/(1+e)), the same
    elimination without the cancellation d ≈ 1 + √σ_b causes for the low modes (DESIGN.md
    reading A26: the plain form loses 4.7e-10 in s_1 at N = 8192); σ_b = 4 sin²(θ_b/2) (A18).
    """
    n = N - 1
    k = np.arange(1, n + 1)
    sig = 4.0 * np.sin(0.5 * np.pi * k / (n + 1)) ** 2
    e = 1.0 + sig
    for _ in range(N - 2):
        e = sig + e / (1.0 + e)
    return 0.5 * sig + e / (1.0 + e)


def schur_modes_3d(N: int) -> np.ndarray:
    """Eigenvalues s_(b,c) of S_unit in the 2D sine basis of the Γ face (3D, K = 1), shape (n, n).

    Kuhn P1 stiffness in mode (b,c): interior layer diagonal h(6 - 2cosθ_b - 2cosθ_c),
    coupling -h, Γ-row diagonal h(3 - cosθ_b - cosθ_c).
    """
    n = N - 1
    h = 1.0 / N
    c = _cos_theta(n)
    cb, cc = np.meshgrid(c, c, indexing="ij")
    diag = h * (6.0 - 2.0 * cb - 2.0 * cc)
    d = diag.copy()
    for _ in range(N - 2):
        d = diag - h * h / d
    return h * (3.0 - cb - cc) - h * h / d


def dst_ortho(X: np.ndarray, axis: int = 0) -> np.ndarray:
    """Orthonormal DST-I (a library FFT routine; symmetric and involutory)."""
    from scipy.fft import dst
    return dst(X, type=1, norm="ortho", axis=axis)
