"""Preconditioned conjugate gradients (oracle; test infra only).

PAPER.md:225-232 (§3): "the PCG solver is always started from 0 initial vector and
terminates upon reducing the preconditioned residual norm by factor 10^10."
Readings: A1 η = sqrt(r·z) (norm_kind 0) or ||z||_2 (norm_kind 1);
A2 iteration count = number of operator applications after which the criterion first
holds, reference η0 at iteration 0 with r0 = b; A19 p·Ap <= 0 or r·z < 0 -> not SPD;
A14 columns freeze individually on convergence.
"""
from __future__ import annotations

import numpy as np


class NotSPD(RuntimeError):
    pass


def _eta(r, z, norm_kind):
    if norm_kind == 0:
        rho = float(r @ z)
        if rho < 0:
            raise NotSPD("r.z < 0: preconditioner not SPD")
        return np.sqrt(rho)
    return float(np.linalg.norm(z))


def pcg(apply_A, apply_B, b: np.ndarray, rtol: float = 1e-10, maxit: int = 500, norm_kind: int = 0):
    """Single right-hand side.  Returns (x, iters, rel_res, hist, converged)."""
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    r = b.copy()
    z = apply_B(r)
    rho = float(r @ z)
    eta0 = _eta(r, z, norm_kind)
    hist = [eta0]
    if eta0 == 0.0:
        return x, 0, 0.0, hist, True
    p = z.copy()
    for k in range(1, maxit + 1):
        q = apply_A(p)
        pi = float(p @ q)
        if pi <= 0.0:
            raise NotSPD("p.Ap <= 0")
        alpha = rho / pi
        x = x + alpha * p
        r = r - alpha * q
        z = apply_B(r)
        rho_new = float(r @ z)
        eta = _eta(r, z, norm_kind)
        hist.append(eta)
        if eta <= rtol * eta0:
            return x, k, eta / eta0, hist, True
        p = z + (rho_new / rho) * p
        rho = rho_new
    return x, maxit, hist[-1] / eta0, hist, False


def pcg_batch(apply_A_cols, apply_B_cols, Bm: np.ndarray, rtol=1e-10, maxit=500, norm_kind=0):
    """Column-wise PCG on a batch Bm (n, C); each column follows `pcg` exactly and freezes
    on convergence (A14).  apply_*_cols(X, cols) applies the operator of the listed
    columns (each column may have its own parameter set).
    Returns (X, iters[C], rel_res[C], hist_col0)."""
    Bm = np.asarray(Bm, dtype=np.float64)
    n, C = Bm.shape
    X = np.zeros_like(Bm); R = Bm.copy()
    allc = np.arange(C)
    Z = apply_B_cols(R, allc)
    rho = np.einsum("ij,ij->j", R, Z)
    if norm_kind == 0:
        if np.any(rho < 0):
            raise NotSPD("r.z < 0")
        eta0 = np.sqrt(rho)
    else:
        eta0 = np.linalg.norm(Z, axis=0)
    iters = np.zeros(C, dtype=np.int64); rel = np.zeros(C)
    active = eta0 > 0.0
    hist = [float(eta0[0])] if C else []
    P = Z.copy()
    for k in range(1, maxit + 1):
        cols = np.nonzero(active)[0]
        if cols.size == 0:
            break
        Q = apply_A_cols(P[:, cols], cols)
        pi = np.einsum("ij,ij->j", P[:, cols], Q)
        if np.any(pi <= 0):
            raise NotSPD("p.Ap <= 0")
        alpha = rho[cols] / pi
        X[:, cols] += alpha * P[:, cols]
        R[:, cols] -= alpha * Q
        Zc = apply_B_cols(R[:, cols], cols)
        rho_new = np.einsum("ij,ij->j", R[:, cols], Zc)
        if norm_kind == 0:
            if np.any(rho_new < 0):
                raise NotSPD("r.z < 0")
            eta = np.sqrt(rho_new)
        else:
            eta = np.linalg.norm(Zc, axis=0)
        if active[0] and 0 in cols:
            hist.append(float(eta[np.searchsorted(cols, 0)]))
        done = eta <= rtol * eta0[cols]
        iters[cols] = k
        rel[cols] = eta / eta0[cols]
        beta = rho_new / rho[cols]
        P[:, cols] = Zc + beta * P[:, cols]
        rho[cols] = rho_new
        active[cols[done]] = False
    return X, iters, rel, hist
