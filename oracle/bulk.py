"""The full bulk problem of Eq.(2) on all free nodes (oracle; test infra only).

PAPER.md:43-45 (Eq.(2)) discretised by P1 elements with the DOF split
V = V0 ⊕ VΓ:  𝒜 = K A_h + γ T^T L_h^t T  with A_h the element-assembled
stiffness on the free nodes and the fractional term acting on the Γ block (T restricted to Γ is
the identity on the Γ DOFs, reading A6).  The oracle solves 𝒜 x = b directly — the
plain definition the DD solver (block elimination, Eq.(5) with exact blocks) must reproduce.

Product layout (include/dd_api.h dd_bulk_solve): per column [interior nodes x-major, Γ nodes];
BulkProblem's order is [Γ nodes, interior nodes (i-major)] — `to_product` / `from_product`
convert between the two.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import fem, spectral


class BulkSystem:
    def __init__(self, dim: int, N: int, t: float = -0.5, sigma: float = 0.0):
        self.dim, self.N = dim, N
        P = fem.BulkProblem(dim, N)
        self.A = P.A.tocsr()                        # [Γ, interior]
        self.g, self.ni = P.n_gamma, P.n_int
        A_g, M_g = fem.trace_pair(dim, N)
        self.F = spectral.GEVP(A_g, M_g).power(t, sigma)

    def matrix(self, K: float, gamma: float) -> sp.csr_matrix:
        """𝒜 = K A_h + γ T^T F T (sparse, with the dense Γ block)."""
        g = self.g
        rows, cols = np.meshgrid(np.arange(g), np.arange(g), indexing="ij")
        Fs = sp.csr_matrix((gamma * self.F.ravel(), (rows.ravel(), cols.ravel())), shape=self.A.shape)
        return (K * self.A + Fs).tocsc()

    def apply(self, K, gamma, x):
        """𝒜 x for x in BulkProblem order ([Γ, interior])."""
        y = K * (self.A @ x)
        y[: self.g] += gamma * (self.F @ x[: self.g])
        return y

    def solve(self, K, gamma, b):
        """x = 𝒜^-1 b: dense Cholesky for small systems, sparse LU (SuperLU) otherwise."""
        if self.A.shape[0] <= 3000:
            M = self.matrix(K, gamma).toarray()
            return sla.cho_solve(sla.cho_factor(M), b)
        return spla.spsolve(self.matrix(K, gamma), b)

    # layouts
    def to_product(self, x):
        """[Γ, interior] -> [interior, Γ] (per column along the last axis)."""
        x = np.asarray(x)
        return np.concatenate([x[..., self.g:], x[..., : self.g]], axis=-1)

    def from_product(self, y):
        y = np.asarray(y)
        return np.concatenate([y[..., self.ni:], y[..., : self.ni]], axis=-1)

    # ----------------------------------------------------------------------- Eq.(5)
    def _lu00(self, K):
        key = float(K)
        if getattr(self, "_lu_key", None) != key:
            A = (K * self.A).tocsc()
            g = self.g
            self._lu = spla.splu(A[g:, g:].tocsc())
            self._A0i = A[g:, :g].tocsr()
            self._Ai0 = A[:g, g:].tocsr()
            self._lu_key = key
        return self._lu, self._A0i, self._Ai0

    def dd_precond(self, K, apply_SG_inv, r):
        """𝓑 r of Eq.(5), in BulkProblem order [Γ, interior]:
        y0 = (A^00)^-1 r0,  zΓ = S_Γ^-1 (rΓ - A^{i0} y0),  z0 = (A^00)^-1 (r0 - A^{0i} zΓ)
        — the three factors applied right to left; (A^00)^-1 exact (sparse LU)."""
        lu, A0i, Ai0 = self._lu00(K)
        g = self.g
        r = np.asarray(r, dtype=np.float64)
        y0 = lu.solve(r[g:])
        zg = apply_SG_inv(r[:g] - Ai0 @ y0)
        z0 = lu.solve(r[g:] - A0i @ zg)
        return np.concatenate([zg, z0])
