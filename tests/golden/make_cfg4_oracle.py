"""Write tests/golden/cfg4_oracle.npz: the CPU oracle's results on BASELINE.json config 4
(3D, N = 128, Γ = the face {x=0}, n_Γ = 127² = 16129, K = 1, μ⁻¹ = 1e4, 20 poles, 8 seeded RHS).

TEST INFRASTRUCTURE (run by hand, ~10 min and ~16 GB of host memory; the output is committed so
the GPU parity test does not redo the 16129² generalised eigensolve):

    python tests/golden/make_cfg4_oracle.py

Every stored value comes from `oracle/` only:
  * the face pair (A_Γ, M_Γ): `fem.trace_pair_face` (P1 element integrals on the trace mesh;
    pinned equal to the bulk Kuhn-mesh trace `fem.trace_pair(3, N)` in test_oracle_pins);
  * F = (MU) Λ^{-1/2} (MU)^T: `spectral.GEVP` = scipy.linalg.eigh(A_Γ, M_Γ) (Eq.(7));
  * S_unit: `schur.schur_modes_3d` in the face's sine basis (the layer elimination mode by mode,
    pinned to dense Cholesky elimination and dense layer elimination at small N);
  * P_RA: `ra.apply_ra` (sparse direct LU per shifted matrix, Eq.(8)) and `ra.apply_ra_eigen`;
  * PCG: `pcg.pcg_batch`, norm_kind 0 and 1.
Inputs (not method arithmetic): the seeded RHS of `paper_2211_15308_b200.inputs` and the RA
fit's poles / residues (`rafit.fit_ra` on the oracle's own spectral interval) — setup data passed
to both sides, stored here so the GPU test feeds the identical fit to the library.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import fem, pcg, ra, schur, spectral  # noqa: E402
from paper_2211_15308_b200 import inputs, rafit  # noqa: E402  (input generation only)

N, K, GAMMA, M_POLES, NRHS = int(os.environ.get("CFG4_N", "128")), 1.0, 1e4, 20, 8
OUT = os.environ.get("CFG4_OUT", os.path.join(os.path.dirname(os.path.abspath(__file__)), "cfg4_oracle.npz"))


def main():
    n = N - 1
    ng = n * n
    t0 = time.time()
    A, M = fem.trace_pair_face(N)
    G = spectral.GEVP(A.toarray(), M.toarray())
    t_eig = time.time() - t0
    print(f"gevp {t_eig:.0f} s", flush=True)
    lam = G.lam
    F = G.power(-0.5)
    del G.L, G.M
    fit = rafit.fit_ra(K, GAMMA, float(lam[0]), float(lam[-1]), M_POLES)
    c0, poles, res = float(fit.c0), np.asarray(fit.poles), np.asarray(fit.residues)
    xs = np.concatenate([np.geomspace(lam[0], lam[-1], 20000), lam])
    kappa_c = ra.cancellation_factor(c0, poles, res, K, GAMMA, xs)
    ra_err = ra.ra_rel_error(c0, poles, res, K, GAMMA, lam)

    s = schur.schur_modes_3d(N)

    def s_unit(X):                       # X: (n_Γ, C), j-major faces
        C = X.shape[1]
        Y = X.T.reshape(C, n, n)
        Yh = schur.dst_ortho(schur.dst_ortho(Y, axis=1), axis=2)
        Y = schur.dst_ortho(schur.dst_ortho(s[None] * Yh, axis=1), axis=2)
        return Y.reshape(C, ng).T

    def apply_S(X):
        return K * s_unit(X) + GAMMA * (F @ X)

    def apply_P(X):
        return ra.apply_ra(A, M, c0, poles, res, X)

    B, colp = inputs.batch(ng, 1, NRHS)
    Bc = B.T.copy()
    y = apply_S(Bc)
    z_par = apply_P(Bc)
    z_eig = ra.apply_ra_eigen(G, c0, poles, res, Bc)
    # self-check of Eq.(7): F M^-1 F = L^-1 = M A^-1 M on the RHS columns
    import scipy.sparse.linalg as spla
    Mlu, Alu = spla.splu(M.tocsc()), spla.splu(A.tocsc())
    lhs = F @ Mlu.solve(F @ Bc)
    rhs = M @ Alu.solve(M @ Bc)
    ident = float(np.linalg.norm(lhs - rhs) / np.linalg.norm(rhs))
    print(f"F M^-1 F = M A^-1 M: {ident:.2e}", flush=True)
    assert ident <= 1e-10

    t1 = time.time()
    X, iters, rel, hist = pcg.pcg_batch(lambda P, cols: apply_S(P), lambda R, cols: apply_P(R), Bc,
                                        rtol=1e-10, maxit=500, norm_kind=0)
    t_solve = time.time() - t1
    _, iters1, _, _ = pcg.pcg_batch(lambda P, cols: apply_S(P), lambda R, cols: apply_P(R), Bc,
                                    rtol=1e-10, maxit=500, norm_kind=1)
    print(f"pcg iters {iters.tolist()} (norm_kind 1: {iters1.tolist()}), {t_solve:.0f} s", flush=True)
    np.savez(OUT, N=N, K=K, gamma=GAMMA, c0=c0, poles=poles, residues=res, lam_min=float(lam[0]),
             lam_max=float(lam[-1]), kappa_c=kappa_c, ra_err=ra_err, y=y.T, z_par=z_par.T, z_eig=z_eig.T,
             x=X.T, iters=iters, rel=rel, hist=np.asarray(hist), iters_norm1=iters1,
             eq7_identity=ident, oracle_gevp_s=t_eig, oracle_solve_s=t_solve)
    print(f"wrote {OUT}  (total {time.time() - t0:.0f} s)")


if __name__ == "__main__":
    main()
