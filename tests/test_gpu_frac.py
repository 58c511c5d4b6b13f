"""Parity of the general fractional perturbation γ L^t, L = -Δ_Γ + σ I_Γ (dd_setup_ex / dd_frac;
Eq.(9)) with the CPU oracle.  Needs a B200: -m gpu.

Same bars as test_gpu_parity: operator 1e-10 relative ℓ2, preconditioner max(1e-10, 1e-15 κ_c)
(+ the oracle's own banded-vs-eigen discrepancy), solutions 1e-8, iterations ±1.
"""
import numpy as np
import pytest

from helpers import check_precond, rel_l2_cols
from oracle import pcg as opcg
from oracle import problem as oprob
from paper_2211_15308_b200 import rafit

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2211_15308_b200 import binding
    binding.load()
    return binding


def _cols(B):
    return torch.as_tensor(B, device="cuda")


def _fits(N, params, m, t, sigma, dim=2):
    lo, hi = rafit.interval_1d(N) if dim == 2 else rafit.interval_face(N)
    return [rafit.fit_ra(K, g, lo, hi, m, t=t, sigma=sigma) for K, g in params]


CASES = [(8, -0.75, 0.0), (33, 0.25, 1.0), (200, 0.75, 0.0), (200, -0.25, 1.0), (64, -0.5, 1.0)]


@pytest.mark.parametrize("N,t,sigma", CASES, ids=lambda v: str(v))
def test_general_t_parity_dense(lib, N, t, sigma):
    params = [(1.0, 1e2), (1e-3, 1.0)]
    m = 14
    ras = _fits(N, params, m, t, sigma)
    D = oprob.DenseProblem(2, N, t=t, sigma=sigma)
    C = 6
    B = np.random.default_rng(N).uniform(-1, 1, (C, N - 1))
    colp = np.arange(C) % 2
    S = lib.Solver(2, N, params, ras, max_cols=C, frac=lib.Frac(t=t, shifted=bool(sigma)))
    try:
        y = S.apply_schur(_cols(B), colp).cpu().numpy()
        ref = np.stack([D.apply_S(*params[colp[c]], B[c]) for c in range(C)])
        assert rel_l2_cols(y, ref) <= 1e-10
        z = S.apply_precond(_cols(B), colp).cpu().numpy()
        ra = lambda c: ras[colp[c]]
        zb = np.stack([D.apply_P_ra(ra(c).c0, ra(c).poles, ra(c).residues, B[c]) for c in range(C)])
        ze = np.stack([D.apply_P_ra_eigen(ra(c).c0, ra(c).poles, ra(c).residues, B[c]) for c in range(C)])
        check_precond(z, zb, ze, ras)
        res = S.pcg_solve(_cols(B), colp)
        x = res.x.cpu().numpy()
        for c in range(C):
            K, g = params[colp[c]]
            xo, it, rel, hist, conv = opcg.pcg(lambda v: D.apply_S(K, g, v),
                                               lambda v: D.apply_P_ra(ra(c).c0, ra(c).poles, ra(c).residues, v), B[c])
            assert conv and abs(int(res.iters[c]) - it) <= 1, (c, res.iters[c], it)
            assert np.linalg.norm(x[c] - xo) <= 1e-8 * np.linalg.norm(xo)
            # the solve answers the paper's system: S x = b to the PCG tolerance
            assert np.linalg.norm(D.apply_S(K, g, x[c]) - B[c]) <= 1e-6 * np.linalg.norm(B[c])
    finally:
        S.close()


@pytest.mark.parametrize("t,sigma", [(0.25, 1.0), (-0.75, 0.0)])
def test_general_t_full_size(lib, t, sigma):
    """Config-2 size (N = 1024) against the oracle's mode tier: every (t, γ) iteration count ±1."""
    N = 1024
    params = [(1.0, 1.0), (1.0, 1e4)]
    ras = _fits(N, params, 16, t, sigma)
    Mo = oprob.ModeProblem2D(N, t=t, sigma=sigma)
    C = 32
    B = np.random.default_rng(5).uniform(-1, 1, (C, N - 1))
    colp = np.arange(C) % 2
    S = lib.Solver(2, N, params, ras, max_cols=C, frac=lib.Frac(t=t, shifted=bool(sigma)))
    try:
        y = S.apply_schur(_cols(B), colp).cpu().numpy()
        ref = np.stack([Mo.apply_S(*params[colp[c]], B[c]) for c in range(C)])
        assert rel_l2_cols(y, ref) <= 1e-10
        res = S.pcg_solve(_cols(B), colp)
        x = res.x.cpu().numpy()
        for p, (K, g) in enumerate(params):
            sel = np.nonzero(colp == p)[0]
            ra = ras[p]
            X, its, rel, _ = opcg.pcg_batch(lambda V, cols: Mo.apply_S(K, g, V),
                                            lambda V, cols: Mo.apply_P_ra(ra.c0, ra.poles, ra.residues, V),
                                            B[sel].T, rtol=1e-10, maxit=500)
            assert np.all(np.abs(res.iters[sel] - its) <= 1)
            assert rel_l2_cols(x[sel], X.T) <= 1e-8
    finally:
        S.close()


def test_general_t_3d(lib):
    N, t, sigma = 8, 0.25, 1.0
    params = [(1.0, 1e2)]
    ras = _fits(N, params, 12, t, sigma, dim=3)
    D = oprob.DenseProblem(3, N, t=t, sigma=sigma)
    B = np.random.default_rng(3).uniform(-1, 1, (3, (N - 1) ** 2))
    S = lib.Solver(3, N, params, ras, max_cols=3, frac=lib.Frac(t=t, shifted=True))
    try:
        y = S.apply_schur(_cols(B), [0, 0, 0]).cpu().numpy()
        assert rel_l2_cols(y, D.apply_S(*params[0], B.T).T) <= 1e-10
        res = S.pcg_solve(_cols(B), [0, 0, 0])
        ra = ras[0]
        for c in range(3):
            xo, it, *_ = opcg.pcg(lambda v: D.apply_S(*params[0], v),
                                  lambda v: D.apply_P_ra(ra.c0, ra.poles, ra.residues, v), B[c])
            assert abs(int(res.iters[c]) - it) <= 1
            assert np.linalg.norm(res.x.cpu().numpy()[c] - xo) <= 1e-8 * np.linalg.norm(xo)
    finally:
        S.close()


def test_frac_validation(lib):
    params = [(1.0, 1.0)]
    ras = _fits(16, params, 6, -0.5, 0.0)
    for bad in (lib.Frac(t=1.0), lib.Frac(t=-1.0), lib.Frac(t=0.2, mode="bogus")):
        with pytest.raises(lib.DDError):
            lib.Solver(2, 16, params, ras, max_cols=1, frac=bad)
