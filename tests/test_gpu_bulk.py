"""Full DD solve on bulk right-hand sides (dd_bulk_solve) against the
oracle's direct solve of the assembled bulk system 𝒜 = K A_h + γ T^T L^t T (oracle/bulk.py).
Needs a B200 (-m gpu).  Bar: the interface PCG runs to rtol 1e-10, so solutions agree to 1e-8
relative (north star); the bulk residual ||𝒜x - b|| <= 1e-8 ||b||.
"""
import numpy as np
import pytest

from helpers import fit_all
from oracle import bulk as obulk
from paper_2211_15308_b200 import rafit

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2211_15308_b200 import binding
    binding.load()
    return binding


@pytest.mark.parametrize("N,t,sigma", [(8, -0.5, 0.0), (12, -0.5, 0.0), (24, 0.25, 1.0), (33, -0.5, 0.0)])
def test_bulk_solve_parity_small(lib, N, t, sigma):
    params = [(1.0, 1e2), (1e-3, 1.0)]
    lo, hi = rafit.interval_1d(N)
    ras = [rafit.fit_ra(K, g, lo, hi, 12, t=t, sigma=sigma) for K, g in params]
    Bs = obulk.BulkSystem(2, N, t=t, sigma=sigma)
    C = 4
    rng = np.random.default_rng(N)
    Bp = rng.uniform(-1, 1, (C, Bs.A.shape[0]))          # product layout [interior, Γ]
    colp = np.arange(C) % 2
    S = lib.Solver(2, N, params, ras, max_cols=C, frac=lib.Frac(t=t, shifted=bool(sigma)))
    try:
        res = S.bulk_solve(torch.as_tensor(Bp, device="cuda"), colp)
        x = res.x.cpu().numpy()
        for c in range(C):
            K, g = params[colp[c]]
            xo = Bs.to_product(Bs.solve(K, g, Bs.from_product(Bp[c])))
            assert np.linalg.norm(x[c] - xo) <= 1e-8 * np.linalg.norm(xo), c
            r = Bs.apply(K, g, Bs.from_product(x[c])) - Bs.from_product(Bp[c])
            assert np.linalg.norm(r) <= 1e-8 * np.linalg.norm(Bp[c])
        assert np.all(res.rel_res <= 1e-10)
    finally:
        S.close()


def test_bulk_solve_medium(lib):
    """N = 256 (65 280 bulk unknowns): sparse-LU oracle on two columns, residual on all."""
    N = 256
    params = [(1.0, 1e4)]
    ras = fit_all(N, params, 16)
    Bs = obulk.BulkSystem(2, N)
    C = 3
    Bp = np.random.default_rng(9).uniform(-1, 1, (C, Bs.A.shape[0]))
    S = lib.Solver(2, N, params, ras, max_cols=C)
    try:
        res = S.bulk_solve(torch.as_tensor(Bp, device="cuda"), [0] * C)
        x = res.x.cpu().numpy()
        for c in range(C):
            r = Bs.apply(1.0, 1e4, Bs.from_product(x[c])) - Bs.from_product(Bp[c])
            assert np.linalg.norm(r) <= 1e-8 * np.linalg.norm(Bp[c])
        for c in range(2):
            xo = Bs.to_product(Bs.solve(1.0, 1e4, Bs.from_product(Bp[c])))
            assert np.linalg.norm(x[c] - xo) <= 1e-8 * np.linalg.norm(xo)
    finally:
        S.close()


def test_bulk_solve_interface_rhs_matches_schur_solve(lib):
    """With b_0 = 0 the bulk solve's Γ part is exactly the Schur PCG solution of b_Γ."""
    N = 200
    params = [(1.0, 1e2)]
    ras = fit_all(N, params, 14)
    n = N - 1
    C = 3
    bg = np.random.default_rng(4).uniform(-1, 1, (C, n))
    Bp = np.concatenate([np.zeros((C, n * n)), bg], axis=1)
    S = lib.Solver(2, N, params, ras, max_cols=C)
    try:
        xb = S.bulk_solve(torch.as_tensor(Bp, device="cuda"), [0] * C).x.cpu().numpy()
        xs = S.pcg_solve(torch.as_tensor(bg, device="cuda"), [0] * C).x.cpu().numpy()
        assert np.array_equal(xb[:, n * n:], xs)
    finally:
        S.close()
