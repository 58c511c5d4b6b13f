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


@pytest.mark.parametrize("N", [12, 33])
def test_bulk_pcg_parity(lib, N):
    """The paper's protocol (dd_bulk_pcg_solve): PCG on the bulk system with the Eq.(5) DD
    preconditioner — iterations ±1 and solution 1e-8 against the oracle's bulk PCG (sparse LU
    A^00, same RA), solution against the direct bulk solve."""
    params = [(1.0, 1e2), (1e-3, 1.0)]
    ras = fit_all(N, params, 12)
    Bs = obulk.BulkSystem(2, N)
    from oracle import pcg as opcg
    from oracle import problem as oprob
    D = oprob.DenseProblem(2, N)
    C = 4
    Bp = np.random.default_rng(N + 1).uniform(-1, 1, (C, Bs.A.shape[0]))
    colp = np.arange(C) % 2
    S = lib.Solver(2, N, params, ras, max_cols=C)
    try:
        res = S.bulk_pcg_solve(torch.as_tensor(Bp, device="cuda"), colp)
        x = res.x.cpu().numpy()
        for c in range(C):
            K, g = params[colp[c]]; ra = ras[colp[c]]
            P = lambda w: D.apply_P_ra(ra.c0, ra.poles, ra.residues, w)
            bo = Bs.from_product(Bp[c])
            xo, it, *_ = opcg.pcg(lambda v: Bs.apply(K, g, v), lambda v: Bs.dd_precond(K, P, v), bo)
            assert abs(int(res.iters[c]) - it) <= 1, (c, res.iters[c], it)
            assert np.linalg.norm(x[c] - Bs.to_product(xo)) <= 1e-8 * np.linalg.norm(xo)
            xd = Bs.solve(K, g, bo)
            assert np.linalg.norm(Bs.from_product(x[c]) - xd) <= 1e-8 * np.linalg.norm(xd)
        assert np.all(res.rel_res <= 1e-10)
    finally:
        S.close()


def test_bulk_pcg_matches_schur_pcg_iterations(lib):
    """N = 256: with the exact leading block the bulk PCG's preconditioned spectrum is
    {1} ∪ spec(P S), so it needs at most the interface PCG's iteration count (+1); it can stop
    earlier because its η0 = sqrt(r0·𝓑r0) also carries the interior component, which the first
    step removes (measured: 14 vs 16).  Its solution equals dd_bulk_solve's to 1e-8."""
    N = 256
    params = [(1.0, 1e4)]
    ras = fit_all(N, params, 16)
    n = N - 1
    C = 3
    Bp = np.random.default_rng(17).uniform(-1, 1, (C, n * n + n))
    S = lib.Solver(2, N, params, ras, max_cols=C)
    try:
        a = S.bulk_pcg_solve(torch.as_tensor(Bp, device="cuda"), [0] * C)
        b = S.bulk_solve(torch.as_tensor(Bp, device="cuda"), [0] * C)
        assert np.all(a.iters <= b.iters + 1) and np.all(a.iters >= b.iters - 4), (a.iters, b.iters)
        xa, xb = a.x.cpu().numpy(), b.x.cpu().numpy()
        assert np.max(np.linalg.norm(xa - xb, axis=1) / np.linalg.norm(xb, axis=1)) <= 1e-8
    finally:
        S.close()


@pytest.mark.parametrize("N", [6, 9, 13])
def test_bulk_solve_3d_parity(lib, N):
    """3D full DD solve (block elimination, (A^00)^-1 by fast diagonalisation along x, y, z) against
    the oracle's direct solve of the assembled Kuhn-mesh bulk system with the dense F block."""
    params = [(1.0, 1e2)]
    lo, hi = rafit.interval_face(N)
    ras = [rafit.fit_ra(K, g, lo, hi, 12) for K, g in params]
    Bs = obulk.BulkSystem(3, N)
    C = 3
    Bp = np.random.default_rng(N).uniform(-1, 1, (C, Bs.A.shape[0]))     # product layout [interior, Γ]
    S = lib.Solver(3, N, params, ras, max_cols=C)
    try:
        res = S.bulk_solve(torch.as_tensor(Bp, device="cuda"), [0] * C)
        x = res.x.cpu().numpy()
        K, g = params[0]
        for c in range(C):
            xo = Bs.to_product(Bs.solve(K, g, Bs.from_product(Bp[c])))
            assert np.linalg.norm(x[c] - xo) <= 1e-8 * np.linalg.norm(xo), (c, np.linalg.norm(x[c] - xo) / np.linalg.norm(xo))
            r = Bs.apply(K, g, Bs.from_product(x[c])) - Bs.from_product(Bp[c])
            assert np.linalg.norm(r) <= 1e-8 * np.linalg.norm(Bp[c])
        assert np.all(res.rel_res <= 1e-10)
    finally:
        S.close()


def test_bulk_solve_3d_medium(lib):
    """N = 32 (29 791 interior + 961 Γ unknowns): sparse-LU oracle on one column, residual on all."""
    N = 32
    params = [(1.0, 1e4)]
    lo, hi = rafit.interval_face(N)
    ras = [rafit.fit_ra(K, g, lo, hi, 16) for K, g in params]
    Bs = obulk.BulkSystem(3, N)
    C = 2
    Bp = np.random.default_rng(11).uniform(-1, 1, (C, Bs.A.shape[0]))
    S = lib.Solver(3, N, params, ras, max_cols=C)
    try:
        res = S.bulk_solve(torch.as_tensor(Bp, device="cuda"), [0] * C)
        x = res.x.cpu().numpy()
        K, g = params[0]
        xo = Bs.to_product(Bs.solve(K, g, Bs.from_product(Bp[0])))
        assert np.linalg.norm(x[0] - xo) <= 1e-8 * np.linalg.norm(xo)
        for c in range(C):
            r = Bs.apply(K, g, Bs.from_product(x[c])) - Bs.from_product(Bp[c])
            assert np.linalg.norm(r) <= 1e-8 * np.linalg.norm(Bp[c])
    finally:
        S.close()


@pytest.mark.parametrize("N", [6, 9])
def test_bulk_pcg_3d_parity(lib, N):
    """The paper's protocol in 3D (dd_bulk_pcg_solve on a 3D handle): PCG on the Kuhn-mesh bulk system
    with the Eq.(5) preconditioner (exact leading block by fast diagonalisation, S_Γ^-1 by the RA with
    the face systems solved by inner CG to 1e-13, reading A12) — iterations ±1 and the solution against
    the oracle's bulk PCG with the same RA (sparse-direct face solves) and against the direct solve."""
    from oracle import pcg as opcg
    from oracle import problem as oprob
    params = [(1.0, 1e2)]
    lo, hi = rafit.interval_face(N)
    ras = [rafit.fit_ra(K, g, lo, hi, 12) for K, g in params]
    Bs = obulk.BulkSystem(3, N)
    D = oprob.DenseProblem(3, N)
    C = 2
    Bp = np.random.default_rng(N + 3).uniform(-1, 1, (C, Bs.A.shape[0]))
    S = lib.Solver(3, N, params, ras, max_cols=C)
    try:
        res = S.bulk_pcg_solve(torch.as_tensor(Bp, device="cuda"), [0] * C)
        x = res.x.cpu().numpy()
        K, g = params[0]; ra = ras[0]
        P = lambda w: D.apply_P_ra(ra.c0, ra.poles, ra.residues, w)
        for c in range(C):
            bo = Bs.from_product(Bp[c])
            xo, it, *_ = opcg.pcg(lambda v: Bs.apply(K, g, v), lambda v: Bs.dd_precond(K, P, v), bo)
            assert abs(int(res.iters[c]) - it) <= 1, (c, res.iters[c], it)
            assert np.linalg.norm(x[c] - Bs.to_product(xo)) <= 1e-8 * np.linalg.norm(xo)
            xd = Bs.solve(K, g, bo)
            assert np.linalg.norm(Bs.from_product(x[c]) - xd) <= 1e-8 * np.linalg.norm(xd)
        assert np.all(res.rel_res <= 1e-10)
    finally:
        S.close()


def test_bulk_pcg_3d_long_columns(lib):
    """N = 65 (266 240 bulk unknowns per column, 3 columns): the bulk PCG's vector steps take the
    many-CTAs-per-column path (deterministic per-CTA partial dots); its solution equals the
    block-elimination bulk solve's to 1e-8 and it needs at most the interface PCG's iterations + 1."""
    N = 65
    params = [(1.0, 1e4)]
    lo, hi = rafit.interval_face(N)
    ras = [rafit.fit_ra(K, g, lo, hi, 16) for K, g in params]
    n = N - 1
    C = 3
    Bp = np.random.default_rng(21).uniform(-1, 1, (C, n ** 3 + n * n))
    S = lib.Solver(3, N, params, ras, max_cols=C)
    try:
        a = S.bulk_pcg_solve(torch.as_tensor(Bp, device="cuda"), [0] * C)
        b = S.bulk_solve(torch.as_tensor(Bp, device="cuda"), [0] * C)
        assert np.all(a.iters <= b.iters + 1) and np.all(a.iters >= b.iters - 4), (a.iters, b.iters)
        xa, xb = a.x.cpu().numpy(), b.x.cpu().numpy()
        assert np.max(np.linalg.norm(xa - xb, axis=1) / np.linalg.norm(xb, axis=1)) <= 1e-8
        a2 = S.bulk_pcg_solve(torch.as_tensor(Bp, device="cuda"), [0] * C)
        assert np.array_equal(a2.x.cpu().numpy(), xa)          # deterministic reductions
    finally:
        S.close()


@pytest.mark.parametrize("dim,N", [(2, 24), (3, 8)])
def test_bulk_pcg_ra_operator(lib, dim, N):
    """Remark 1's experiment (Fig. 4 left in 3D): bulk PCG with the Eq.(5)
    preconditioner where BOTH the operator's fractional term and S_Γ^-1 are evaluated by RA
    (dd_frac mode "ra") — against the oracle's direct solve of the bulk system whose dense block
    is the RA-evaluated F = M r_F(L) M (oracle DenseProblem(frac_ra)), and iterations ±1 against
    the oracle's bulk PCG with the same two RAs."""
    from oracle import pcg as opcg
    from oracle import problem as oprob
    params = [(1.0, 1e2)]
    lo, hi = rafit.interval_1d(N) if dim == 2 else rafit.interval_face(N)
    ras = [rafit.fit_ra(K, g, lo, hi, 12) for K, g in params]
    fr = rafit.fit_power(-0.5, lo, hi, 16, 0.0)
    Bs = obulk.BulkSystem(dim, N)
    D = oprob.DenseProblem(dim, N, frac_ra=(fr.c0, fr.poles, fr.residues))
    Bs.F = D.F                                                 # the bulk system with the RA-evaluated block
    C = 2
    Bp = np.random.default_rng(N + 5).uniform(-1, 1, (C, Bs.A.shape[0]))
    S = lib.Solver(dim, N, params, ras, max_cols=C, frac=lib.Frac(mode="ra", fra=fr))
    try:
        res = S.bulk_pcg_solve(torch.as_tensor(Bp, device="cuda"), [0] * C)
        x = res.x.cpu().numpy()
        K, g = params[0]; ra = ras[0]
        P = lambda w: D.apply_P_ra(ra.c0, ra.poles, ra.residues, w)
        for c in range(C):
            bo = Bs.from_product(Bp[c])
            xd = Bs.solve(K, g, bo)
            assert np.linalg.norm(Bs.from_product(x[c]) - xd) <= 1e-8 * np.linalg.norm(xd)
            xo, it, *_ = opcg.pcg(lambda v: Bs.apply(K, g, v), lambda v: Bs.dd_precond(K, P, v), bo)
            assert abs(int(res.iters[c]) - it) <= 1, (c, res.iters[c], it)
        assert np.all(res.rel_res <= 1e-10)
    finally:
        S.close()
