"""Parity of the CUDA path (through the C ABI) with the CPU oracle.  Needs a B200: -m gpu.

Tolerances (north star, BASELINE.json): operator applications 1e-10 relative ℓ2 (precond:
max(1e-10, 1e-15 κ_c), reading A11), solutions 1e-8 relative, iteration counts ±1.
"""
import numpy as np
import pytest

from helpers import check_precond, fit_all, precond_tol, rel_l2_cols
from oracle import pcg as opcg
from oracle import problem as oprob
from paper_2211_15308_b200 import configs, inputs

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    from paper_2211_15308_b200 import binding
    binding.load()
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    return binding


def _solver(lib, N, params, ras, max_cols):
    return lib.Solver(2, N, params, ras, max_cols=max_cols, device=0)


def _cols(B):
    return torch.as_tensor(B, device="cuda")


# ------------------------------------------------------------------------- GEMM core
@pytest.mark.parametrize("M,N,K,sk", [(64, 64, 16, 1), (100, 37, 70, 1), (199, 130, 400, 3), (1023, 256, 2046, 2),
                                      (300, 5, 1000, 7), (64, 64, 16, 0), (199, 130, 400, 0), (1023, 256, 2046, 0),
                                      (2047, 100, 4094, 0), (300, 5, 1000, 0)])
def test_dgemm_core(lib, M, N, K, sk):
    rng = np.random.default_rng(M + N + K)
    A = rng.standard_normal((M, K)); B = rng.standard_normal((N, K))
    C = lib.test_dgemm(torch.as_tensor(A, device="cuda"), torch.as_tensor(B, device="cuda"), splitk=sk).cpu().numpy()
    ref = (A @ B.T).T
    assert np.abs(C - ref).max() <= 1e-13 * np.sqrt(K) * np.abs(ref).max()


# ------------------------------------------------------------------------- small / ragged parity vs dense oracle
SMALL = [
    (8, [(1.0, 1e2)], 8, 3),
    (33, [(1.0, 1.0), (1e-4, 1e6)], 10, 5),
    (200, [(1.0, 1e2), (1e-4, 1e6), (1.0, 0.0)], 14, 37),
]


@pytest.fixture(scope="module", params=SMALL, ids=lambda p: f"N{p[0]}")
def small_case(request, lib):
    N, params, m, C = request.param
    ras = fit_all(N, params, m)
    D = oprob.DenseProblem(2, N)
    S = _solver(lib, N, params, ras, max_cols=C + 3)
    rng = np.random.default_rng(N)
    B = rng.uniform(-1, 1, (C, N - 1))
    colp = np.arange(C) % len(params)
    yield N, params, ras, D, S, B, colp
    S.close()


MODES = ["grouped", "assembled", "factored"]


@pytest.mark.parametrize("mode", MODES)
def test_schur_apply_parity_small(small_case, mode):
    N, params, ras, D, S, B, colp = small_case
    S.set_schur_mode(mode)
    try:
        y = S.apply_schur(_cols(B), colp).cpu().numpy()
    finally:
        S.set_schur_mode("grouped")
    ref = np.stack([D.apply_S(*params[colp[c]], B[c]) for c in range(B.shape[0])])
    assert rel_l2_cols(y, ref) <= 1e-10


def test_precond_apply_parity_small(small_case):
    N, params, ras, D, S, B, colp = small_case
    z = S.apply_precond(_cols(B), colp).cpu().numpy()
    ra = lambda c: ras[colp[c]]
    zb = np.stack([D.apply_P_ra(ra(c).c0, ra(c).poles, ra(c).residues, B[c]) for c in range(B.shape[0])])
    ze = np.stack([D.apply_P_ra_eigen(ra(c).c0, ra(c).poles, ra(c).residues, B[c]) for c in range(B.shape[0])])
    check_precond(z, zb, ze, ras)


def test_pcg_parity_small(small_case):
    N, params, ras, D, S, B, colp = small_case
    res = S.pcg_solve(_cols(B), colp, rtol=1e-10, maxit=500, want_hist=True)
    x = res.x.cpu().numpy()
    for c in range(B.shape[0]):
        K, g = params[colp[c]]; ra = ras[colp[c]]
        xo, it, rel, hist, conv = opcg.pcg(lambda v: D.apply_S(K, g, v),
                                           lambda v: D.apply_P_ra(ra.c0, ra.poles, ra.residues, v), B[c])
        assert conv
        assert abs(int(res.iters[c]) - it) <= 1, (c, res.iters[c], it)
        assert np.linalg.norm(x[c] - xo) <= 1e-8 * np.linalg.norm(xo)
        if c == 0:
            assert len(res.hist) == res.iters[0] + 1
            assert res.hist[0] == pytest.approx(hist[0], rel=1e-12)
    assert np.all(res.rel_res <= 1e-10)


def test_determinism_and_host_api(small_case):
    N, params, ras, D, S, B, colp = small_case
    a = S.pcg_solve(_cols(B), colp).x.cpu().numpy()
    b = S.pcg_solve(_cols(B), colp).x.cpu().numpy()
    assert np.array_equal(a, b)                         # fixed reduction trees: bitwise
    h = S.pcg_solve_host(B, colp)
    assert np.array_equal(h.x, a)


def test_host_api_pinned_input(small_case):
    # dd_pcg_solve_host reads a page-locked b in place (zero copy) and stages a pageable one: same bits
    N, params, ras, D, S, B, colp = small_case
    pinned = torch.as_tensor(B).pin_memory().numpy()
    a = S.pcg_solve_host(B, colp)
    b = S.pcg_solve_host(pinned, colp)
    assert np.array_equal(a.x, b.x) and np.array_equal(a.iters, b.iters)


def test_batch_columns_match_single(small_case):
    # A14: columns freeze individually; each column reproduces its single-column run.
    N, params, ras, D, S, B, colp = small_case
    full = S.pcg_solve(_cols(B), colp)
    for c in (0, B.shape[0] - 1):
        one = S.pcg_solve(_cols(B[c:c + 1]), colp[c:c + 1])
        assert one.iters[0] == full.iters[c]
        xf = full.x.cpu().numpy()[c]; xs = one.x.cpu().numpy()[0]
        assert np.linalg.norm(xf - xs) <= 1e-12 * np.linalg.norm(xs)


# ------------------------------------------------------------------------- edge cases
def test_edge_cases(lib):
    N = 16; params = [(1.0, 1e2)]; ras = fit_all(N, params, 6)
    S = _solver(lib, N, params, ras, max_cols=4)
    try:
        # ncols = 0 is a no-op
        e = torch.empty(0, N - 1, dtype=torch.float64, device="cuda")
        S.apply_schur(e, np.zeros(0, dtype=np.int32)); S.apply_precond(e, np.zeros(0, dtype=np.int32))
        # zero right-hand side: 0 iterations, x = 0
        B = np.zeros((2, N - 1)); B[1] = 1.0
        r = S.pcg_solve(_cols(B), [0, 0])
        assert r.iters[0] == 0 and np.all(r.x.cpu().numpy()[0] == 0) and r.iters[1] > 0
        # maxit reached -> DD_ENOCONV (non-fatal, outputs valid)
        r = S.pcg_solve(_cols(np.ones((1, N - 1))), [0], maxit=2)
        assert r.status == lib.DD_ENOCONV and r.iters[0] == 2
        # ncols > max_cols -> DD_EINVAL
        with pytest.raises(lib.DDError):
            S.pcg_solve(_cols(np.ones((5, N - 1))), [0] * 5)
    finally:
        S.close()
    # invalid setup arguments
    class Bad:
        c0 = 0.0; poles = np.array([0.5]); residues = np.array([1.0])
    with pytest.raises(lib.DDError):
        lib.Solver(2, N, params, [Bad()], max_cols=1)
    with pytest.raises(lib.DDError):
        lib.Solver(2, N, [(0.0, 1.0)], ras, max_cols=1)
    with pytest.raises(lib.DDError):
        lib.Solver(2, 1, params, ras, max_cols=1)


@pytest.mark.parametrize("mode", MODES)
def test_edge_cases_general_path(lib, mode):
    """The batched path (GEMM + fused PCG kernel in the WHILE graph, n > 63): a zero right-hand side
    next to live ones, maxit reached (DD_ENOCONV, outputs valid), maxit = 0, an out-of-range
    parameter id (DD_EINVAL from the device-side check) and a 33-column batch (ragged tiles)."""
    N = 128; params = [(1.0, 1e2), (1e-3, 1e5)]; ras = fit_all(N, params, 12)
    S = _solver(lib, N, params, ras, max_cols=40)
    S.set_schur_mode(mode)
    try:
        B = np.random.default_rng(3).uniform(-1, 1, (33, N - 1)); B[5] = 0.0
        colp = (np.arange(33) // 17).astype(np.int32)
        r = S.pcg_solve(_cols(B), colp)
        assert S.query_config()["graph_while"] == 1
        assert r.iters[5] == 0 and np.all(r.x.cpu().numpy()[5] == 0) and np.all(np.delete(r.iters, 5) > 0)
        assert np.all(r.rel_res <= 1e-10)
        r2 = S.pcg_solve(_cols(B), colp, maxit=3)
        assert r2.status == lib.DD_ENOCONV and r2.iters.max() == 3
        r0 = S.pcg_solve(_cols(B), colp, maxit=0)
        assert r0.status == lib.DD_ENOCONV and np.all(r0.iters == 0) and np.all(r0.x.cpu().numpy() == 0)
        bad = colp.copy(); bad[7] = 9
        with pytest.raises(lib.DDError):
            S.pcg_solve(_cols(B), bad)
        r3 = S.pcg_solve(_cols(B), colp)          # the handle is still usable after the error
        assert np.array_equal(r3.x.cpu().numpy(), r.x.cpu().numpy())
    finally:
        S.close()


@pytest.mark.parametrize("N", [32, 48, 64])
def test_small_persistent_kernel_matches_general_path(lib, N, monkeypatch):
    # n <= 63 runs the whole PCG in one launch (K7); it must agree with the GEMM/graph path.
    params = [(1.0, 1e2), (1e-4, 1e6)]; ras = fit_all(N, params, 12)
    B = np.random.default_rng(N).uniform(-1, 1, (5, N - 1)); colp = [0, 1, 0, 1, 1]
    S1 = _solver(lib, N, params, ras, max_cols=5)
    monkeypatch.setenv("DD_NO_SMALL", "1")
    S2 = _solver(lib, N, params, ras, max_cols=5)
    try:
        a = S1.pcg_solve(_cols(B), colp, want_hist=True); ca = S1.query_config()
        b = S2.pcg_solve(_cols(B), colp, want_hist=True); cb = S2.query_config()
        assert ca["graph_while"] == 2 and cb["graph_while"] != 2
        assert np.array_equal(a.iters, b.iters)
        assert rel_l2_cols(a.x.cpu().numpy(), b.x.cpu().numpy()) <= 1e-12
        assert np.allclose(a.hist, b.hist, rtol=1e-10)
    finally:
        S1.close(); S2.close()


@pytest.mark.parametrize("mode", MODES)
def test_profile_and_launch_counts(lib, mode):
    N = 96; params = [(1.0, 1e2)]; ras = fit_all(N, params, 8)
    S = _solver(lib, N, params, ras, max_cols=8)
    S.set_schur_mode(mode)
    try:
        B = np.random.default_rng(0).uniform(-1, 1, (8, N - 1))
        S.launch_count()
        r = S.pcg_solve(_cols(B), [0] * 8)
        k = int(r.iters.max())
        n_launch = S.launch_count()
        S.profile(True)
        r2 = S.pcg_solve(_cols(B), [0] * 8)
        prof = S.profile_read()
        S.profile(False)
        assert np.array_equal(r2.x.cpu().numpy(), r.x.cpu().numpy())
        assert prof["polesum_pcg"][1] == k and prof["gemm_schur"][1] == k
        if mode == "factored":
            assert prof["gemm_dst"][1] == k
            assert n_launch == 2 + 3 * k        # solve prologue, init, then K1 + K2 + pole sum per iteration
            assert all(v[0] > 0 for v in prof.values())
        elif mode == "assembled":
            assert prof["gemm_dst"][1] == 0     # the interior solve lives in G (setup)
            assert n_launch == 2 + 2 * k        # solve prologue, init, then [F | G] GEMM + pole sum
        else:
            assert prof["gemm_dst"][1] == 0
            assert n_launch == 2 + 2 * k        # solve prologue (incl. the tile check), init, H_p GEMM + pole sum
        with pytest.raises(lib.DDError):
            S.set_schur_mode("bogus")
    finally:
        S.close()


# ------------------------------------------------------------------------- ragged large sizes (G = 2, 4 groups)
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("N,C", [(1500, 13), (3001, 7), (2049, 3)])
def test_ragged_large_parity(lib, N, C, mode):
    """Interfaces whose chunking uses 2- and 4-warp groups with a partial last chunk, and column
    counts that leave ragged GEMM tiles; against the oracle's mode tier."""
    params = [(1.0, 1e2), (1e-3, 1e5)]
    ras = fit_all(N, params, 18)
    Mo = oprob.ModeProblem2D(N)
    rng = np.random.default_rng(N)
    B = rng.uniform(-1, 1, (C, N - 1))
    colp = np.arange(C) % 2
    S = _solver(lib, N, params, ras, max_cols=C)
    S.set_schur_mode(mode)
    try:
        y = S.apply_schur(_cols(B), colp).cpu().numpy()
        z = S.apply_precond(_cols(B), colp).cpu().numpy()
        ref_y = np.stack([Mo.apply_S(*params[colp[c]], B[c]) for c in range(C)])
        ra = lambda c: ras[colp[c]]
        zb = np.stack([Mo.apply_P_ra(ra(c).c0, ra(c).poles, ra(c).residues, B[c]) for c in range(C)])
        ze = np.stack([Mo.apply_P_ra_eigen(ra(c).c0, ra(c).poles, ra(c).residues, B[c]) for c in range(C)])
        assert rel_l2_cols(y, ref_y) <= 1e-10
        check_precond(z, zb, ze, ras)
        res = S.pcg_solve(_cols(B), colp)
        x = res.x.cpu().numpy()
        for c in range(C):
            K, g = params[colp[c]]
            xo, it, rel, hist, conv = opcg.pcg(lambda v: Mo.apply_S(K, g, v),
                                               lambda v: Mo.apply_P_ra(ra(c).c0, ra(c).poles, ra(c).residues, v), B[c])
            assert abs(int(res.iters[c]) - it) <= 1
            assert np.linalg.norm(x[c] - xo) <= 1e-8 * np.linalg.norm(xo)
    finally:
        S.close()


# ------------------------------------------------------------------------- full config sizes
@pytest.mark.parametrize("cfg", [c for c in configs.CONFIGS if c.dim == 2], ids=lambda c: c.name)
def test_full_config_parity(lib, cfg):
    """BASELINE.json configs at full size, in the launch configuration bench.py times, against
    the oracle's mode tier (pinned to dense elimination in test_oracle_pins)."""
    ras = fit_all(cfg.N, cfg.params, cfg.n_poles)
    B, colp = inputs.batch(cfg.n_gamma, len(cfg.params), cfg.rhs_per_param)
    Mo = oprob.ModeProblem2D(cfg.N)
    S = _solver(lib, cfg.N, cfg.params, ras, max_cols=cfg.n_cols)
    try:
        Bt = _cols(B)
        # operator and preconditioner applications on every column
        y = S.apply_schur(Bt, colp).cpu().numpy()
        z = S.apply_precond(Bt, colp).cpu().numpy()
        ref_y = np.empty_like(B); ref_z = np.empty_like(B); ref_ze = np.empty_like(B)
        for p, (K, g) in enumerate(cfg.params):
            sel = colp == p
            ref_y[sel] = Mo.apply_S(K, g, B[sel].T).T
            ref_z[sel] = Mo.apply_P_ra(ras[p].c0, ras[p].poles, ras[p].residues, B[sel].T).T
            ref_ze[sel] = Mo.apply_P_ra_eigen(ras[p].c0, ras[p].poles, ras[p].residues, B[sel].T).T
        assert rel_l2_cols(y, ref_y) <= 1e-10
        check_precond(z, ref_z, ref_ze, ras)
        # the PCG solve
        res = S.pcg_solve(Bt, colp, rtol=cfg.rtol, maxit=cfg.maxit)
        x = res.x.cpu().numpy()
        for p, (K, g) in enumerate(cfg.params):
            sel = np.nonzero(colp == p)[0]
            ra = ras[p]
            X, its, rel, _ = opcg.pcg_batch(lambda V, cols: Mo.apply_S(K, g, V),
                                            lambda V, cols: Mo.apply_P_ra(ra.c0, ra.poles, ra.residues, V),
                                            B[sel].T, rtol=cfg.rtol, maxit=cfg.maxit)
            assert np.all(np.abs(res.iters[sel] - its) <= 1), (p, res.iters[sel], its)
            assert rel_l2_cols(x[sel], X.T) <= 1e-8
        assert np.all(res.rel_res <= cfg.rtol)
    finally:
        S.close()


@pytest.mark.parametrize("name", ["cfg2_2d_N1024_sweep", "cfg5_2d_N2048_darcy"])
def test_schur_modes_agree_full_size(lib, name):
    """The grouped apply (H_p = K_p G + γ_p F per parameter set), the assembled one ([F | G]
    [γX ; KX]) and the factored one (fast diagonalisation per apply) are the same operator: at
    full config size they agree to rounding and give the same PCG iterates (each is pinned to
    the oracle above at smaller sizes)."""
    cfg = configs.BY_NAME[name]
    ras = fit_all(cfg.N, cfg.params, cfg.n_poles)
    B, colp = inputs.batch(cfg.n_gamma, len(cfg.params), cfg.rhs_per_param)
    S = _solver(lib, cfg.N, cfg.params, ras, max_cols=cfg.n_cols)
    try:
        Bt = _cols(B)
        out = {}
        for mode in MODES:
            S.set_schur_mode(mode)
            out[mode] = (S.apply_schur(Bt, colp).cpu().numpy(), S.pcg_solve(Bt, colp, rtol=cfg.rtol, maxit=cfg.maxit))
        yg, rg = out["grouped"]
        for mode in ("assembled", "factored"):
            y, r = out[mode]
            assert rel_l2_cols(y, yg) <= 1e-13
            assert np.all(np.abs(r.iters - rg.iters) <= 1)
            assert rel_l2_cols(r.x.cpu().numpy(), rg.x.cpu().numpy()) <= 1e-8
    finally:
        S.close()


@pytest.mark.parametrize("layout", ["grouped32", "grouped_ragged", "mixed"])
def test_grouped_layouts(lib, layout):
    """Grouped apply on column layouts whose 32-column tiles hold one parameter set each (the
    H_p path, incl. a ragged last group and a multi-tile group) and on an interleaved layout
    (a tile holds several sets: the device-side fallback to [F | G]); against the oracle."""
    N = 700
    params = [(1.0, 1e2), (1e-4, 1e6), (1e-2, 1.0)]
    ras = fit_all(N, params, 16)
    Mo = oprob.ModeProblem2D(N)
    colp = {"grouped32": np.repeat([0, 1, 2], 32),
            "grouped_ragged": np.concatenate([np.repeat([2], 64), np.repeat([0], 32), np.repeat([1], 7)]),
            "mixed": np.arange(45) % 3}[layout].astype(np.int32)
    C = len(colp)
    B = np.random.default_rng(C).uniform(-1, 1, (C, N - 1))
    S = _solver(lib, N, params, ras, max_cols=C)
    try:
        y = S.apply_schur(_cols(B), colp).cpu().numpy()
        assert S.query_config()["splitk_dst"] == -2          # grouped is the dense-F default
        ref = np.stack([Mo.apply_S(*params[colp[c]], B[c]) for c in range(C)])
        assert rel_l2_cols(y, ref) <= 1e-10
        res = S.pcg_solve(_cols(B), colp)
        x = res.x.cpu().numpy()
        for p in range(len(params)):
            sel = np.nonzero(colp == p)[0]
            K, g = params[p]; ra = ras[p]
            X, its, rel, _ = opcg.pcg_batch(lambda V, cols: Mo.apply_S(K, g, V),
                                            lambda V, cols: Mo.apply_P_ra(ra.c0, ra.poles, ra.residues, V),
                                            B[sel].T)
            assert np.all(np.abs(res.iters[sel] - its) <= 1)
            assert rel_l2_cols(x[sel], X.T) <= 1e-8
    finally:
        S.close()


# ------------------------------------------------------------------------- inexact inner PCG (NEXT-4)
@pytest.mark.parametrize("cfg", configs.INEXACT, ids=lambda c: c.name)
def test_inexact_inner_pcg_parity(lib, cfg):
    """The Darcy-pressure Riesz-map block at the paper's inner tolerances (1e-4 / 1e-5) on the
    full config-5 sweep: per-column iteration counts ±1 and per-(K, μ) max / mean against the
    oracle; where the counts agree the iterates agree to 1e-8, otherwise within 10·rtol."""
    ras = fit_all(cfg.N, cfg.params, cfg.n_poles)
    B, colp = inputs.batch(cfg.n_gamma, len(cfg.params), cfg.rhs_per_param)
    Mo = oprob.ModeProblem2D(cfg.N)
    S = _solver(lib, cfg.N, cfg.params, ras, max_cols=cfg.n_cols)
    try:
        res = S.pcg_solve(_cols(B), colp, rtol=cfg.rtol, maxit=cfg.maxit)
        x = res.x.cpu().numpy()
        assert np.all(res.rel_res <= cfg.rtol)
        for p, (K, g) in enumerate(cfg.params):
            sel = np.nonzero(colp == p)[0]
            ra = ras[p]
            X, its, rel, _ = opcg.pcg_batch(lambda V, cols: Mo.apply_S(K, g, V),
                                            lambda V, cols: Mo.apply_P_ra(ra.c0, ra.poles, ra.residues, V),
                                            B[sel].T, rtol=cfg.rtol, maxit=cfg.maxit)
            gi = res.iters[sel]
            assert np.all(np.abs(gi - its) <= 1), (p, gi, its)
            assert abs(int(gi.max()) - int(its.max())) <= 1 and abs(gi.mean() - its.mean()) <= 1
            for j, c in enumerate(sel):
                tol = 1e-8 if gi[j] == its[j] else 10 * cfg.rtol
                assert np.linalg.norm(x[c] - X[:, j]) <= tol * np.linalg.norm(X[:, j])
    finally:
        S.close()


def test_maximum_1d_interface(lib):
    """The largest 1D interface the pole-sum kernels take (n = 8191: 8-warp groups with 32-row
    chunks, the LL = 32 instantiation) against the oracle's mode tier."""
    N = 8192
    params = [(1.0, 1e2), (1e-4, 1e6)]
    ras = fit_all(N, params, 20)
    Mo = oprob.ModeProblem2D(N)
    C = 4
    B = np.random.default_rng(81).uniform(-1, 1, (C, N - 1))
    colp = np.arange(C) % 2
    S = _solver(lib, N, params, ras, max_cols=C)
    try:
        y = S.apply_schur(_cols(B), colp).cpu().numpy()
        ref_y = np.stack([Mo.apply_S(*params[colp[c]], B[c]) for c in range(C)])
        assert rel_l2_cols(y, ref_y) <= 1e-10
        z = S.apply_precond(_cols(B), colp).cpu().numpy()
        ra = lambda c: ras[colp[c]]
        zb = np.stack([Mo.apply_P_ra(ra(c).c0, ra(c).poles, ra(c).residues, B[c]) for c in range(C)])
        ze = np.stack([Mo.apply_P_ra_eigen(ra(c).c0, ra(c).poles, ra(c).residues, B[c]) for c in range(C)])
        check_precond(z, zb, ze, ras)
        res = S.pcg_solve(_cols(B), colp)
        x = res.x.cpu().numpy()
        for c in range(C):
            K, g = params[colp[c]]
            xo, it, *_ = opcg.pcg(lambda v: Mo.apply_S(K, g, v),
                                  lambda v: Mo.apply_P_ra(ra(c).c0, ra(c).poles, ra(c).residues, v), B[c])
            assert abs(int(res.iters[c]) - it) <= 1
            assert np.linalg.norm(x[c] - xo) <= 1e-8 * np.linalg.norm(xo)
    finally:
        S.close()
