"""GPU parity, round 2: the norm_kind = 1 stopping rule (reading A1), the DD_ENOTSPD breakdown
(reading A19), maxit beyond the history buffer, the config-4 full-size solve against the stored
oracle run, and the pole-split partial sums (row a-6) against the oracle's P_RA.  Needs a B200.

Tolerances (north star): applies 1e-10 relative ℓ2 (preconditioner max(1e-10, 1e-15 κ_c), plus
the A12 inner-CG allowance in 3D), solutions 1e-8, iteration counts ±1.
"""
import os

import numpy as np
import pytest

from helpers import fit_all, kappa_c, rel_l2_cols
from oracle import pcg as opcg
from oracle import problem as oprob
from paper_2211_15308_b200 import inputs, rafit

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "cfg4_oracle.npz")


@pytest.fixture(scope="module")
def lib():
    from paper_2211_15308_b200 import binding
    binding.load()
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    return binding


class _RA:
    def __init__(self, c0, poles, residues):
        self.c0, self.poles, self.residues = float(c0), np.asarray(poles, float), np.asarray(residues, float)


def _fit3(N, params, m):
    lo, hi = rafit.interval_face(N)
    return [rafit.fit_ra(K, g, lo, hi, m) for K, g in params]


# ------------------------------------------------------------------------- norm_kind = 1 (reading A1)
@pytest.mark.parametrize("N,C", [(33, 3), (200, 37), (1024, 64)], ids=["small-kernel", "graph", "grouped-1024"])
def test_norm_kind1_parity_2d(lib, N, C):
    """η = ||P r||_2 on every 2D path (persistent small-n kernel, WHILE graph, grouped GEMM at
    the config-2 size): iteration counts ±1, x within 1e-8, column-0 history within 1e-8."""
    params = [(1.0, 1e2), (1e-4, 1e6)]
    ras = fit_all(N, params, 14)
    colp = (np.arange(C) * len(params)) // C
    B = np.random.default_rng(N + 1).uniform(-1, 1, (C, N - 1))
    D = oprob.DenseProblem(2, N) if N <= 200 else oprob.ModeProblem2D(N)
    S = lib.Solver(2, N, params, ras, max_cols=C, device=0)
    try:
        res = S.pcg_solve(torch.as_tensor(B, device="cuda"), colp, norm_kind=1, want_hist=True)
        x = res.x.cpu().numpy()
    finally:
        S.close()
    for c in sorted({0, C // 2, C - 1}):
        K, g = params[colp[c]]; ra = ras[colp[c]]
        xo, it, rel, hist, conv = opcg.pcg(lambda v: D.apply_S(K, g, v),
                                           lambda v: D.apply_P_ra(ra.c0, ra.poles, ra.residues, v), B[c], norm_kind=1)
        assert conv and abs(int(res.iters[c]) - it) <= 1, (c, res.iters[c], it)
        assert np.linalg.norm(x[c] - xo) <= 1e-8 * np.linalg.norm(xo)
        assert res.rel_res[c] <= 1e-10
        if c == 0:
            k = min(len(hist), len(res.hist))
            assert np.allclose(res.hist[:k], hist[:k], rtol=1e-8, atol=0)


def test_norm_kind1_parity_3d(lib):
    N, params = 8, [(1.0, 1e4)]
    ras = _fit3(N, params, 10)
    D = oprob.DenseProblem(3, N)
    B = np.random.default_rng(9).uniform(-1, 1, (3, (N - 1) ** 2))
    S = lib.Solver(3, N, params, ras, max_cols=3, device=0)
    try:
        res = S.pcg_solve(torch.as_tensor(B, device="cuda"), [0, 0, 0], norm_kind=1, want_hist=True)
        x = res.x.cpu().numpy()
    finally:
        S.close()
    K, g = params[0]; ra = ras[0]
    for c in range(3):
        xo, it, rel, hist, conv = opcg.pcg(lambda v: D.apply_S(K, g, v),
                                           lambda v: D.apply_P_ra(ra.c0, ra.poles, ra.residues, v), B[c], norm_kind=1)
        assert conv and abs(int(res.iters[c]) - it) <= 1
        assert np.linalg.norm(x[c] - xo) <= 1e-8 * np.linalg.norm(xo)


# ------------------------------------------------------------------------- DD_ENOTSPD (reading A19)
@pytest.mark.parametrize("dim,N", [(2, 33), (2, 200), (3, 8)], ids=["2d-small-kernel", "2d-graph", "3d"])
def test_enotspd_on_indefinite_preconditioner(lib, dim, N):
    """A 'fit' with r(λ) = -1 < 0 on the whole spectrum (c0 = -1, the one pole switched off by a
    zero residue): P = -M^-1 is negative definite, r.Pr < 0 at the first step.  The oracle raises
    NotSPD; the library returns DD_ENOTSPD for every column."""
    params = [(1.0, 1e2)]
    ras = [_RA(-1.0, [-1.0], [0.0])]
    n_g = (N - 1) ** (dim - 1)
    B = np.random.default_rng(5).uniform(-1, 1, (2, n_g))
    D = oprob.DenseProblem(dim, N)
    with pytest.raises(opcg.NotSPD):
        opcg.pcg(lambda v: D.apply_S(1.0, 1e2, v), lambda v: D.apply_P_ra(-1.0, [-1.0], [0.0], v), B[0])
    S = lib.Solver(dim, N, params, ras, max_cols=2, device=0)
    try:
        res = S.pcg_solve(torch.as_tensor(B, device="cuda"), [0, 0])
        assert res.status == lib.DD_ENOTSPD
        assert np.all(res.iters == 0)
    finally:
        S.close()


# ------------------------------------------------------------------------- maxit beyond the history buffer
@pytest.mark.parametrize("dim,N,maxit", [(2, 128, 4200), (3, 4, 4110)])
def test_maxit_beyond_history_buffer(lib, dim, N, maxit):
    """rtol = 0 and maxit > 4096 with no history requested: the solve runs maxit iterations
    (DD_ENOCONV, or DD_OK if η reaches exactly 0) without writing past the device history
    buffer, and the handle still solves correctly afterwards; with a history, maxit + 1 > 4096
    is DD_EINVAL."""
    params = [(1.0, 1e2)]
    ras = fit_all(N, params, 8) if dim == 2 else _fit3(N, params, 8)
    n_g = (N - 1) ** (dim - 1)
    B = np.random.default_rng(2).uniform(-1, 1, (2, n_g))
    S = lib.Solver(dim, N, params, ras, max_cols=2, device=0)
    try:
        Bt = torch.as_tensor(B, device="cuda")
        ref = S.pcg_solve(Bt, [0, 0])
        r = S.pcg_solve(Bt, [0, 0], rtol=0.0, maxit=maxit)
        assert r.status in (lib.DD_ENOCONV, lib.DD_OK)
        assert r.iters.max() <= maxit
        again = S.pcg_solve(Bt, [0, 0])
        assert np.array_equal(again.x.cpu().numpy(), ref.x.cpu().numpy())
        assert np.array_equal(again.iters, ref.iters)
        with pytest.raises(lib.DDError):
            S.pcg_solve(Bt, [0, 0], maxit=4096, want_hist=True)
    finally:
        S.close()


# ------------------------------------------------------------------------- row a-6 vs the oracle
def test_pole_split_partials_sum_to_oracle(lib):
    """Row a-6: the rank partials of the pole split (each rank's share of Eq.(8),
    no communicator: the allreduce's inputs) summed in rank order equal the ORACLE's P_RA
    (sparse-direct parity form) within the 3D preconditioner bar — for world 2, 3 and 4."""
    N = 16; n = N - 1
    params = [(1.0, 1e4)]
    ras = _fit3(N, params, 10)
    ra = ras[0]
    D = oprob.DenseProblem(3, N)
    B = np.random.default_rng(8).uniform(-1, 1, (2, n * n))
    zb = D.apply_P_ra(ra.c0, ra.poles, ra.residues, B.T).T
    ze = D.apply_P_ra_eigen(ra.c0, ra.poles, ra.residues, B.T).T
    kc = kappa_c(ra)
    tol = max(1e-10, 1e-15 * kc) + 20e-13 * kc
    Bt = torch.as_tensor(B, device="cuda")
    for world in (2, 3, 4):
        acc = np.zeros_like(B)
        for rank in range(world):
            S = lib.Solver(3, N, params, ras, max_cols=2, device=0, dist=(rank, world, 1, None))
            try:
                acc += S.apply_precond(Bt, [0, 0]).cpu().numpy()
            finally:
                S.close()
        assert rel_l2_cols(acc, ze) <= tol, world
        assert rel_l2_cols(acc, zb) <= tol + rel_l2_cols(zb, ze), world


# ------------------------------------------------------------------------- config 4 at full size
@pytest.fixture(scope="module")
def cfg4(lib):
    if not os.path.exists(GOLDEN):
        pytest.skip("tests/golden/cfg4_oracle.npz not generated (tests/golden/make_cfg4_oracle.py)")
    g = np.load(GOLDEN)
    N = int(g["N"]); n = N - 1
    ra = _RA(g["c0"], g["poles"], g["residues"])
    B, colp = inputs.batch(n * n, 1, 8)
    return g, N, ra, B, colp


def test_cfg4_full_size_parity(lib, cfg4):
    """BASELINE.json config 4 (3D, N = 128, n_Γ = 16129, K = 1, μ^-1 = 1e4, 20 poles, 8 seeded RHS;
    PAPER.md:237-240, 258-272) element by element against the stored oracle run (dense gevp F,
    mode-tier S_unit, sparse-direct P_RA, plain PCG): S x <= 1e-10, P r <= max(1e-10, 1e-15 κ_c) +
    the A12 inner-CG allowance, iterations ±1, x <= 1e-8 on all 8 columns."""
    g, N, ra, B, colp = cfg4
    K, gam = float(g["K"]), float(g["gamma"])
    kc = float(g["kappa_c"])
    S = lib.Solver(3, N, [(K, gam)], [ra], max_cols=8, device=0)
    try:
        Bt = torch.as_tensor(B, device="cuda")
        y = S.apply_schur(Bt, colp).cpu().numpy()
        assert rel_l2_cols(y, g["y"]) <= 1e-10
        z = S.apply_precond(Bt, colp).cpu().numpy()
        tol = max(1e-10, 1e-15 * kc) + 20e-13 * kc
        assert rel_l2_cols(z, g["z_eig"]) <= tol
        assert rel_l2_cols(z, g["z_par"]) <= tol + rel_l2_cols(g["z_par"], g["z_eig"])
        res = S.pcg_solve(Bt, colp, rtol=1e-10, maxit=500, want_hist=True)
        x = res.x.cpu().numpy()
        assert np.all(np.abs(res.iters - g["iters"]) <= 1), (res.iters, g["iters"])
        assert rel_l2_cols(x, g["x"]) <= 1e-8
        assert np.all(res.rel_res <= 1e-10)
        k = min(len(res.hist), len(g["hist"]))
        assert np.allclose(res.hist[:k], g["hist"][:k], rtol=1e-7, atol=0)
        r1 = S.pcg_solve(Bt, colp, rtol=1e-10, maxit=500, norm_kind=1)
        assert np.all(np.abs(r1.iters - g["iters_norm1"]) <= 1)
    finally:
        S.close()


def test_cfg4_full_size_pole_split_partials(lib, cfg4):
    """Row a-6 at the config-4 size: the partial pole sums of a 4-way split (the NCCL allreduce's
    inputs, balanced by the inner-CG cost model) add up to the oracle's P_RA."""
    g, N, ra, B, colp = cfg4
    K, gam = float(g["K"]), float(g["gamma"])
    kc = float(g["kappa_c"])
    Bt = torch.as_tensor(B[:2], device="cuda")
    acc = np.zeros_like(B[:2])
    world = 4
    for rank in range(world):
        S = lib.Solver(3, N, [(K, gam)], [ra], max_cols=2, device=0, dist=(rank, world, 1, None))
        try:
            acc += S.apply_precond(Bt, colp[:2]).cpu().numpy()
        finally:
            S.close()
    tol = max(1e-10, 1e-15 * kc) + 20e-13 * kc
    assert rel_l2_cols(acc, g["z_eig"][:2]) <= tol


# ------------------------------------------------------------------------- grouped apply from the shared pair
@pytest.mark.parametrize("N", [200, 1024])
def test_grouped_pair_kernel_parity(lib, monkeypatch, N):
    """The grouped Schur apply through the shared-pair kernel (gemm_pair.cu: each warp forms
    K_p G + γ_p F from the G, F tiles; forced with DD_GROUPED_PAIR=1 at sizes where it is not the
    default): group-aligned 32-column tiles, a mixed batch (tiles spanning two parameter sets: the
    F (γX) + G (KX) fallback) and a ragged batch, against the oracle; PCG parity on the aligned batch."""
    monkeypatch.setenv("DD_GROUPED_PAIR", "1")
    params = [(1.0, 1e2), (1e-4, 1e6), (1.0, 0.0)]
    ras = fit_all(N, params, 14)
    Mo = oprob.ModeProblem2D(N)
    C = 96
    B = np.random.default_rng(N).uniform(-1, 1, (C, N - 1))
    S = lib.Solver(2, N, params, ras, max_cols=C, device=0)
    try:
        cases = {"aligned": np.repeat(np.arange(3), 32), "mixed": np.arange(C) % 3,
                 "ragged": np.repeat(np.arange(3), 32)[:33]}
        for name, colp in cases.items():
            Bc = B[:len(colp)]
            y = S.apply_schur(torch.as_tensor(Bc, device="cuda"), colp).cpu().numpy()
            assert S.query_config()["splitk_dst"] == -3, name
            ref = np.stack([Mo.apply_S(*params[colp[c]], Bc[c]) for c in range(len(colp))])
            assert rel_l2_cols(y, ref) <= 1e-10, name
        colp = cases["aligned"]
        res = S.pcg_solve(torch.as_tensor(B, device="cuda"), colp)
        x = res.x.cpu().numpy()
        for c in (0, 40, 95):
            K, g = params[colp[c]]; ra = ras[colp[c]]
            xo, it, *_ = opcg.pcg(lambda v: Mo.apply_S(K, g, v),
                                  lambda v: Mo.apply_P_ra(ra.c0, ra.poles, ra.residues, v), B[c])
            assert abs(int(res.iters[c]) - it) <= 1 and np.linalg.norm(x[c] - xo) <= 1e-8 * np.linalg.norm(xo)
        mixed = S.pcg_solve(torch.as_tensor(B, device="cuda"), cases["mixed"])
        for c in (1, 50):
            K, g = params[cases["mixed"][c]]; ra = ras[cases["mixed"][c]]
            xo, it, *_ = opcg.pcg(lambda v: Mo.apply_S(K, g, v),
                                  lambda v: Mo.apply_P_ra(ra.c0, ra.poles, ra.residues, v), B[c])
            assert abs(int(mixed.iters[c]) - it) <= 1
            assert np.linalg.norm(mixed.x.cpu().numpy()[c] - xo) <= 1e-8 * np.linalg.norm(xo)
    finally:
        S.close()


# ------------------------------------------------------------------------- row-sharded F (SURVEY §8(e) option)
def test_row_sharded_f_emulated_ranks(lib):
    """Config-4 pole split with the F stream row-sharded over the ranks (each rank holds rows
    [r0, r1) of F; with no communicator its Schur apply returns those rows and zeros elsewhere, the
    input of the ncclAllGather): the ranks' outputs add up to the single-GPU apply and to the
    oracle's S x (dense gevp F), for 2 and 3 ranks (N = 32: F has 4 row tiles of 256)."""
    N = 32; n = N - 1
    params = [(1.0, 1e4)]
    ras = _fit3(N, params, 10)
    D = oprob.DenseProblem(3, N)
    B = np.random.default_rng(11).uniform(-1, 1, (3, n * n))
    Bt = torch.as_tensor(B, device="cuda")
    ref = D.apply_S(*params[0], B.T).T
    full = lib.Solver(3, N, params, ras, max_cols=3, device=0)
    try:
        yf = full.apply_schur(Bt, [0, 0, 0]).cpu().numpy()
    finally:
        full.close()
    assert rel_l2_cols(yf, ref) <= 1e-10
    for world in (2, 3):
        acc = np.zeros_like(B)
        nonzero_ranks = 0
        for rank in range(world):
            S = lib.Solver(3, N, params, ras, max_cols=3, device=0, dist=(rank, world, 1, None))
            try:
                y = S.apply_schur(Bt, [0, 0, 0]).cpu().numpy()
            finally:
                S.close()
            nonzero_ranks += int(np.any(y != 0))
            acc += y
        assert nonzero_ranks == world               # every rank owns rows
        assert rel_l2_cols(acc, ref) <= 1e-10, world
        assert rel_l2_cols(acc, yf) <= 1e-13, world


# ------------------------------------------------------------------------- parity-blocked D̂ (K-half skip)
@pytest.mark.parametrize("inner_cg", ["0", "1"])
def test_cfg4_parity_blocked_dhat_bitwise(lib, cfg4, monkeypatch, inner_cg):
    """In the parity-ordered sine domain D̂ = [[0, E], [E', 0]] (D̂_ab = 0 for a + b even); the slab
    GEMMs skip the zero half of K at N = 128 (block edge 64).  The skipped products are exact zeros,
    so P r and S x through the RA-mode Schur operator (r_F systems, same passes) must be BITWISE
    those of the full-K loop (DD_NO_KPAR=1), for the Chebyshev and the CG inner solver."""
    g, N, ra, B, colp = cfg4
    K, gam = float(g["K"]), float(g["gamma"])
    lo, hi = rafit.interval_face(N)
    fr = rafit.fit_power(-0.5, lo, hi, 16, 0.0)
    monkeypatch.setenv("DD_INNER_CG", inner_cg)
    monkeypatch.setenv("DD_CHEB_FUSED", "0")             # the two-pass form (slab GEMMs with kpar)
    Bt = torch.as_tensor(B[:3], device="cuda")
    out = {}
    for nk in ("0", "1"):
        monkeypatch.setenv("DD_NO_KPAR", nk)
        S = lib.Solver(3, N, [(K, gam)], [ra], max_cols=3, device=0, frac=lib.Frac(mode="ra", fra=fr))
        try:
            out[nk] = (S.apply_precond(Bt, colp[:3]).cpu().numpy(), S.apply_schur(Bt, colp[:3]).cpu().numpy())
        finally:
            S.close()
    assert np.array_equal(out["0"][0], out["1"][0])
    assert np.array_equal(out["0"][1], out["1"][1])
    z = out["0"][0]
    tol = max(1e-10, 1e-15 * float(g["kappa_c"])) + 20e-13 * float(g["kappa_c"])
    assert rel_l2_cols(z, g["z_eig"][:3]) <= tol


def test_cfg4_fused_chebyshev_step_matches_two_pass(lib, cfg4, monkeypatch):
    """The fused Chebyshev step (k_cheb_step: per (pair, 64x64 parity block) V = L X̂ M^T with the
    step's epilogue and the loop condition in one persistent kernel) against the two-pass form
    (DD_CHEB_FUSED=0) on the same systems: same arithmetic up to summation order, so P r agrees to
    rounding (1e-12, the Chebyshev polynomial's stable recurrence), both within the oracle
    tolerance; in RA mode the r_F systems (S x) run through the same kernel."""
    g, N, ra, B, colp = cfg4
    K, gam = float(g["K"]), float(g["gamma"])
    lo, hi = rafit.interval_face(N)
    fr = rafit.fit_power(-0.5, lo, hi, 16, 0.0)
    Bt = torch.as_tensor(B[:4], device="cuda")
    out = {}
    for fz in ("1", "0"):
        monkeypatch.setenv("DD_CHEB_FUSED", fz)
        S = lib.Solver(3, N, [(K, gam)], [ra], max_cols=4, device=0, frac=lib.Frac(mode="ra", fra=fr))
        try:
            z = S.apply_precond(Bt, colp[:4]).cpu().numpy()
            y = S.apply_schur(Bt, colp[:4]).cpu().numpy()
            res = S.pcg_solve(Bt, colp[:4], rtol=1e-10, maxit=200)
            out[fz] = (z, y, res.iters.copy(), res.x.cpu().numpy())
        finally:
            S.close()
    assert rel_l2_cols(out["1"][0], out["0"][0]) <= 1e-12
    assert rel_l2_cols(out["1"][1], out["0"][1]) <= 1e-12
    assert np.all(np.abs(out["1"][2] - out["0"][2]) <= 1)
    assert rel_l2_cols(out["1"][3], out["0"][3]) <= 1e-9
    tol = max(1e-10, 1e-15 * float(g["kappa_c"])) + 20e-13 * float(g["kappa_c"])
    assert rel_l2_cols(out["1"][0], g["z_eig"][:4]) <= tol


@pytest.mark.parametrize("ncols,world", [(1, 1), (3, 1), (8, 8)])
def test_cfg4_fused_step_small_batches(lib, cfg4, monkeypatch, ncols, world):
    """The fused Chebyshev step with fewer work items than CTAs (1 column: 84 items for one CTA per
    SM; 3 columns; a W = 8 pole-split rank: 3 systems x 8 columns) against the two-pass form, and
    the summed partials of all 8 ranks against the oracle's P_RA."""
    g, N, ra, B, colp = cfg4
    K, gam = float(g["K"]), float(g["gamma"])
    kc = float(g["kappa_c"])
    Bt = torch.as_tensor(B[:ncols], device="cuda")
    acc = np.zeros_like(B[:ncols])
    for rank in range(world):
        out = {}
        for fz in ("1", "0"):
            monkeypatch.setenv("DD_CHEB_FUSED", fz)
            dist = (rank, world, 1, None) if world > 1 else None
            S = lib.Solver(3, N, [(K, gam)], [ra], max_cols=ncols, device=0, dist=dist)
            try:
                out[fz] = S.apply_precond(Bt, colp[:ncols]).cpu().numpy()
            finally:
                S.close()
        assert rel_l2_cols(out["1"], out["0"]) <= 1e-12, rank
        acc += out["1"]
    tol = max(1e-10, 1e-15 * kc) + 20e-13 * kc
    assert rel_l2_cols(acc, g["z_eig"][:ncols]) <= tol


@pytest.mark.parametrize("cap", ["1", "4", "7"])
def test_cfg4_fused_step_truncated_loop(lib, cfg4, monkeypatch, cap):
    """DD_INNER_MAXIT caps the inner loop below the Chebyshev step counts (K_s - 1 = 18): the fused
    kernel's x̂ ping-pong must hand the combine the buffer of each system's last step
    (min(K_s - 1, J) parity) — the truncated operator equals the two-pass form's (1e-12)."""
    g, N, ra, B, colp = cfg4
    K, gam = float(g["K"]), float(g["gamma"])
    Bt = torch.as_tensor(B[:2], device="cuda")
    monkeypatch.setenv("DD_INNER_MAXIT", cap)
    out = {}
    for fz in ("1", "0"):
        monkeypatch.setenv("DD_CHEB_FUSED", fz)
        S = lib.Solver(3, N, [(K, gam)], [ra], max_cols=2, device=0)
        try:
            out[fz] = S.apply_precond(Bt, colp[:2]).cpu().numpy()
            assert S.inner_iterations() == int(cap)
        finally:
            S.close()
    assert rel_l2_cols(out["1"], out["0"]) <= 1e-12
    assert np.all(np.isfinite(out["1"])) and np.linalg.norm(out["1"]) > 0


def test_cfg4_class_sparse_stream_matches_dense_blocks(lib, cfg4, monkeypatch):
    """The sine-domain H̃ is block-diagonal in the face-index parity classes (A sine-diagonal, M - M̃
    couples opposite parities in both indices): the class-sparse packed stream (one 64 x 64 quadrant
    per half block) against the full packed blocks (DD_FX_CLASS_SPARSE=0) — the dropped quadrants
    are rounding — for S x and the whole PCG."""
    g, N, ra, B, colp = cfg4
    K, gam = float(g["K"]), float(g["gamma"])
    Bt = torch.as_tensor(B[:4], device="cuda")
    out = {}
    for cs in ("1", "0"):
        monkeypatch.setenv("DD_FX_CLASS_SPARSE", cs)
        S = lib.Solver(3, N, [(K, gam)], [ra], max_cols=4, device=0)
        try:
            y = S.apply_schur(Bt, colp[:4]).cpu().numpy()
            res = S.pcg_solve(Bt, colp[:4], rtol=1e-10, maxit=200)
            out[cs] = (y, res.iters.copy(), res.x.cpu().numpy())
        finally:
            S.close()
    assert rel_l2_cols(out["1"][0], out["0"][0]) <= 1e-13
    assert np.all(np.abs(out["1"][1] - out["0"][1]) <= 1)
    assert rel_l2_cols(out["1"][2], out["0"][2]) <= 1e-10
    assert rel_l2_cols(out["1"][0], g["y"][:4]) <= 1e-10


# ------------------------------------------------------------------------- pole-sum layouts under load
def test_cfg5_geometry_polesum_repeat_bitwise(lib):
    """Config-5 geometry (N = 2048, 20 poles, 128 chunks of 16 rows: the compact merged-interior
    layout, three CTAs per SM) with 512 columns, i.e. every SM holding co-resident columns: repeated
    preconditioner applies and PCG solves are bitwise identical (the pole sum's reduction orders are
    fixed, so a shared-memory race between phases A/B/C or with the aliased Z rows would show up as
    run-to-run differences); the apply also matches the oracle-free identity z(αr) = α z(r) exactly
    for α = 2 (power-of-two scaling commutes with every rounding)."""
    N, m = 2048, 20
    params = [(1e-6, 1.0), (1e-2, 1e4), (1.0, 1e2), (1.0, 1e6)]
    ras = fit_all(N, params, m)
    B, colp = inputs.batch(N - 1, len(params), 128)
    S = lib.Solver(2, N, params, ras, max_cols=B.shape[0], device=0)
    try:
        Bt = torch.as_tensor(B, device="cuda")
        z0 = S.apply_precond(Bt, colp).cpu().numpy()
        for _ in range(4):
            assert np.array_equal(S.apply_precond(Bt, colp).cpu().numpy(), z0)
        z2 = S.apply_precond(2.0 * Bt, colp).cpu().numpy()
        assert np.array_equal(z2, 2.0 * z0)
        a = S.pcg_solve(Bt, colp, rtol=1e-10, maxit=100)
        b = S.pcg_solve(Bt, colp, rtol=1e-10, maxit=100)
        assert np.array_equal(a.x.cpu().numpy(), b.x.cpu().numpy())
        assert np.array_equal(a.iters, b.iters)
        assert np.all(a.rel_res <= 1e-10)
    finally:
        S.close()


# ------------------------------------------------------------------------- x written back by the freezing kernel
@pytest.mark.parametrize("maxit", [0, 3, 200])
def test_host_api_pinned_output(lib, maxit):
    """dd_pcg_solve_host with a page-locked x: each column's final x goes to the host buffer from the
    kernel that freezes it (zero copy, overlapped with the columns still iterating).  Bitwise equal
    to the device-buffer solve for converged, maxit-stopped (ENOCONV) and never-iterated columns;
    the buffer starts as NaN, so an entry the kernels skip would show."""
    N = 512
    params = [(1.0, 1e6), (1e-4, 1.0), (1.0, 1e2)]          # 3 / 16 / ~11 iterations: staggered freezes
    ras = fit_all(N, params, 16)
    B, colp = inputs.batch(N - 1, len(params), 40)
    B[5] = 0.0                                              # η0 = 0: frozen at k = 0 with x = 0
    S = lib.Solver(2, N, params, ras, max_cols=B.shape[0], device=0)
    try:
        dev = S.pcg_solve(torch.as_tensor(B, device="cuda"), colp, rtol=1e-10, maxit=maxit)
        xd = dev.x.cpu().numpy()
        xh = torch.full(B.shape, float("nan"), dtype=torch.float64).pin_memory().numpy()
        bh = torch.as_tensor(B).pin_memory().numpy()
        h = S.pcg_solve_host(bh, colp, rtol=1e-10, maxit=maxit, x_out=xh)
        assert h.status == dev.status
        assert np.array_equal(h.iters, dev.iters)
        assert np.array_equal(xh, xd)
        assert np.all(xh[5] == 0.0)
        if maxit == 200:
            assert dev.status == lib.DD_OK and np.all(h.rel_res <= 1e-10)
    finally:
        S.close()


# ------------------------------------------------------------------------- phase B: registers vs shared memory
@pytest.mark.parametrize("N", [512, 1024, 2048, 4096])
def test_pcr_register_form_bitwise(lib, monkeypatch, N):
    """The separator PCR of the merged-interior pole sum (phase B) in its register / warp-shuffle
    form (default) performs the same operations in the same order as the shared-memory form
    (DD_PCR_SMEM=1, read at setup): bitwise equal preconditioner applies for T = 32, 64, 128, 256
    chunks (S = 1, 2, 4, 8 separators per lane), including the reflections of the antisymmetric
    extension at both ends; and the PCG result matches bitwise."""
    params = [(1.0, 1e2), (1e-4, 1e6)]
    ras = fit_all(N, params, 16)
    B, colp = inputs.batch(N - 1, len(params), 8)
    out = {}
    for smem in ("0", "1"):
        monkeypatch.setenv("DD_PCR_SMEM", smem)
        S = lib.Solver(2, N, params, ras, max_cols=B.shape[0], device=0)
        try:
            Bt = torch.as_tensor(B, device="cuda")
            out[smem] = (S.apply_precond(Bt, colp).cpu().numpy(),
                         S.pcg_solve(Bt, colp, rtol=1e-10, maxit=100).x.cpu().numpy())
        finally:
            S.close()
    assert np.array_equal(out["0"][0], out["1"][0])
    assert np.array_equal(out["0"][1], out["1"][1])
