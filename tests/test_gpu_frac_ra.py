"""The fractional term evaluated by rational approximation (Remark 1, PAPER.md:274-288;
dd_frac mode DD_FRAC_RA): y = K S_unit x + γ M r_F(L) M x with r_F ≈ L^t
applied as a second pole sum (no dense F).  Parity with the oracle's same-RA operator; closeness
to the dense Eq.(7) operator within the fit error.  Needs a B200 (-m gpu)."""
import numpy as np
import pytest

from helpers import rel_l2_cols
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


@pytest.mark.parametrize("mode", ["assembled", "factored"])
@pytest.mark.parametrize("N,t,sigma", [(9, -0.5, 0.0), (64, -0.5, 0.0), (200, -0.25, 1.0), (1024, -0.5, 0.0),
                                         (2048, -0.5, 0.0)])
def test_ra_operator_parity(lib, N, t, sigma, mode):
    # N = 2048 with 20 preconditioner poles and the 16-pole r_F: both pole sums (k_frac_ra and the
    # fused PCG kernel) take the compact 3-CTA layout of the 128-chunk geometry
    params = [(1.0, 1e2), (1e-3, 1e4)]
    lo, hi = rafit.interval_1d(N)
    ras = [rafit.fit_ra(K, g, lo, hi, 20 if N >= 2048 else 14, t=t, sigma=sigma) for K, g in params]
    fr = rafit.fit_power(t, lo, hi, 16, sigma)
    fra = (fr.c0, fr.poles, fr.residues)
    if N <= 200:
        O = oprob.DenseProblem(2, N, t=t, sigma=sigma, frac_ra=fra)
        Oex = oprob.DenseProblem(2, N, t=t, sigma=sigma)
    else:
        O = oprob.ModeProblem2D(N, t=t, sigma=sigma, frac_ra=fra)
        Oex = oprob.ModeProblem2D(N, t=t, sigma=sigma)
    C = 8
    B = np.random.default_rng(N).uniform(-1, 1, (C, N - 1))
    colp = np.arange(C) % 2
    S = lib.Solver(2, N, params, ras, max_cols=C, frac=lib.Frac(t=t, shifted=bool(sigma), mode="ra", fra=fr))
    S.set_schur_mode(mode)
    try:
        y = S.apply_schur(_cols(B), colp).cpu().numpy()
        ref = np.stack([O.apply_S(*params[colp[c]], B[c]) for c in range(C)])
        assert rel_l2_cols(y, ref) <= max(1e-10, 1e-15 * fr.cancel * 1e2)
        ex = np.stack([Oex.apply_S(*params[colp[c]], B[c]) for c in range(C)])
        assert rel_l2_cols(y, ex) <= 2 * fr.rel_err + 1e-12
        res = S.pcg_solve(_cols(B), colp)
        x = res.x.cpu().numpy()
        for c in range(C):
            K, g = params[colp[c]]; ra = ras[colp[c]]
            xo, it, *_ = opcg.pcg(lambda v: O.apply_S(K, g, v),
                                  lambda v: O.apply_P_ra(ra.c0, ra.poles, ra.residues, v), B[c])
            assert abs(int(res.iters[c]) - it) <= 1
            assert np.linalg.norm(x[c] - xo) <= 1e-8 * np.linalg.norm(xo)
        cfg = S.query_config()
        assert cfg["graph_while"] != 2          # the dense-F persistent small kernel is not used
    finally:
        S.close()


def test_ra_mode_rejects_bad_fit(lib):
    lo, hi = rafit.interval_face(6)
    ras = [rafit.fit_ra(1.0, 1.0, lo, hi, 8)]

    class Bad:
        c0 = 1.0; poles = np.array([0.5]); residues = np.array([1.0])
    with pytest.raises(lib.DDError):
        lib.Solver(3, 6, [(1.0, 1.0)], ras, max_cols=1, frac=lib.Frac(mode="ra", fra=Bad()))


def test_schur_mode_rules(lib):
    """dd_set_schur_mode (include/dd_api.h): RA handles default to assembled and refuse grouped
    (no dense F to fold in); 3D handles refuse every 2D mode switch."""
    N = 64
    lo, hi = rafit.interval_1d(N)
    params = [(1.0, 1e2)]
    ras = [rafit.fit_ra(K, g, lo, hi, 10) for K, g in params]
    S = lib.Solver(2, N, params, ras, max_cols=2,
                   frac=lib.Frac(mode="ra", fra=rafit.fit_power(-0.5, lo, hi, 12, 0.0)))
    try:
        S.apply_schur(torch.zeros((2, N - 1), dtype=torch.float64, device="cuda"), [0, 0])
        assert S.query_config()["splitk_dst"] == -1      # assembled
        with pytest.raises(lib.DDError):
            S.set_schur_mode("grouped")
        S.set_schur_mode("factored")
    finally:
        S.close()
    lo3, hi3 = rafit.interval_face(8)
    S3 = lib.Solver(3, 8, params, [rafit.fit_ra(1.0, 1e2, lo3, hi3, 10)], max_cols=1)
    try:
        for mode in ("factored", "assembled", "grouped"):
            with pytest.raises(lib.DDError):
                S3.set_schur_mode(mode)
    finally:
        S3.close()


@pytest.mark.parametrize("N", [8, 13])
def test_ra_operator_3d(lib, N):
    """Remark 1 on a 3D face (the survey's motivation for NEXT-2: no dense n_Γ^2 F): y = K S_unit x
    + γ M r_F(L) M x with r_F's face systems solved by the batched sine-domain CG, against the
    oracle's same-RA operator; and within the fit error of the Eq.(7) operator."""
    n = N - 1
    params = [(1.0, 1e2)]
    lo, hi = rafit.interval_face(N)
    ras = [rafit.fit_ra(K, g, lo, hi, 10) for K, g in params]
    fr = rafit.fit_power(-0.5, lo, hi, 12)
    fra = (fr.c0, fr.poles, fr.residues)
    O = oprob.DenseProblem(3, N, frac_ra=fra)
    Oex = oprob.DenseProblem(3, N)
    B = np.random.default_rng(N).uniform(-1, 1, (3, n * n))
    S = lib.Solver(3, N, params, ras, max_cols=3, frac=lib.Frac(mode="ra", fra=fr))
    try:
        y = S.apply_schur(_cols(B), [0] * 3).cpu().numpy()
        ref = O.apply_S(*params[0], B.T).T
        assert rel_l2_cols(y, ref) <= 1e-10 + 2e-12 * fr.cancel
        ex = Oex.apply_S(*params[0], B.T).T
        assert rel_l2_cols(y, ex) <= 2 * fr.rel_err + 1e-10
        res = S.pcg_solve(_cols(B), [0] * 3)
        ra = ras[0]
        for c in range(3):
            xo, it, *_ = opcg.pcg(lambda v: O.apply_S(*params[0], v),
                                  lambda v: O.apply_P_ra(ra.c0, ra.poles, ra.residues, v), B[c])
            assert abs(int(res.iters[c]) - it) <= 1
            assert np.linalg.norm(res.x.cpu().numpy()[c] - xo) <= 1e-8 * np.linalg.norm(xo)
    finally:
        S.close()
