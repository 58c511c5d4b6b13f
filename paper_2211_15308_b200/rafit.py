"""Host-side rational-approximation fit (setup data for `dd_setup`; not on the GPU path).

PAPER.md:188-199 (footnote, Eq.(8)): the preconditioner S_Γ^-1 = (K L^{1/2} + γ L^{-1/2})^-1
is realised as  c0 M^-1 + Σ_k c_k (L + p_k M)^-1  from a rational approximation f_RA of
f(x) = (K x^{1/2} + γ x^{-1/2})^-1 on the spectral interval; "the number of poles m does
not depend on the dimensionality of Q_h and is instead determined by the accuracy ε_RA".
The paper defers the construction to its references; this module's
choice (reading A9'):

 1. g(x) = x^{-1/2} on [λ_min, λ_max] by Zolotarev's best relative rational approximation
    of type (n, n) (closed form in Jacobi elliptic functions, evaluated with mpmath at 50
    digits): g_RA(x) = d0 Π_l (x + c_{2l}) / Π_l (x + c_{2l-1}),
    c_j = sn^2(jK'/(2n+1); k') / cn^2(jK'/(2n+1); k'), k'^2 = 1 - λ_min/λ_max,
    with x scaled to [1, λ_max/λ_min] and d0 set so the relative error equioscillates.
    All poles are real and negative and all residues positive (Stieltjes function).
 2. f(x) = x g(x) / (K (x + γ/K)) exactly, expanded in partial fractions; this adds the pole
    -γ/K and keeps the relative error of g (f_RA/f = g_RA/g).
 Poles are returned with the sign convention of reading A7: r(x) = c0 + Σ c_k/(x - p_k),
 p_k < 0, and the library forms A_Γ - p_k M_Γ.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class RationalApprox:
    c0: float
    poles: np.ndarray        # p_k < 0
    residues: np.ndarray     # c_k (may be negative after step 2)
    lam_min: float
    lam_max: float
    K: float
    gamma: float
    n_zolo: int
    rel_err: float = float("nan")      # max |r/f - 1| on a 2e4-point geometric grid
    cancel: float = float("nan")       # κ_c of reading A11
    t: float = -0.5                    # fractional exponent of f (dd_frac.t)
    sigma: float = 0.0                 # shift of L (dd_frac.shifted): eigenvalues λ + σ
    method: str = "zolotarev"

    @property
    def m(self) -> int:
        return len(self.poles)

    def __call__(self, x):
        x = np.asarray(x, dtype=np.float64)
        out = np.full_like(x, self.c0)
        for p, c in zip(self.poles, self.residues):
            out = out + c / (x - p)
        return out

    def to_json(self):
        return {"c0": self.c0, "poles": list(map(float, self.poles)),
                "residues": list(map(float, self.residues)), "lam_min": self.lam_min,
                "lam_max": self.lam_max, "K": self.K, "gamma": self.gamma,
                "n_zolo": self.n_zolo, "rel_err": self.rel_err, "cancel": self.cancel, "t": self.t,
                "sigma": self.sigma, "method": self.method}


def _zolotarev_invsqrt(kappa: float, n: int, dps: int = 50):
    """Type-(n,n) Zolotarev approximation of x^{-1/2} on [1, kappa] in pole-residue form.

    Returns (d0, q, r) as mpmath numbers: g(x) = d0 + Σ_l r_l / (x - q_l), q_l < 0."""
    import mpmath as mp
    with mp.workdps(dps):
        kappa = mp.mpf(kappa)
        m = 1 - 1 / kappa                     # parameter k'^2
        Kp = mp.ellipk(m)
        c = []
        for j in range(1, 2 * n + 1):
            u = j * Kp / (2 * n + 1)
            sn = mp.ellipfun("sn", u, m=m)
            cn = mp.ellipfun("cn", u, m=m)
            c.append((sn / cn) ** 2)
        num = [c[2 * l + 1] for l in range(n)]     # c_2, c_4, ..., c_2n
        den = [c[2 * l] for l in range(n)]         # c_1, c_3, ..., c_2n-1
        # equioscillation constant: extrema of sqrt(x) g0(x) on [1, kappa] are attained
        # at the endpoints and at interior alternation points; sample densely in log x.
        def g0(x):
            v = mp.mpf(1)
            for a in num:
                v *= (x + a)
            for b in den:
                v /= (x + b)
            return v
        xs = [mp.power(kappa, mp.mpf(t) / 4000) for t in range(4001)]
        vals = [mp.sqrt(x) * g0(x) for x in xs]
        d0 = 2 / (max(vals) + min(vals))
        q, r = [], []
        for l, b in enumerate(den):
            pole = -b
            res = d0
            for a in num:
                res *= (pole + a)
            for j, b2 in enumerate(den):
                if j != l:
                    res /= (pole + b2)
            q.append(pole); r.append(res)
        return d0, q, r


def f_general(lam, K: float, gamma: float, t: float = -0.5, sigma: float = 0.0):
    """f(λ) = 1/(K (λ+σ)^{1/2} + γ (λ+σ)^t)  (Eq.(6)/(9): S_Γ = K L^{1/2} + γ L^t, L = A_Γ + σ M_Γ)."""
    x = np.asarray(lam, dtype=np.float64) + sigma
    return 1.0 / (K * np.sqrt(x) + gamma * x ** t)


def _finish(ra: RationalApprox, fvals) -> RationalApprox:
    xs = np.geomspace(ra.lam_min, ra.lam_max, 20000)
    f = fvals(xs)
    ra.rel_err = float(np.max(np.abs(ra(xs) / f - 1.0)))
    acc = np.full_like(xs, abs(ra.c0))
    for p, c in zip(ra.poles, ra.residues):
        acc += np.abs(c / (xs - p))
    ra.cancel = float(np.max(acc / f))
    return ra


def _relative_refit(xs, fv, poles):
    """c0, c_k minimising max-ish relative error: least squares of (c0 + Σ c_k/(x-p_k))/f(x) = 1."""
    A = np.column_stack([np.ones_like(xs)] + [1.0 / (xs - p) for p in poles]) / fv[:, None]
    sc = np.linalg.norm(A, axis=0)
    c, *_ = np.linalg.lstsq(A / sc, np.ones_like(xs), rcond=None)
    c = c / sc
    return float(c[0]), np.asarray(c[1:], dtype=np.float64)


def fit_function_aaa(fx, x_lo: float, x_hi: float, n_poles: int):
    """Rational approximation c0 + Σ c_k/(x - q_k) of a positive function fx on [x_lo, x_hi]
    with real negative poles q_k (host setup data; PAPER.md:196-198 leaves the construction to the
    references).  AAA (scipy) proposes poles for several degrees <= n_poles; complex or
    non-negative ones are dropped, the coefficients are refitted for relative accuracy, and the
    candidate with the smallest relative error on a dense geometric grid wins."""
    import warnings
    from scipy.interpolate import AAA
    xs = np.geomspace(x_lo, x_hi, 3000)
    fv = fx(xs)
    xe = np.geomspace(x_lo, x_hi, 20000)
    fe = fx(xe)
    best = None
    for deg in range(max(1, n_poles - 6), n_poles + 1):
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            r = AAA(xs, fv, max_terms=deg + 1, rtol=0.0)
            q = np.asarray(r.poles())
        q = q[(np.abs(q.imag) <= 1e-8 * np.abs(q)) & (q.real < 0)].real
        q = np.sort(q)[::-1][:n_poles]
        c0, c = _relative_refit(xs, fv, q)
        val = np.full_like(xe, c0)
        for qk, ck in zip(q, c):
            val += ck / (xe - qk)
        err = float(np.max(np.abs(val / fe - 1.0)))
        if np.isfinite(err) and (best is None or err < best[0]):
            best = (err, c0, q, c)
    if best is None:
        raise ValueError("no valid rational approximation with real negative poles")
    return best[1], best[2], best[3]


def fit_ra(K: float, gamma: float, lam_min: float, lam_max: float, n_poles: int, t: float = -0.5,
           sigma: float = 0.0) -> RationalApprox:
    """RA of f(λ) = 1/(K (λ+σ)^{1/2} + γ (λ+σ)^t) on [lam_min, lam_max] (λ: eigenvalues of the
    pair (A_Γ, M_Γ)) with `n_poles` poles in total, returned in the library convention
    r(λ) = c0 + Σ c_k/(λ - p_k) (the shift is folded into the poles: p_k = q_k - σ).
    t = -1/2 (Eq.(2), Eq.(6)): n_poles - 1 from the Zolotarev fit of x^{-1/2}, plus -γ/K.
    Other t (Eq.(9) sweep, NEXT-3): AAA with real negative poles (fit_function_aaa)."""
    if not (K > 0 and gamma >= 0 and 0 < lam_min < lam_max and np.isfinite(lam_max)):
        raise ValueError("need K > 0, gamma >= 0, 0 < lam_min < lam_max")
    if not (-1.0 < t < 1.0) or sigma < 0:
        raise ValueError("need -1 < t < 1 and sigma >= 0")
    if t != -0.5:
        fx = lambda x: 1.0 / (K * np.sqrt(x) + gamma * x ** t)
        c0, q, c = fit_function_aaa(fx, lam_min + sigma, lam_max + sigma, n_poles)
        order = np.argsort(-q)
        ra = RationalApprox(c0, q[order] - sigma, c[order], float(lam_min), float(lam_max), float(K), float(gamma),
                            0, t=float(t), sigma=float(sigma), method="aaa")
        return _finish(ra, lambda lam: f_general(lam, K, gamma, t, sigma))
    if sigma != 0.0:
        base = fit_ra(K, gamma, lam_min + sigma, lam_max + sigma, n_poles)
        ra = RationalApprox(base.c0, base.poles - sigma, base.residues, float(lam_min), float(lam_max), float(K),
                            float(gamma), base.n_zolo, t=-0.5, sigma=float(sigma))
        return _finish(ra, lambda lam: f_general(lam, K, gamma, -0.5, sigma))
    import mpmath as mp
    nz = n_poles - 1 if gamma > 0 else n_poles
    if nz < 1:
        raise ValueError("n_poles too small")
    with mp.workdps(50):
        d0, q, r = _zolotarev_invsqrt(lam_max / lam_min, nz)
        lm = mp.mpf(lam_min)
        C0 = d0 / mp.sqrt(lm)                      # λ^{-1/2} ≈ C0 + Σ R_l/(λ - P_l)
        P = [ql * lm for ql in q]
        R = [rl * mp.sqrt(lm) for rl in r]
        Kq, a = mp.mpf(K), mp.mpf(gamma) / mp.mpf(K)
        c0 = C0 / Kq
        poles, res = [], []
        for Pl, Rl in zip(P, R):
            poles.append(Pl)
            res.append(Rl * Pl / ((Pl + a) * Kq))
        if gamma > 0:
            poles.append(-a)
            res.append((-C0 * a + sum(Rl * a / (a + Pl) for Pl, Rl in zip(P, R))) / Kq)
        order = sorted(range(len(poles)), key=lambda i: float(poles[i]))[::-1]  # p closest to 0 first
        ra = RationalApprox(float(c0), np.array([float(poles[i]) for i in order]),
                            np.array([float(res[i]) for i in order]), float(lam_min),
                            float(lam_max), float(K), float(gamma), nz)
    return _finish(ra, lambda lam: f_general(lam, K, gamma))


def fit_power(t: float, lam_min: float, lam_max: float, n_poles: int, sigma: float = 0.0) -> RationalApprox:
    """RA r_F(λ) = c0 + Σ c_k/(λ - p_k) of (λ + σ)^t, -1 < t < 0, on [lam_min, lam_max] — the
    fractional term evaluated by RA (Remark 1: "action of the perturbation can
    instead be computed via RA"; dd_frac mode DD_FRAC_RA).  t = -1/2: Zolotarev's best relative
    approximation of x^{-1/2} (all poles real negative, residues positive); other t: AAA.
    Returned in the library convention (poles of the pair (A_Γ, M_Γ): p_k = q_k - σ)."""
    if not (-1.0 < t < 0.0) or sigma < 0 or not (0 < lam_min < lam_max):
        raise ValueError("need -1 < t < 0, sigma >= 0, 0 < lam_min < lam_max")
    lo, hi = lam_min + sigma, lam_max + sigma
    if t == -0.5:
        import mpmath as mp
        with mp.workdps(50):
            d0, q, r = _zolotarev_invsqrt(hi / lo, n_poles)
            lm = mp.mpf(lo)
            c0 = float(d0 / mp.sqrt(lm))
            poles = np.array([float(ql * lm) for ql in q])
            res = np.array([float(rl * mp.sqrt(lm)) for rl in r])
        method = "zolotarev"
    else:
        c0, poles, res = fit_function_aaa(lambda x: x ** t, lo, hi, n_poles)
        method = "aaa"
    order = np.argsort(-poles)
    ra = RationalApprox(float(c0), poles[order] - sigma, res[order], float(lam_min), float(lam_max), 1.0, 0.0,
                        n_poles, t=float(t), sigma=float(sigma), method=method)
    return _finish(ra, lambda lam: (np.asarray(lam, dtype=np.float64) + sigma) ** t)


def face_pair(N: int):
    """Sparse P1 pair of the Kuhn-mesh face Γ = {x=0} with Dirichlet ∂Γ (stencils of SURVEY §8
    "verified stencils", pinned against element assembly in the oracle tests):
    A = [4; -1 at (±1,0),(0,±1)],  M = (h^2/12)[6; 1 at (±1,0),(0,±1),(1,1),(-1,-1)]."""
    import scipy.sparse as sp
    n = N - 1
    h = 1.0 / N
    I = sp.identity(n, format="csr")
    T = sp.diags([np.ones(n - 1), np.ones(n - 1)], [-1, 1], format="csr")     # neighbours
    U = sp.diags([np.ones(n - 1)], [1], format="csr")                           # +1 shift
    A = 4.0 * sp.kron(I, I) - sp.kron(T, I) - sp.kron(I, T)
    D = sp.kron(U, U) + sp.kron(U.T, U.T)                                       # (1,1) and (-1,-1)
    M = (h * h / 12.0) * (6.0 * sp.kron(I, I) + sp.kron(T, I) + sp.kron(I, T) + D)
    return A.tocsc(), M.tocsc()


def interval_face(N: int):
    """Spectral interval [λ_min, λ_max] of the face pair (A_Γ, M_Γ) (3D configs), by ARPACK
    (shift-invert at 0 for λ_min, largest for λ_max) — host setup data for the RA fit."""
    import scipy.sparse.linalg as spla
    A, M = face_pair(N)
    if A.shape[0] <= 400:
        import scipy.linalg as sla
        lam = sla.eigh(A.toarray(), M.toarray(), eigvals_only=True)
        return float(lam[0]), float(lam[-1])
    lo = spla.eigsh(A, k=1, M=M, sigma=0.0, which="LM", return_eigenvectors=False, tol=1e-12)[0]
    hi = spla.eigsh(A, k=1, M=M, which="LA", return_eigenvectors=False, tol=1e-10, maxiter=20000)[0]
    return float(lo), float(hi * (1.0 + 1e-9))


def interval_1d(N: int):
    """Spectral interval of the 1D P1 pair on Γ with Dirichlet ends, closed form
    λ_k = (6/h^2)(1 - cos θ_k)/(2 + cos θ_k), θ_k = kπ/N, k = 1..N-1 (north star)."""
    h = 1.0 / N
    def lam(k):
        s2 = np.sin(0.5 * np.pi * k / N) ** 2          # (1 - cos θ)/2 without cancellation
        return (6.0 / h ** 2) * (2.0 * s2) / (3.0 - 2.0 * s2)
    return float(lam(1)), float(lam(N - 1))
