"""CPU ORACLE for the Schur-complement PCG of arXiv 2211.15308 — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import, call or execute anything under `oracle/`.
The product path (`paper_2211_15308_b200`) never imports it, and the oracle never
imports the product path: the two share no code.  The only shared module is
`paper_2211_15308_b200.inputs` (seeded RHS generator; holds none of the method's
arithmetic).

Plain, slow, obviously-correct NumPy/SciPy fp64 implementation of what the hot path
computes, each function citing the passage of PAPER.md it follows:

* `fem`      — P1 assembly on the Freudenthal (2D) / Kuhn (3D) meshes, the discrete
               trace pair (A_Gamma, M_Gamma) on Gamma = {x=0}  (§3).
* `schur`    — the Steklov-Poincare / Schur complement  S = A^ii - A^i0 (A^00)^-1 A^0i
               (Eq.(4), 146-148) by (1) brute-force dense Cholesky
               elimination, (2) dense layer-by-layer block elimination, and (3) for 2D,
               the same elimination carried out mode-by-mode in the sine basis.
* `spectral` — the generalised eigen-factorisation L U = M U Lambda, U^T M U = I and
               L^s = (MU) Lambda^s (MU)^T (Eq.(7)).
* `ra`       — the rational-approximation solution operator
               c0 M^-1 + sum_k c_k (A - p_k M)^-1  (Eq.(8)),
               plus the exact inverse of S_Gamma = K L^{1/2} + gamma L^{-1/2}.
* `pcg`      — preconditioned CG from x0 = 0, stopping on a 1e10 reduction of the
               preconditioned residual norm.

Parity status of each function is listed in DESIGN.md §"Oracle pins".
"""
