"""Time the kernel classes of a config in isolation (tool): python tools/prof_kernel.py --config cfg5_2d_N2048_darcy
Prints the instrumented per-class average launch times (µs) of a few solves (iterations capped with --maxit;
statuses ignored — for A/B timing of diagnostic switches only)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2211_15308_b200 import binding, configs, inputs, rafit  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default=configs.HEADLINE.name)
ap.add_argument("--maxit", type=int, default=8)
ap.add_argument("--solves", type=int, default=3)
a = ap.parse_args()
cfg = configs.BY_NAME[a.config]
lo, hi = rafit.interval_1d(cfg.N)
ras = [rafit.fit_ra(K, g, lo, hi, cfg.n_poles) for K, g in cfg.params]
B, colp = inputs.batch(cfg.n_gamma, len(cfg.params), cfg.rhs_per_param)
S = binding.Solver(cfg.dim, cfg.N, cfg.params, ras, max_cols=B.shape[0], device=0)
Bt = torch.as_tensor(B, device="cuda")
S.pcg_solve(Bt, colp, rtol=0.0, maxit=a.maxit)
S.profile(True)
for _ in range(a.solves):
    S.pcg_solve(Bt, colp, rtol=0.0, maxit=a.maxit)
p = S.profile_read()
print(os.environ.get("DD_V2_SKIP", "0"), {k: round(v[0] / v[1] * 1e3, 2) for k, v in p.items() if v[1]})
S.close()
