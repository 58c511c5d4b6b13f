"""Small driver for ncu captures: set up a config, run `--solves` PCG solves (the first ones are
warm-up).  Usage: python tools/prof_step.py [--config cfg2_2d_N1024_sweep] [--solves 3]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2211_15308_b200 import binding, configs, inputs, rafit  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default=configs.HEADLINE.name)
ap.add_argument("--solves", type=int, default=3)
ap.add_argument("--precond", action="store_true")
a = ap.parse_args()
cfg = configs.BY_NAME[a.config]
lo, hi = rafit.interval_1d(cfg.N)
ras = [rafit.fit_ra(K, g, lo, hi, cfg.n_poles) for K, g in cfg.params]
B, colp = inputs.batch(cfg.n_gamma, len(cfg.params), cfg.rhs_per_param)
S = binding.Solver(cfg.dim, cfg.N, cfg.params, ras, max_cols=B.shape[0], device=0)
Bt = torch.as_tensor(B, device="cuda")
for i in range(a.solves):
    if a.precond:
        S.apply_precond(Bt, colp)
    r = S.pcg_solve(Bt, colp, rtol=cfg.rtol, maxit=cfg.maxit)
torch.cuda.synchronize()
print("ok", int(r.iters.max()), S.query_config())
S.close()
