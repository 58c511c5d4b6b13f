"""Time dd_apply_precond (and one PCG solve) on a config's full batch with CUDA events.
Usage: python tools/time_precond.py [--config cfg5_2d_N2048_darcy] [--reps 50]
(environment switches such as DD_V2_SKIP are read at setup)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2211_15308_b200 import binding, configs, inputs, rafit  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default=configs.HEADLINE.name)
ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()
cfg = configs.BY_NAME[a.config]
lo, hi = rafit.interval_1d(cfg.N) if cfg.dim == 2 else rafit.interval_face(cfg.N)
ras = [rafit.fit_ra(K, g, lo, hi, cfg.n_poles) for K, g in cfg.params]
B, colp = inputs.batch(cfg.n_gamma, len(cfg.params), cfg.rhs_per_param)
S = binding.Solver(cfg.dim, cfg.N, cfg.params, ras, max_cols=B.shape[0], device=0)
Bt = torch.as_tensor(B, device="cuda")
colp = torch.as_tensor(colp, dtype=torch.int32, device="cuda")   # device col_param: no per-call conversion
Z = torch.empty_like(Bt)
for _ in range(5):
    S.apply_precond(Bt, colp, Z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    S.apply_precond(Bt, colp, Z)
e1.record()
torch.cuda.synchronize()
print(f"{a.config} precond apply {e0.elapsed_time(e1) / a.reps * 1e3:.2f} us  (cols {B.shape[0]}, "
      f"V2_SKIP={os.environ.get('DD_V2_SKIP', '0')})")
S.close()
