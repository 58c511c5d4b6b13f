"""Remark 1 at a Fig.-4 scale (tool): 3D, RA-evaluated fractional term (no dense F), N cells per side,
8 seeded RHS; prints setup time, PCG iterations and solves/s.  Usage: python tools/ra3d_large.py [N]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2211_15308_b200 import binding, inputs, rafit  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n = N - 1
K, gam = 1.0, 1e4
t0 = time.time()
lo, hi = rafit.interval_face(N)
ra = rafit.fit_ra(K, gam, lo, hi, 20)
fr = rafit.fit_power(-0.5, lo, hi, 16, 0.0)
t1 = time.time()
B, colp = inputs.batch(n * n, 1, 8)
S = binding.Solver(3, N, [(K, gam)], [ra], max_cols=8, device=0, frac=binding.Frac(mode="ra", fra=fr))
torch.cuda.synchronize()
t2 = time.time()
Bt = torch.as_tensor(B, device="cuda")
r = S.pcg_solve(Bt, colp, rtol=1e-10, maxit=200)
torch.cuda.synchronize()
reps = 3
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    r = S.pcg_solve(Bt, colp, rtol=1e-10, maxit=200)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"N={N} n_gamma={n*n} fit {t1-t0:.1f}s setup {t2-t1:.1f}s iters {r.iters.tolist()} rel {float(r.rel_res.max()):.2e} "
      f"solve {ms:.1f} ms = {8/ms*1e3:.1f} solves/s inner {S.inner_iterations()}")
S.close()
