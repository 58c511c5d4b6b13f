"""Diagnostic (tool): PCG time per iteration at the cfg2 shape vs the number of RA systems per
column (m poles + the mass term): 4 groups per CTA -> ceil((m+1)/4) rounds of systems."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_15308_b200 import binding, inputs, rafit
N = 1024
lo, hi = rafit.interval_1d(N)
params = [(1.0, 1.0), (1.0, 1e2), (1.0, 1e4), (1.0, 1e6)]
B, colp = inputs.batch(N - 1, 4, 64)
Bt = torch.as_tensor(B, device="cuda"); cp = torch.as_tensor(colp.astype(np.int32), device="cuda")
X = torch.empty_like(Bt)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for m in (11, 12, 14, 15, 16, 18, 19):
    ras = [rafit.fit_ra(K, g, lo, hi, m) for K, g in params]
    S = binding.Solver(2, N, params, ras, max_cols=256, device=0)
    for _ in range(3):
        r = S.pcg_solve(Bt, cp, x=X)
    ts, its = [], []
    for _ in range(10):
        flush.fill_(1.0)
        r = S.pcg_solve(Bt, cp, x=X)
        ts.append(S.last_solve_ms()); its.append(int(r.iters.max()))
    print(f"m={m} systems={m + 1} rounds={(m + 1 + 3) // 4} ms={np.median(ts):.4f} iters={its[0]} "
          f"us/iter={np.median(ts) / its[0] * 1e3:.2f}", flush=True)
    S.close()
