"""Diagnostic: pole-sum time vs number of systems per column (m poles + mass term) at the cfg2 shape
(tool, not product).  Times dd_apply_precond on 256 columns with CUDA events."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_15308_b200 import binding, inputs, rafit
N = 1024
lo, hi = rafit.interval_1d(N)
params = [(1.0, 1.0), (1.0, 1e2), (1.0, 1e4), (1.0, 1e6)]
B, colp = inputs.batch(N - 1, 4, 64)
Bt = torch.as_tensor(B, device="cuda"); cp = torch.as_tensor(colp.astype(np.int32), device="cuda")
for m in (11, 12, 13, 14, 15, 16, 17, 18, 19):
    ras = [rafit.fit_ra(K, g, lo, hi, m) for K, g in params]
    S = binding.Solver(2, N, params, ras, max_cols=256, device=0)
    Z = torch.empty_like(Bt)
    for _ in range(3): S.apply_precond(Bt, cp, z=Z)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(S.stream)
    for _ in range(50): S.apply_precond(Bt, cp, z=Z)
    e1.record(S.stream); torch.cuda.synchronize()
    nsys = [1 + len(r.poles) for r in ras]
    print(f"m={m} systems={nsys} precond us={e0.elapsed_time(e1) / 50 * 1e3:.2f}", flush=True)
    S.close()
