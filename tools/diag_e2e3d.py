"""Diagnostic: device-timed vs host-buffer solve time on one config, in alternating order."""
import sys, time, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_15308_b200 import configs, inputs, rafit, binding
import bench
cfg = configs.BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "cfg4_3d_N128"]
ras = bench.fit_ras(cfg)
B, colp = inputs.batch(cfg.n_gamma, len(cfg.params), cfg.rhs_per_param)
S = binding.Solver(cfg.dim, cfg.N, cfg.params, ras, max_cols=B.shape[0], device=0)
Bt = torch.as_tensor(B, device="cuda:0"); cp = torch.as_tensor(colp.astype(np.int32), device="cuda:0")
X = torch.empty_like(Bt)
Bh = torch.as_tensor(B).pin_memory().numpy(); Xh = torch.empty(B.shape, dtype=torch.float64).pin_memory().numpy()
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda:0")
def dev():
    flush.fill_(1.0); torch.cuda.synchronize(); t0 = time.perf_counter()
    r = S.pcg_solve(Bt, cp, x=X, rtol=cfg.rtol, maxit=cfg.maxit); torch.cuda.synchronize()
    return S.last_solve_ms(), (time.perf_counter() - t0) * 1e3, int(r.iters.max())
def host():
    flush.fill_(1.0); torch.cuda.synchronize(); t0 = time.perf_counter()
    r = S.pcg_solve_host(Bh, colp, rtol=cfg.rtol, maxit=cfg.maxit, x_out=Xh)
    return S.last_solve_ms(), (time.perf_counter() - t0) * 1e3, int(np.max(r.iters))
for i in range(4):
    print("dev ", dev(), flush=True)
for i in range(4):
    print("host", host(), flush=True)
for i in range(4):
    print("dev ", dev(), flush=True)
print("diff", float(np.max(np.abs(X.cpu().numpy() - Xh))))
