"""Diagnostic: does running the batch as L independent lanes (handles on separate streams) raise
throughput?  Times L concurrent dd_pcg_solve calls with CUDA events (tool, not product)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2211_15308_b200 import configs, inputs, binding
import bench
cfg = configs.BY_NAME[sys.argv[1] if len(sys.argv) > 1 else "cfg2_2d_N1024_sweep"]
ras = bench.fit_ras(cfg)
B, colp = inputs.batch(cfg.n_gamma, len(cfg.params), cfg.rhs_per_param)
C = B.shape[0]
for L in (1, 2, 4):
    if C % L: continue
    w = C // L
    streams = [torch.cuda.Stream() for _ in range(L)]
    S = [binding.Solver(cfg.dim, cfg.N, cfg.params, ras, max_cols=w, device=0, stream=streams[i]) for i in range(L)]
    Bt = [torch.as_tensor(B[i * w:(i + 1) * w], device="cuda") for i in range(L)]
    cp = [torch.as_tensor(colp[i * w:(i + 1) * w].astype(np.int32), device="cuda") for i in range(L)]
    X = [torch.empty_like(b) for b in Bt]
    torch.cuda.synchronize()
    import threading
    def run(i, reps):
        for _ in range(reps):
            S[i].pcg_solve(Bt[i], cp[i], x=X[i], rtol=cfg.rtol, maxit=cfg.maxit)
    for _ in range(2):
        ths = [threading.Thread(target=run, args=(i, 3)) for i in range(L)]
        [t.start() for t in ths]; [t.join() for t in ths]
    torch.cuda.synchronize()
    reps = 20
    t0 = time.perf_counter()
    ths = [threading.Thread(target=run, args=(i, reps)) for i in range(L)]
    [t.start() for t in ths]; [t.join() for t in ths]
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"lanes={L} solves/s (wall) = {C * reps / dt:.0f}  per-lane device ms = {[round(s.last_solve_ms(), 3) for s in S]}", flush=True)
    for s in S: s.close()
