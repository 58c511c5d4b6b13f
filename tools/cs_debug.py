import os, sys, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
from paper_2211_15308_b200 import binding, inputs, rafit
N = 128
lo, hi = rafit.interval_face(N)
ra = rafit.fit_ra(1.0, 1e4, lo, hi, 20)
B, colp = inputs.batch((N - 1) ** 2, 1, 2)
out = {}
for cs in ("1", "0"):
    os.environ["DD_FX_CLASS_SPARSE"] = cs
    S = binding.Solver(3, N, [(1.0, 1e4)], [ra], max_cols=2, device=0)
    out[cs] = S.apply_schur(torch.as_tensor(B, device="cuda"), colp).cpu().numpy()
    S.close()
d = out["1"] - out["0"]
print("rel diff", np.linalg.norm(d) / np.linalg.norm(out["0"]))
n = N - 1
D = d[0].reshape(n, n); R = out["0"][0].reshape(n, n)
print("max |diff| by row block (first index < 64 / >= 64):", np.abs(D[:64]).max(), np.abs(D[64:]).max())
