"""Time the 3D preconditioner apply (inner Chebyshev solves) for several column counts (tool):
python tools/time_precond3d.py [N] — RA mode (no eigensolve) so setup is quick; P is the same."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2211_15308_b200 import binding, inputs, rafit  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
lo, hi = rafit.interval_face(N)
ra = rafit.fit_ra(1.0, 1e4, lo, hi, 20)
fr = rafit.fit_power(-0.5, lo, hi, 16, 0.0)
B, colp = inputs.batch((N - 1) ** 2, 1, 16)
S = binding.Solver(3, N, [(1.0, 1e4)], [ra], max_cols=16, device=0, frac=binding.Frac(mode="ra", fra=fr))
for C in (4, 6, 7, 8, 9, 12, 14, 16):
    Bt = torch.as_tensor(B[:C], device="cuda")
    for _ in range(3):
        S.apply_precond(Bt, colp[:C])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        S.apply_precond(Bt, colp[:C])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"C={C:2d} pairs={21*C:3d} items={84*C:4d} precond {ms*1e3:.1f} us  per column {ms*1e3/C:.1f} us")
S.close()
