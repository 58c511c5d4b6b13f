"""The five BASELINE.json workloads as plain data (no method arithmetic).

The bench's default (headline) workload at N=1 is config 5 (index 4): the largest single-GPU
configuration (512 independent solves at n_Γ = 2047), the one the multi-GPU split shards.
Citations: BASELINE.json "configs"; SURVEY.md §8(d) table.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from itertools import product


@dataclass(frozen=True)
class Config:
    name: str
    dim: int                 # 2: unit square, Gamma = edge x=0;  3: unit cube, Gamma = face x=0
    N: int                   # cells per side
    params: tuple            # ((K, mu_inv), ...)  parameter sets, K-major then mu_inv
    n_poles: int             # total RA poles m (the c0 M^-1 term is extra)
    rhs_per_param: int
    rtol: float = 1e-10      # PAPER.md:231-232 "reducing the preconditioned residual norm by factor 10^10"
    maxit: int = 500
    pole_split: bool = False  # config 4: RA poles split across GPUs + allreduce

    @property
    def n(self) -> int:
        return self.N - 1

    @property
    def n_gamma(self) -> int:
        return self.n if self.dim == 2 else self.n * self.n

    @property
    def n_cols(self) -> int:
        return len(self.params) * self.rhs_per_param


def _grid(Ks, mus):
    return tuple((float(K), float(m)) for K, m in product(Ks, mus))


CONFIGS = (
    Config("cfg1_2d_N32", 2, 32, _grid([1.0], [1e2]), 12, 1),
    Config("cfg2_2d_N1024_sweep", 2, 1024, _grid([1.0], [1.0, 1e2, 1e4, 1e6]), 16, 64),
    Config("cfg3_2d_N4096", 2, 4096, _grid([1e-4, 1.0], [1.0, 1e6]), 24, 32),
    Config("cfg4_3d_N128", 3, 128, _grid([1.0], [1e4]), 20, 8, pole_split=True),
    Config("cfg5_2d_N2048_darcy", 2, 2048, _grid([1e-6, 1e-4, 1e-2, 1.0], [1.0, 1e2, 1e4, 1e6]), 20, 32),
)

# NEXT-4: the same kernels as the inexact Riesz-map block of the Darcy-Stokes
# preconditioner — PCG on the config-5 sweep at the paper's inner tolerances (PAPER.md:372-373
# "relative tolerance of 10^-4"; Appendix, "10^-5"), reported as max / mean
# inner iteration counts per (K, μ) point (Fig. 7's ○ / × markers).
INEXACT = (
    Config("cfg5i_2d_N2048_darcy_rtol1e-5", 2, 2048, _grid([1e-6, 1e-4, 1e-2, 1.0], [1.0, 1e2, 1e4, 1e6]), 20, 32,
           rtol=1e-5),
    Config("cfg5i_2d_N2048_darcy_rtol1e-4", 2, 2048, _grid([1e-6, 1e-4, 1e-2, 1.0], [1.0, 1e2, 1e4, 1e6]), 20, 32,
           rtol=1e-4),
)

BY_NAME = {c.name: c for c in CONFIGS + INEXACT}
HEADLINE = CONFIGS[4]
