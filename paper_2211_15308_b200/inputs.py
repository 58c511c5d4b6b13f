"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method (no operators, no solves): only the
seeded right-hand-side generator and the column layout of a batch.  It is the one
module both `oracle/` and the product path may import ("Input recipe").

RHS recipe (the paper never states b): a dual vector on Γ,
``numpy.random.default_rng(seed).uniform(-1.0, 1.0, size=(R, n_Gamma))``, one row per
right-hand side; the seed is the parameter-set index within the config (K-major,
then mu^-1), plus ``seed_offset`` (used to give each rank of a multi-GPU weak-scaling
run its own draws).
"""
from __future__ import annotations

import numpy as np


def rhs_block(n_gamma: int, count: int, seed: int) -> np.ndarray:
    """`count` right-hand sides of length n_gamma, shape (count, n_gamma), fp64 uniform[-1,1]."""
    if n_gamma < 0 or count < 0:
        raise ValueError("negative size")
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(count, n_gamma))


def batch(n_gamma: int, n_param: int, rhs_per_param: int, seed_offset: int = 0):
    """A full batch: (B, col_param) with B of shape (n_param*rhs_per_param, n_gamma).

    Row c of B is column c of the column-major n_Gamma x C device layout; columns are
    grouped parameter-major, col_param[c] is the parameter-set index of column c.
    """
    blocks = [rhs_block(n_gamma, rhs_per_param, seed_offset + p) for p in range(n_param)]
    B = np.concatenate(blocks, axis=0) if blocks else np.zeros((0, n_gamma))
    col_param = np.repeat(np.arange(n_param, dtype=np.int32), rhs_per_param)
    return np.ascontiguousarray(B), col_param


def mode_vectors(n: int, modes, weights=None) -> np.ndarray:
    """Test input built from discrete sine modes: x_j = sum_b w_b sin(j b pi/(n+1)), j=1..n.

    Used only to build full-size property checks (a combination of a few DST modes);
    integer argument reduction keeps it exact to rounding at any n.
    """
    N = n + 1
    j = np.arange(1, n + 1, dtype=np.int64)
    x = np.zeros(n)
    if weights is None:
        weights = np.ones(len(modes))
    for b, w in zip(modes, weights):
        arg = (j * int(b)) % (2 * N)
        x += w * np.sin(np.pi * arg / N)
    return x
