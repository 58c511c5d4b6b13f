"""Multi-GPU plumbing (host logic only; no method arithmetic).

SURVEY §8(e): configs 2, 3, 5 shard by columns — independent (K, μ, RHS) instances, no
data-path collective; config 4 splits the RA systems (poles) across ranks and sums the partial
pole sums with one allreduce per preconditioner apply (the only exchange step of the method).
One process per GPU; torch.distributed (NCCL on GPUs, gloo in the CPU tests) carries the timing
reductions and the NCCL unique-id bootstrap of libdd's communicator.
"""
from __future__ import annotations

import math

import numpy as np


def column_shard(n_param: int, rhs_per_param: int, rank: int, world: int):
    """Stripe every parameter set's right-hand sides across ranks: rank r gets
    RHS j of set p for j ≡ r (mod world).  Returns (global column indices, col_param).
    Columns are global indices into the parameter-major batch of `inputs.batch`.  Striping keeps
    every rank's mix of parameter sets (and so of iteration counts) identical."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    cols, cp = [], []
    for p in range(n_param):
        for j in range(rank, rhs_per_param, world):
            cols.append(p * rhs_per_param + j)
            cp.append(p)
    return np.asarray(cols, dtype=np.int64), np.asarray(cp, dtype=np.int32)


def column_blocks(n_param: int, rhs_per_param: int, bn: int = 32):
    """The batch cut into blocks of <= bn consecutive columns of ONE parameter set (columns
    parameter-major as in `inputs.batch`): [(param, first global column, width), ...].  bn = 32 is
    the grouped Schur GEMM's column tile (one H_p per tile)."""
    out = []
    for p in range(n_param):
        for j0 in range(0, rhs_per_param, bn):
            out.append((p, p * rhs_per_param + j0, min(bn, rhs_per_param - j0)))
    return out


def block_shard(n_param: int, rhs_per_param: int, rank: int, world: int, iters, bn: int = 32):
    """Strong-scaling split of a FIXED batch of independent solves over `world` ranks (SURVEY
    §8(e); config 5: the 512 solves of the Appendix sweep).  Units are whole
    bn-column single-parameter blocks (`column_blocks`), so every rank's grouped-GEMM tiles keep
    one parameter set each; blocks go to ranks by LPT (`pole_partition`) on their predicted work
    iters[param] x width — the PCG iteration count of the block's parameter set (a pilot solve;
    counts range 3..16 over the config-5 grid), the GEMM and pole-sum work per live column being
    the same for every block.  Deterministic: every rank computes the same partition.
    Returns (global column indices, col_param) of `rank`, blocks in ascending column order."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    blocks = column_blocks(n_param, rhs_per_param, bn)
    parts = pole_partition([float(iters[p]) * w for p, _, w in blocks], world)
    cols, cp = [], []
    for b in parts[rank]:
        p, c0, w = blocks[b]
        cols.extend(range(c0, c0 + w))
        cp.extend([p] * w)
    return np.asarray(cols, dtype=np.int64), np.asarray(cp, dtype=np.int32)


def pole_partition(costs, world: int):
    """Split systems (weights = predicted solve cost) over `world` ranks, balancing total cost
    (longest-processing-time greedy, deterministic ties by index).  Returns a list of sorted
    index lists, one per rank.  Config 4: inner-CG cost per pole ∝ sqrt(cond(A_Γ - p M_Γ))."""
    if world < 1:
        raise ValueError("world >= 1")
    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    load = [0.0] * world
    parts = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda q: (load[q], q))
        parts[r].append(i)
        load[r] += float(costs[i])
    return [sorted(p) for p in parts]


def shifted_cost(lam_min: float, lam_max: float, pole: float) -> float:
    """Predicted iterations of PLAIN CG on (A - pM) with spectrum [λmin, λmax] of the pair: ∝ sqrt(κ),
    κ = (λmax - p)/(λmin - p).  Not the library's cost model: its inner CG is preconditioned by the
    sine-diagonal part (κ <= 3 for every shift), see `inner_cost`."""
    return math.sqrt((lam_max - pole) / (lam_min - pole))


def inner_cost(lam_min: float, lam_max: float, pole: float) -> float:
    """Cost model of one shifted face system in libdd (dd3d.cpp): the sine-preconditioned inner CG
    takes about the same ~20 iterations for every shift (171 iterations over 21
    systems), batched over (system, column) pairs — a unit cost per system, so the pole split
    balances the COUNT of systems per rank."""
    return 1.0


def max_over_ranks(value: float, device=None) -> float:
    """Max of a float over all ranks (the timing rule of the bench)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def broadcast_bytes(payload: bytes | None, nbytes: int, src: int = 0, device=None) -> bytes:
    """Broadcast `nbytes` raw bytes from rank `src` (e.g. a 128-byte ncclUniqueId)."""
    import torch
    import torch.distributed as dist
    buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
    if payload is not None:
        buf[:len(payload)] = torch.frombuffer(bytearray(payload), dtype=torch.uint8)[:nbytes].to(device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.broadcast(buf, src=src)
    return bytes(buf.cpu().numpy().tobytes())
