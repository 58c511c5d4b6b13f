"""Multi-rank host logic with world_size 2 over gloo on CPU (no GPU): column sharding covers
every column exactly once, timing reductions take the max, byte broadcast works, and the
config-4 pole partition is balanced."""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2211_15308_b200 import configs, dist

# config-5 PCG iteration counts per (K, μ^-1) pair (round-1 GPU run, K-major): the pilot costs
PILOT5 = [16, 11, 4, 3, 16, 16, 11, 4, 16, 16, 16, 11, 16, 16, 16, 16]


def _worker(rank, world, port, out):
    import torch.distributed as td
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = configs.BY_NAME["cfg5_2d_N2048_darcy"]
        cols, cp = dist.column_shard(len(cfg.params), cfg.rhs_per_param, rank, world)
        bcols, bcp = dist.block_shard(len(cfg.params), cfg.rhs_per_param, rank, world, PILOT5)
        bg = [None] * world
        td.all_gather_object(bg, (bcols.tolist(), bcp.tolist()))
        gathered = [None] * world
        td.all_gather_object(gathered, cols.tolist())
        mx = dist.max_over_ranks(float(rank + 1))
        sm = dist.sum_over_ranks(float(len(cols)))
        payload = bytes(range(128)) if rank == 0 else None
        got = dist.broadcast_bytes(payload, 128)
        out[rank] = (gathered, mx, sm, got == bytes(range(128)), cp.tolist(), bg)
    finally:
        td.destroy_process_group()


def test_two_rank_gloo():
    world = 2
    port = 29500 + (os.getpid() % 1000)
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    cfg = configs.BY_NAME["cfg5_2d_N2048_darcy"]
    allcols = sorted(c for c in res[0][0][0] + res[0][0][1])
    assert allcols == list(range(cfg.n_cols))                # every column exactly once
    assert not set(res[0][0][0]) & set(res[0][0][1])
    # strong-scaling block shard: the same partition on both ranks, every column once, 32-column
    # single-parameter blocks, LPT-balanced predicted work
    bg = res[0][5]
    assert bg == res[1][5]
    bcols = sorted(c for r in range(world) for c in bg[r][0])
    assert bcols == list(range(cfg.n_cols))
    loads = []
    for r in range(world):
        cols, cp = np.asarray(bg[r][0]), np.asarray(bg[r][1])
        assert np.all(cp == cols // cfg.rhs_per_param)
        for b in range(0, len(cols), 32):
            assert len(set(cp[b:b + 32])) == 1 and cols[b] % 32 == 0
        loads.append(sum(PILOT5[p] for p in cp))
    assert max(loads) - min(loads) <= 32 * max(PILOT5)
    for r in range(world):
        gathered, mx, sm, ok, cp, _ = res[r]
        assert mx == 2.0 and sm == cfg.n_cols and ok
        # every rank holds the same mix of parameter sets
        assert np.bincount(cp).tolist() == [cfg.rhs_per_param // world] * len(cfg.params)


def test_column_shard_single_rank_is_identity():
    cols, cp = dist.column_shard(4, 64, 0, 1)
    assert cols.tolist() == list(range(256)) and cp.tolist() == list(np.repeat(np.arange(4), 64))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_pole_partition_balanced(world):
    lo, hi = 19.74, 423472.9          # config-4 face-pair interval
    poles = -np.geomspace(0.5, 4e6, 21)
    costs = [dist.shifted_cost(lo, hi, p) for p in poles]
    parts = dist.pole_partition(costs, world)
    assert sorted(i for p in parts for i in p) == list(range(21))
    loads = [sum(costs[i] for i in p) for p in parts]
    assert max(loads) <= max(max(costs), sum(costs) / world) * 1.0001 + 1e-9 or max(loads) - min(loads) <= max(costs)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_block_shard_config5(world):
    """Config 5's 512 solves as 16 blocks of 32 columns, LPT on iterations x width: the heaviest
    rank carries no more than the LPT bound (max block + average) and all blocks are placed."""
    cfg = configs.BY_NAME["cfg5_2d_N2048_darcy"]
    parts = [dist.block_shard(len(cfg.params), cfg.rhs_per_param, r, world, PILOT5) for r in range(world)]
    allc = sorted(int(c) for cols, _ in parts for c in cols)
    assert allc == list(range(cfg.n_cols))
    loads = [sum(PILOT5[p] for p in cp) for _, cp in parts]
    total = sum(PILOT5) * cfg.rhs_per_param
    assert max(loads) <= total / world + 32 * max(PILOT5)
    if world == 8:
        assert max(loads) == 32 * 32          # two 16-iteration blocks on the heaviest ranks


def test_pole_partition_counts_config4():
    """Config 4 (20 poles + the mass term = 21 systems): the library's cost model (a unit per
    sine-preconditioned inner-CG system) splits them 3,3,3,3,3,2,2,2 over 8 ranks."""
    lo, hi = 19.74, 423472.9
    costs = [dist.inner_cost(lo, hi, p) for p in -np.geomspace(0.5, 4e6, 21)]
    parts = dist.pole_partition(costs, 8)
    assert sorted(len(p) for p in parts) == [2, 2, 2, 3, 3, 3, 3, 3]
