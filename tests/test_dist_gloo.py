"""Multi-rank host logic with world_size 2 over gloo on CPU (no GPU): column sharding covers
every column exactly once, timing reductions take the max, byte broadcast works, and the
config-4 pole partition is balanced."""
import os

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2211_15308_b200 import configs, dist


def _worker(rank, world, port, out):
    import torch.distributed as td
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = configs.BY_NAME["cfg5_2d_N2048_darcy"]
        cols, cp = dist.column_shard(len(cfg.params), cfg.rhs_per_param, rank, world)
        gathered = [None] * world
        td.all_gather_object(gathered, cols.tolist())
        mx = dist.max_over_ranks(float(rank + 1))
        sm = dist.sum_over_ranks(float(len(cols)))
        payload = bytes(range(128)) if rank == 0 else None
        got = dist.broadcast_bytes(payload, 128)
        out[rank] = (gathered, mx, sm, got == bytes(range(128)), cp.tolist())
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
    for r in range(world):
        gathered, mx, sm, ok, cp = res[r]
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
