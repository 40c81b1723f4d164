"""Multi-process host logic on CPU (gloo, world size 2).

The device path shards chains across GPUs with no collective.
Here two gloo ranks each run their shard of chains through the CPU oracle
(the same per-chain function the device implements) and gather the results:
they must equal the single-process run bit for bit, the device analogue of
the reference's sequential == parallel invariance (tests/test_chains.py:75-91).
The bench's max-over-ranks timing reduction is checked the same way.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1912_11554_b200 as ts


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.join(here, "..", "oracle"))
    import torch
    import turnstile_oracle as o

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    C, W, S, seed = 5, 30, 12, 11
    ids = ts.chains.shard_range(C, rank, world)
    keys = o.chain_keys(seed, C)
    model = o.Model("std_normal", 3)
    local = np.zeros((C, S, 3))
    lf = np.zeros(C)
    for c in ids:
        r = o.run_chain(model, keys[c], W, S)
        local[c] = np.asarray(r["samples"])
        lf[c] = r["total_leapfrogs"]
    t = torch.from_numpy(local)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)  # disjoint shards: sum == gather
    tl = torch.from_numpy(lf)
    dist.all_reduce(tl, op=dist.ReduceOp.SUM)
    # bench.py's timing rule: the job time is the max over ranks
    mine = torch.tensor([10.0 + rank], dtype=torch.float64)
    dist.all_reduce(mine, op=dist.ReduceOp.MAX)
    if rank == 0:
        np.savez(out_path, samples=t.numpy(), leapfrogs=tl.numpy(), tmax=mine.numpy())
    dist.destroy_process_group()


def test_chain_sharding_two_ranks_matches_single_process(tmp_path, oracle):
    out = str(tmp_path / "gathered.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    keys = oracle.chain_keys(11, 5)
    model = oracle.Model("std_normal", 3)
    for c in range(5):
        r = oracle.run_chain(model, keys[c], 30, 12)
        assert np.array_equal(got["samples"][c], np.asarray(r["samples"]))
        assert got["leapfrogs"][c] == r["total_leapfrogs"]
    assert got["tmax"][0] == 11.0


def test_shard_range_partitions():
    for C in (1, 5, 8, 8192):
        for world in (1, 2, 3, 8):
            parts = [ts.chains.shard_range(C, r, world) for r in range(world)]
            assert sum(parts, []) == list(range(C))
    with pytest.raises(ValueError):
        ts.chains.shard_range(4, 2, 2)
