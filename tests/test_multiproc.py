"""Multi-process host logic on CPU (gloo, world size 2).

The device path shards chains across GPUs with no collective.
Here two gloo ranks each run their shard of chains through the CPU oracle
(the same per-chain function the device implements) and gather the results:
they must equal the single-process run bit for bit, the device analogue of
the reference's sequential == parallel invariance (tests/test_chains.py:75-91).
The bench's max-over-ranks timing reduction is checked the same way.
"""

from __future__ import annotations

import math
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


# ----------------------------------------------------------------------------- row sharding host logic


def test_row_range_whole_tiles():
    for n in (1, 7, 8, 9, 20005, 8_000_000):
        for world in (1, 2, 3, 8):
            rr = [ts.rowshard.row_range(n, r, world) for r in range(world)]
            assert rr[0][0] == 0 and rr[-1][1] == n
            for (a0, b0), (a1, b1) in zip(rr, rr[1:]):
                assert b0 == a1
            for a, b in rr:
                assert a % 32 == 0 and a <= b
            sizes = [-(-(b - a) // 32) for a, b in rr]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        ts.rowshard.row_range(10, 2, 2)


def _fx_split(v):
    """Host restatement of csrc fx_split (|v| < 2^40): round-half-even."""
    a = round(v * 1024.0)
    rem = v - a * (1.0 / 1024.0)
    return int(a), int(round(rem * 2305843009213693952.0))


def test_fixed_point_totals_are_partition_free():
    """Per-tile partials converted exactly to (hi, lo) words: any grouping of
    the tiles (CTAs, GPUs) gives the same canonical total, and the device's
    join of it matches the exact sum to double rounding."""
    from fractions import Fraction

    rng = np.random.default_rng(0)
    tiles = rng.standard_normal(4000) * 10.0 ** rng.integers(-6, 4, 4000)
    words = [_fx_split(float(v)) for v in tiles]
    exact = sum(Fraction(h, 1024) + Fraction(l, 2 ** 61) for h, l in words)
    canon = None
    for world in (1, 2, 3, 8):
        parts = np.array_split(np.arange(len(words)), world)
        tot_hi = tot_lo = 0
        for part in parts:
            h = sum(words[i][0] for i in part)
            l = sum(words[i][1] for i in part)
            tot_hi += h + (l >> 51)  # per-GPU canonical pair (python >> is floor)
            tot_lo += l & ((1 << 51) - 1)
        hi, lo = tot_hi + (tot_lo >> 51), tot_lo & ((1 << 51) - 1)
        assert Fraction(hi, 1024) + Fraction(lo, 2 ** 61) == exact
        canon = canon or (hi, lo)
        assert (hi, lo) == canon
    # rounding below 2^-61 per tile is the only error
    assert abs(Fraction(math.fsum(tiles)) - exact) <= Fraction(1, 2 ** 40) * max(1, abs(exact)) + len(tiles) * Fraction(1, 2 ** 61)


def test_totals_to_potential_gradient_host_restatement():
    p = 3
    q = np.array([0.5, -1.0, 2.0, 0.25])
    sums = [1.5, -2.25, 3.0, 0.75, -10.5]  # 3 features, residual sum, log-likelihood
    w = np.zeros(2 * (p + 2) + 1, dtype=np.uint64)
    for d, v in enumerate(sums):
        h, l = _fx_split(v)
        w[2 * d] = np.uint64(h & (2 ** 64 - 1))
        w[2 * d + 1] = np.uint64(l & (2 ** 64 - 1))
    out = ts.rowshard.totals_to_potential_gradient(w, q)
    prior = 0.5 * q[3] * q[3] + sum(0.5 * q[d] * q[d] for d in range(3))
    assert out[0] == prior - sums[4]
    assert np.array_equal(out[1:], q - np.asarray(sums[:4]))
    w[-1] = 1  # out-of-range flag
    assert np.isnan(ts.rowshard.totals_to_potential_gradient(w, q)[1:]).all()


def _handle_worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gather = ts.rowshard.torch_all_gather()
    got = gather(bytes([rank]) * ts.rowshard.HANDLE_BYTES)
    if rank == 0:
        np.save(out_path, np.frombuffer(b"".join(got), dtype=np.uint8))
    dist.destroy_process_group()


def test_row_shard_handle_exchange_two_ranks(tmp_path):
    out = str(tmp_path / "handles.npy")
    mp.spawn(_handle_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    assert got.size == 2 * ts.rowshard.HANDLE_BYTES
    assert (got[:64] == 0).all() and (got[64:] == 1).all()
