"""Multi-chain runs on the device, with the reference's deterministic keys.

Reference: turnstile/chains.py.  ``run`` keeps the reference's API and
semantics (per-chain keys split off the seed, ``fold(10 + i)`` per draw, the
same warmup recursion), but a whole run is one device launch per GPU:
  * small models: one chain per thread, all chains of the GPU concurrently;
  * logistic regression: one persistent cooperative grid per chain.
Chains can be sharded over several GPUs (``devices=``); because every chain
is a pure function of its key, the output does not depend on the sharding
(the device analogue of the reference's sequential == parallel invariance,
tests/test_chains.py:75-91).
"""

from __future__ import annotations

import os
import threading
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .adapt import da_weights, warmup_schedule
from .integrator import MassMatrix, exec_mode_for
from .models import TargetModel, model_from_descriptor, require_device
from .rng import RngKey
from .sampler import SamplerConfig, TransitionStats
from .tree import sampler_cfg_c

MODE_SEQUENTIAL = "sequential"
MODE_PARALLEL = "parallel"

_KEY_INIT_POSITION = 0
_KEY_STEP_SIZE_SEARCH = 1
_KEY_FIRST_DRAW = 10


@dataclass(frozen=True)
class RunConfig:
    model: dict
    num_chains: int = 4
    num_warmup: int = 1000
    num_samples: int = 1000
    mode: str = MODE_SEQUENTIAL
    seed: int = 0
    sampler: Optional[SamplerConfig] = None
    target_accept: float = 0.8

    def __post_init__(self):
        if self.num_chains < 1:
            raise ValueError("num_chains must be >= 1")
        if self.num_samples < 1:
            raise ValueError("num_samples must be >= 1")
        if self.num_warmup != 0 and self.num_warmup < 20:
            raise ValueError("num_warmup must be 0 (off) or at least 20")
        if self.mode not in (MODE_SEQUENTIAL, MODE_PARALLEL):
            raise ValueError(f"unknown mode {self.mode!r}")


@dataclass
class ChainResult:
    """Samples plus per-draw statistics and the adaptation record (chains.py:60-74)."""

    chain_id: int
    samples: np.ndarray
    stats_array: np.ndarray = field(default_factory=lambda: np.zeros((0, 5)))  # sampling draws (S, 5)
    adaptation: dict = field(default_factory=dict)
    elapsed_ns: int = 0
    total_leapfrogs: int = 0
    sampling_leapfrogs: int = 0
    warmup_stats_array: Optional[np.ndarray] = None

    @property
    def stats(self) -> list:
        return [TransitionStats(int(r[0]), int(r[1]), bool(r[2]), float(r[3]), float(r[4])) for r in self.stats_array]

    @property
    def divergences(self) -> int:
        return int(np.count_nonzero(self.stats_array[:, 2]))


def shard_range(num_chains: int, rank: int, world: int) -> list[int]:
    """Chain ids owned by GPU/rank `rank` of `world`: a contiguous block.

    Chains are independent and each is a pure function of its key, so any
    partition gives the same per-chain output (no collective needed)."""
    if not 0 <= rank < world:
        raise ValueError("rank must lie in [0, world)")
    return list(range(rank * num_chains // world, (rank + 1) * num_chains // world))


def chain_keys(seed: int, num_chains: int) -> list[RngKey]:
    carry = RngKey.from_seed(seed)
    keys = []
    for _ in range(num_chains):
        key, carry = carry.split()
        keys.append(key)
    return keys


def _base_config(config: RunConfig, model: TargetModel) -> SamplerConfig:
    if config.sampler is not None:
        if config.sampler.mass.dim != model.dim:
            raise ValueError(
                f"mass matrix dimension {config.sampler.mass.dim} does not match model dimension {model.dim}"
            )
        return config.sampler
    return SamplerConfig(step_size=1.0, mass=MassMatrix.identity(model.dim))


class DeviceRun:
    """Raw device outputs of one run on one GPU (arrays stay on the device
    until ``fetch``)."""

    def __init__(self, samples, stats, adapt, status, evals, event_ms):
        self.samples = samples
        self.stats = stats
        self.adapt = adapt
        self.status = status
        self.evals = evals
        self.event_ms = event_ms


def run_device(model: TargetModel, config: RunConfig, keys: Sequence[RngKey], device=None, exec_mode=None,
               sync: bool = True, base: Optional[SamplerConfig] = None, keep_warmup: bool = False):
    """Launch the whole warmup + sampling run for ``keys`` on one GPU.

    Returns torch tensors (samples (C,S,D), stats (C,W+S,5), adapt (C,2+W+D),
    status (C,)) still on the device, plus the device time of the launch.
    ``keep_warmup``: samples is (C,W+S,D), the warmup draws first (the
    positions the Welford windows saw; adaptation audits).

    ``base`` overrides the start configuration (run_chain's argument) without
    counting as a user ``config.sampler``: with ``num_warmup == 0`` the
    step-size search still runs unless ``config.sampler`` is set
    (chains.py:132-138).
    """
    spec = require_device(model)
    torch = _lib.torch_cuda()
    dev = _lib.cuda_device(torch, device)
    if base is None:
        base = _base_config(config, model)
    elif base.mass.dim != model.dim:
        raise ValueError(f"mass matrix dimension {base.mass.dim} does not match model dimension {model.dim}")
    C, W, S, D = len(keys), config.num_warmup, config.num_samples, model.dim
    handle = spec.handle(dev)
    with torch.cuda.device(dev):
        kd = torch.tensor(np.array([[k.hi, k.lo] for k in keys], dtype=np.uint64).view(np.int64), device=dev)
        inv0 = torch.from_numpy(base.mass.inv_diag).to(dev)
        if W > 0:
            flags = warmup_schedule(W).device_flags()
            if spec.reparam is not None:
                # a fixed dense mass (dense_gaussian_model): warmup adapts the step size only
                flags = np.zeros_like(flags)
            sched = torch.from_numpy(flags).to(dev)
            weights = torch.from_numpy(da_weights(W)).to(dev)
        else:
            sched = weights = None
        samples = torch.empty((C, S + (W if keep_warmup else 0), D), dtype=torch.float64, device=dev)
        stats = torch.empty((C, W + S, 5), dtype=torch.float64, device=dev)
        adapt = torch.zeros((C, 2 + W + D), dtype=torch.float64, device=dev)
        status = torch.zeros(C, dtype=torch.int32, device=dev)
        evals = torch.zeros(C, dtype=torch.int64, device=dev)
        rc = _lib.RunCfgC(W, S, float(config.target_accept), 1 if config.sampler is not None else 0,
                          1 if keep_warmup else 0,
                          sampler_cfg_c(base))
        lib = _lib.load_library()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        _lib.check(lib.ts_run_chains(handle, rc, _lib.ptr(kd), C, _lib.ptr(inv0), _lib.ptr(sched), _lib.ptr(weights),
                                     _lib.ptr(samples), _lib.ptr(stats), _lib.ptr(adapt), _lib.ptr(status), _lib.ptr(evals),
                                     exec_mode_for(model, exec_mode), _lib.stream_ptr(torch)))
        t1.record()
        if spec.reparam is not None:  # x -> q = L x (dense mass reparametrisation), ts_dense_transform
            Ld = torch.from_numpy(np.ascontiguousarray(spec.reparam)).to(dev)
            q = torch.empty_like(samples)
            _lib.check(lib.ts_dense_transform(_lib.ptr(Ld), _lib.ptr(samples), _lib.ptr(q), samples.numel() // D, D,
                                              _lib.stream_ptr(torch)))
            samples = q
        ms = None
        if sync:
            t1.synchronize()
            ms = t0.elapsed_time(t1)
    return DeviceRun(samples, stats, adapt, status, evals, ms if sync else (t0, t1))


def _results(chain_ids, run: DeviceRun, config: RunConfig, D: int, wall_ns: int) -> list[ChainResult]:
    """Per-chain results of one launch.  The launch's wall time ``wall_ns`` is
    shared out over its chains (remainder to the first ones), so that summing
    ``elapsed_ns`` over chains -- as ``summarize`` does, diagnostics.py:142-155
    -- gives the device time spent, not num_chains times it."""
    W, S = config.num_warmup, config.num_samples
    n = len(chain_ids)
    share = [wall_ns // n + (1 if i < wall_ns % n else 0) for i in range(n)]
    samples = run.samples.cpu().numpy()
    stats = run.stats.cpu().numpy()
    adapt = run.adapt.cpu().numpy()
    status = run.status.cpu().numpy()
    out = []
    for i, c in enumerate(chain_ids):
        if status[i] == _lib.TS_STATUS_SYNC_TIMEOUT:
            raise RuntimeError(_lib.SYNC_TIMEOUT_MSG)
        if status[i] != 0:
            raise ValueError("inverse mass diagonal must be positive and finite")
        st = stats[i]
        a = adapt[i]
        if W > 0:
            adaptation = {
                "initial_step_size": float(a[0]),
                "step_size_trace": a[2:2 + W].tolist(),
                "final_step_size": float(a[1]),
                "inv_mass_diag": a[2 + W:].tolist(),
            }
        else:
            adaptation = {"final_step_size": float(a[1]), "inv_mass_diag": a[2:2 + D].tolist()}
        total = int(st[:, 1].sum())
        samp = int(st[W:, 1].sum())
        out.append(ChainResult(c, samples[i], st[W:].copy(), adaptation, share[i], total, samp, st[:W].copy()))
    return out


def run_chain(chain_id: int, key: RngKey, model: TargetModel, config: RunConfig, base: SamplerConfig,
              device=None) -> ChainResult:
    """Warm up and sample one chain on the device (chains.py:98-163)."""
    t0 = time.perf_counter_ns()
    r = run_device(model, config, [key], device, base=base)
    return _results([chain_id], r, config, model.dim, time.perf_counter_ns() - t0)[0]


def run(config: RunConfig, model: Optional[TargetModel] = None, devices: Optional[Sequence] = None,
        exec_mode=None) -> list[ChainResult]:
    """Run all chains on the device(s); results are identical for any sharding."""
    if model is None:
        model = model_from_descriptor(config.model)
    require_device(model)
    _base_config(config, model)
    keys = chain_keys(config.seed, config.num_chains)
    torch = _lib.torch_cuda()
    if devices is None:
        devices = [torch.cuda.current_device()]
    devices = list(devices)
    C = config.num_chains
    shards = [shard_range(C, g, len(devices)) for g in range(len(devices))]
    runs: list = [None] * len(devices)
    walls: list = [0] * len(devices)
    errors: list = []

    def work(g):
        try:
            if shards[g]:
                t0 = time.perf_counter_ns()
                runs[g] = run_device(model, config, [keys[c] for c in shards[g]], devices[g], exec_mode)
                walls[g] = time.perf_counter_ns() - t0
        except BaseException as e:  # surfaced below
            errors.append(e)

    if len(devices) == 1:
        work(0)
    else:
        threads = [threading.Thread(target=work, args=(g,)) for g in range(len(devices))]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    if errors:
        raise errors[0]
    results: list[ChainResult] = []
    for g in range(len(devices)):
        if shards[g]:
            results += _results(shards[g], runs[g], config, model.dim, walls[g])
    return results


def run_sharded(config: RunConfig, model: Optional[TargetModel] = None, rank: int = 0, world: int = 1, device=None,
                exec_mode=None) -> list[ChainResult]:
    """This process's share of ``run(config)`` when one process drives each
    GPU (torch.distributed-style launch): chains ``shard_range(C, rank,
    world)`` on ``device``.  Concatenating the ranks' results in rank order
    gives exactly ``run(config)`` (chains are pure functions of their keys)."""
    if model is None:
        model = model_from_descriptor(config.model)
    require_device(model)
    _base_config(config, model)
    keys = chain_keys(config.seed, config.num_chains)
    ids = shard_range(config.num_chains, rank, world)
    if not ids:
        return []
    t0 = time.perf_counter_ns()
    r = run_device(model, config, [keys[c] for c in ids], device, exec_mode)
    return _results(ids, r, config, model.dim, time.perf_counter_ns() - t0)


def run_dense_adapted(precision_matrix, config: RunConfig, pilot: Optional[RunConfig] = None,
                      precision: str = "tf32", device=None):
    """Dense-mass NUTS for the correlated-Gaussian model in two device runs.

    1. pilot run (identity mass, step-size warmup) of ``pilot`` (default:
       ``config``) - its draws stay in HBM;
    2. ``pooled_covariance`` of the pilot draws over all chains (regularised)
       becomes the dense inverse mass M^-1;
    3. the sampling run of ``config`` on ``dense_gaussian_model(P, M^-1)``.

    Returns (model, inv_mass (D, D) numpy, DeviceRun).  The reference adapts
    a diagonal mass per chain only (adapt.py:73-108); this is SURVEY.md 8(f)
    item 3, pooled across the chains of config 4.
    """
    from .adapt import pooled_covariance
    from .models import dense_gaussian_model

    pilot = config if pilot is None else pilot
    keys = chain_keys(pilot.seed, pilot.num_chains)
    first = run_device(dense_gaussian_model(precision_matrix, precision=precision), pilot, keys, device)
    _, cov = pooled_covariance(first.samples, regularize=True)
    inv_mass = cov.cpu().numpy()
    model = dense_gaussian_model(precision_matrix, inv_mass=inv_mass, precision=precision)
    final = run_device(model, config, chain_keys(config.seed + 1, config.num_chains), device)
    return model, inv_mass, final
