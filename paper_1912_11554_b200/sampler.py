"""Single NUTS transitions, executed on the device.

Reference: turnstile/sampler.py.  ``nuts_transition_from`` keeps the
reference signature (sampler.py:83-88) and runs
csrc/ts_engine.cuh::transition: momentum refresh (device ziggurat normals
bit-identical to numpy's, or injected), the doubling loop with direction
draws, the iterative builder per doubling, biased progressive acceptance and
the outer U-turn test, in one launch.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .integrator import MassMatrix, PhasePoint, exec_mode_for, pack
from .models import TargetModel, require_device
from .rng import RngKey
from .tree import CLASSIC, GENERALIZED, build_tree_iterative, build_tree_recursive, sampler_cfg_c
from .treemath import MAX_TREE_DEPTH_LIMIT

RECURSIVE = "recursive"
ITERATIVE = "iterative"


@dataclass(frozen=True)
class SamplerConfig:
    """Knobs shared by the tree builder and the transition kernel (sampler.py:38-69)."""

    step_size: float
    mass: MassMatrix
    max_tree_depth: int = 10
    criterion: str = GENERALIZED
    divergence_threshold: float = 1000.0
    tree_builder: str = ITERATIVE

    def __post_init__(self):
        if not (self.step_size > 0 and math.isfinite(self.step_size)):
            raise ValueError("step_size must be positive and finite")
        if not 1 <= self.max_tree_depth <= MAX_TREE_DEPTH_LIMIT:
            raise ValueError(f"max_tree_depth must be in [1, {MAX_TREE_DEPTH_LIMIT}]")
        if self.criterion not in (CLASSIC, GENERALIZED):
            raise ValueError(f"unknown criterion {self.criterion!r}")
        if self.tree_builder not in (RECURSIVE, ITERATIVE):
            raise ValueError(f"unknown tree builder {self.tree_builder!r}")
        if self.divergence_threshold <= 0:
            raise ValueError("divergence_threshold must be positive")

    @property
    def build_tree(self):
        return build_tree_recursive if self.tree_builder == RECURSIVE else build_tree_iterative

    def with_step_size(self, step_size: float) -> "SamplerConfig":
        return replace(self, step_size=step_size)

    def with_mass(self, mass: MassMatrix) -> "SamplerConfig":
        return replace(self, mass=mass)


@dataclass(frozen=True)
class TransitionStats:
    depth_reached: int
    leapfrog_calls: int
    diverged: bool
    accept_stat: float
    energy: float


@dataclass(frozen=True)
class TransitionTrace:
    """Per-transition decision record from the device (integer parity layer)."""

    trees: list  # (j, leapfrog_count, stop, go_right, max_occupied)
    proposals: list  # (j, leaf index, taken)
    outer_checks: list  # (j, turned)
    proposal_tree: int
    proposal_leaf: int


def nuts_transition_from(z0: PhasePoint, config: SamplerConfig, model: TargetModel, rng: RngKey, normals=None,
                         device=None, exec_mode=None, return_trace: bool = False):
    """One NUTS transition from a phase point with cached gradient (device).

    ``normals`` optionally injects the momentum refresh's standard normals
    (otherwise drawn on the device from rng.fold(0), as numpy would).

    Returns ``(z1, stats)``.  ``z1`` carries the proposal's position,
    potential and gradient; unlike the reference (whose proposal PhasePoint
    keeps the leaf's momentum, sampler.py:139-148) its momentum is zeros:
    the device engine does not carry a momentum vector per stored proposal
    (one D-vector copy fewer per merge on the hot path), and the next
    transition resamples the momentum anyway (sampler.py:95).  The proposal's
    total energy is ``stats.energy``.
    """
    if not isinstance(rng, RngKey):
        raise ValueError("rng must be an RngKey")
    spec = require_device(model)
    torch = _lib.torch_cuda()
    dev = _lib.cuda_device(torch, device)
    h = spec.handle(dev)
    D = model.dim
    zin = torch.from_numpy(pack(z0)).to(dev)
    inv = torch.from_numpy(config.mass.inv_diag).to(dev)
    nrm = None
    if normals is not None:
        nrm = torch.from_numpy(np.ascontiguousarray(normals, dtype=np.float64).ravel()).to(dev)
        if nrm.numel() != D:
            raise ValueError("normals must have the model dimension")
    out = torch.empty(2 * D + 8, dtype=torch.float64, device=dev)
    ev = counts = None
    cap = 0
    if return_trace:
        cap = 8 * config.max_tree_depth + 16
        ev = torch.zeros((cap, 5), dtype=torch.int32, device=dev)
        counts = torch.zeros(3, dtype=torch.int32, device=dev)
    lib = _lib.load_library()
    with torch.cuda.device(dev):
        _lib.check(lib.ts_transition(h, sampler_cfg_c(config), _lib.ptr(inv), _lib.ptr(zin), _lib.ptr(nrm), rng.hi, rng.lo,
                                     _lib.ptr(out), _lib.ptr(ev), cap, _lib.ptr(counts), exec_mode_for(model, exec_mode),
                                     _lib.stream_ptr(torch)))
    o = out.cpu().numpy()
    _lib.check_spec(model.device_spec, h)
    s = o[2 * D:]
    z = PhasePoint(o[:D].copy(), np.zeros(D), float(s[0]), o[D:2 * D].copy())
    stats = TransitionStats(int(s[1]), int(s[2]), bool(s[3]), float(s[4]), float(s[5]))
    if not return_trace:
        return z, stats
    c = counts.cpu().numpy()
    trees, props, outer = [], [], []
    from .tree import EV_OUTER, EV_PROPOSAL, EV_TREE_END

    for kind, a, b, cc, e in ev.cpu().numpy()[: min(int(c[0]), cap)].tolist():
        if kind == EV_TREE_END:
            trees.append((a, b, cc // 16, cc % 16, e))
        elif kind == EV_PROPOSAL:
            props.append((a, b, cc))
        elif kind == EV_OUTER:
            outer.append((a, b))
    return z, stats, TransitionTrace(trees, props, outer, int(s[6]), int(s[7]))


def nuts_transition(q: np.ndarray, config: SamplerConfig, model: TargetModel, rng: RngKey):
    """Position-in/position-out wrapper (sampler.py:151-160)."""
    z0 = PhasePoint.from_position(model, q, np.zeros(model.dim))
    z_new, stats = nuts_transition_from(z0, config, model, rng)
    return z_new.position, stats


def hmc_transition(q, config: SamplerConfig, model: TargetModel, rng: RngKey, num_steps: int, normals=None,
                   device=None, exec_mode=None):
    """Fixed-length HMC baseline (sampler.py:163-203), on the device:
    ``num_steps`` leapfrogs then accept/reject.  Returns (position, stats)."""
    if num_steps < 1:
        raise ValueError("num_steps must be >= 1")
    if not isinstance(rng, RngKey):
        raise ValueError("rng must be an RngKey")
    spec = require_device(model)
    torch = _lib.torch_cuda()
    dev = _lib.cuda_device(torch, device)
    h = spec.handle(dev)
    D = model.dim
    q = np.asarray(q, dtype=np.float64)
    z0 = PhasePoint.from_position(model, q, np.zeros(D))
    zin = torch.from_numpy(pack(z0)).to(dev)
    inv = torch.from_numpy(config.mass.inv_diag).to(dev)
    nrm = None
    if normals is not None:
        nrm = torch.from_numpy(np.ascontiguousarray(normals, dtype=np.float64).ravel()).to(dev)
        if nrm.numel() != D:
            raise ValueError("normals must have the model dimension")
    out = torch.empty(2 * D + 7, dtype=torch.float64, device=dev)
    lib = _lib.load_library()
    with torch.cuda.device(dev):
        _lib.check(lib.ts_hmc_transition(h, sampler_cfg_c(config), _lib.ptr(inv), _lib.ptr(zin), _lib.ptr(nrm), rng.hi,
                                         rng.lo, int(num_steps), _lib.ptr(out), exec_mode_for(model, exec_mode),
                                         _lib.stream_ptr(torch)))
    o = out.cpu().numpy()
    s = o[2 * D:]
    stats = TransitionStats(int(s[1]), int(s[2]), bool(s[3]), float(s[4]), float(s[5]))
    return (o[:D].copy() if s[6] != 0 else q), stats
