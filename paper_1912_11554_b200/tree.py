"""Trajectory trees: the iterative builder, executed on the device.

Reference: turnstile/tree.py.  ``build_tree_iterative`` keeps the reference
signature (tree.py:344-353) and runs csrc/ts_engine.cuh::build_tree: the
leaf loop, the popcount/trailing-ones slot schedule, multinomial merges, the
U-turn checks and the divergence exit all happen inside one kernel launch;
the tree's uniforms are regenerated on the device from the Philox key
(bit-identical to numpy's stream).  A ``TreeTrace`` passed in is filled from
the device trace buffer with the reference's event schema.

The recursive builder is the reference's host-only oracle (SURVEY.md 2.1
row 5); the two are bitwise interchangeable by the reference's own
acceptance criterion 1, so ``build_tree_recursive`` maps onto the same device
builder.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional, Union

import numpy as np

from . import _lib
from .integrator import MassMatrix, PhasePoint, exec_mode_for, hamiltonian, pack
from .models import TargetModel, require_device
from .rng import RngKey
from .treemath import MAX_TREE_DEPTH_LIMIT

CLASSIC = "classic"
GENERALIZED = "generalized"

EV_WRITE, EV_CHECK, EV_TREE_END, EV_PROPOSAL, EV_OUTER = 1, 2, 3, 4, 5


@dataclass(frozen=True)
class Tree:
    """Summary of a (sub)trajectory (tree.py:65-85); plus the proposal leaf index."""

    left: PhasePoint
    right: PhasePoint
    proposal: PhasePoint
    log_weight: float
    turning: bool
    diverging: bool
    leapfrog_count: int
    momentum_sum: np.ndarray
    sum_metropolis: float
    proposal_leaf: int = -1


def check_uturn(left: PhasePoint, right: PhasePoint, mass: MassMatrix, criterion: str, momentum_sum=None) -> bool:
    """U-turn test across endpoints given in time order (tree.py:88-109)."""
    if criterion == GENERALIZED:
        if momentum_sum is None:
            raise ValueError("generalized criterion requires the momentum sum")
        rho = np.asarray(momentum_sum, dtype=np.float64)
    elif criterion == CLASSIC:
        rho = right.position - left.position
    else:
        raise ValueError(f"unknown criterion {criterion!r}")
    a = b = 0.0
    for x, iv, rl, rr in zip(rho.tolist(), mass.inv_diag.tolist(), left.momentum.tolist(), right.momentum.tolist()):
        a += x * iv * rl
        b += x * iv * rr
    return a < 0.0 or b < 0.0


@dataclass
class TreeTrace:
    """Instrumentation of one build (tree.py:165-187), filled from the device."""

    writes: list = field(default_factory=list)
    checks: list = field(default_factory=list)
    leaf_log_weights: list = field(default_factory=list)
    max_occupied: int = 0

    def storage_trace(self) -> list:
        events: dict = {}
        for n, slot in self.writes:
            events[(n, "write")] = [slot]
        for n, slot, _leaf in self.checks:
            events.setdefault((n, "check"), []).append(slot)
        return [(kind, n, slots) for (n, kind), slots in sorted(events.items())]


def _validate(depth: int, config) -> None:
    if depth < 0:
        raise ValueError("depth must be non-negative")
    if depth > config.max_tree_depth:
        raise ValueError(f"depth {depth} exceeds max_tree_depth {config.max_tree_depth}")
    if depth > MAX_TREE_DEPTH_LIMIT:
        raise ValueError(f"depth {depth} exceeds the hard limit {MAX_TREE_DEPTH_LIMIT}")


def sampler_cfg_c(config) -> _lib.SamplerCfgC:
    return _lib.SamplerCfgC(
        float(config.step_size),
        int(config.max_tree_depth),
        _lib.TS_GENERALIZED if config.criterion == GENERALIZED else _lib.TS_CLASSIC,
        float(config.divergence_threshold),
    )


def _key_of(rng) -> RngKey:
    if isinstance(rng, RngKey):
        return rng
    raise ValueError("the device builder needs an RngKey (its stream is regenerated on the GPU)")


def build_tree_iterative(
    z: PhasePoint,
    depth: int,
    eps: float,
    config,
    model: TargetModel,
    rng: Union[RngKey, object],
    h_ref: Optional[float] = None,
    trace: Optional[TreeTrace] = None,
    device=None,
    exec_mode=None,
) -> Tree:
    """Iterative builder with one storage slot per tree level, on the device."""
    _validate(depth, config)
    key = _key_of(rng)
    spec = require_device(model)
    if h_ref is None:
        h_ref = hamiltonian(z, config.mass)
    torch = _lib.torch_cuda()
    dev = _lib.cuda_device(torch, device)
    handle = spec.handle(dev)
    D = model.dim
    zin = torch.from_numpy(pack(z)).to(dev)
    inv = torch.from_numpy(config.mass.inv_diag).to(dev)
    out = torch.empty(8 * D + 10, dtype=torch.float64, device=dev)
    ev = lw = counts = None
    cap = lw_cap = 0
    if trace is not None:
        cap = 4 * (1 << depth) + 16
        lw_cap = (1 << depth) + 1
        ev = torch.zeros((cap, 5), dtype=torch.int32, device=dev)
        lw = torch.zeros(lw_cap, dtype=torch.float64, device=dev)
        counts = torch.zeros(3, dtype=torch.int32, device=dev)
    cfg = sampler_cfg_c(config)
    lib = _lib.load_library()
    with torch.cuda.device(dev):
        _lib.check(lib.ts_build_tree(handle, cfg, _lib.ptr(inv), _lib.ptr(zin), int(depth), float(eps), float(h_ref),
                                     key.hi, key.lo, _lib.ptr(out), _lib.ptr(ev), cap, _lib.ptr(lw), lw_cap,
                                     _lib.ptr(counts), exec_mode_for(model, exec_mode), _lib.stream_ptr(torch)))
    o = out.cpu().numpy()
    _lib.check_spec(model.device_spec, handle)
    v = [o[k * D:(k + 1) * D].copy() for k in range(8)]
    s = o[8 * D:]
    left = PhasePoint(v[0], v[1], float(s[8]), np.full(D, np.nan))
    right = PhasePoint(v[2], v[3], float(s[9]), v[4])
    proposal = PhasePoint(v[5], np.full(D, np.nan), float(s[5]), v[6])
    if trace is not None:
        c = counts.cpu().numpy()
        e = ev.cpu().numpy()[: min(int(c[0]), cap)]
        for kind, a, b, cc, _ in e.tolist():
            if kind == EV_WRITE:
                trace.writes.append((a, b))
            elif kind == EV_CHECK:
                trace.checks.append((a, b, cc))
        trace.leaf_log_weights.extend(lw.cpu().numpy()[: min(int(c[1]), lw_cap)].tolist())
        trace.max_occupied = max(trace.max_occupied, int(c[2]))
    return Tree(
        left=left,
        right=right,
        proposal=proposal,
        log_weight=float(s[0]),
        turning=bool(s[3]),
        diverging=bool(s[4]),
        leapfrog_count=int(s[2]),
        momentum_sum=v[7],
        sum_metropolis=float(s[1]),
        proposal_leaf=int(s[7]),
    )


def build_tree_recursive(z, depth, eps, config, model, rng, h_ref=None, trace=None, device=None, exec_mode=None) -> Tree:
    """Same tree as the reference's recursive oracle (bitwise-equal builders,
    reference acceptance criterion 1); served by the device iterative builder.
    The storage trace is that of the iterative schedule."""
    return build_tree_iterative(z, depth, eps, config, model, rng, h_ref, trace, device, exec_mode)


def trees_equal(a: Tree, b: Tree) -> bool:
    """Bitwise agreement on the fields both builders promise (tree.py:456-478)."""

    def arr_eq(x, y):
        return bool(np.array_equal(x, y, equal_nan=True))

    def pp_eq(x, y):
        return arr_eq(x.position, y.position) and (
            x.potential == y.potential or (math.isnan(x.potential) and math.isnan(y.potential))
        )

    return (
        pp_eq(a.left, b.left)
        and arr_eq(a.left.momentum, b.left.momentum)
        and pp_eq(a.right, b.right)
        and arr_eq(a.right.momentum, b.right.momentum)
        and pp_eq(a.proposal, b.proposal)
        and a.log_weight == b.log_weight
        and a.turning == b.turning
        and a.diverging == b.diverging
        and a.leapfrog_count == b.leapfrog_count
        and arr_eq(a.momentum_sum, b.momentum_sum)
    )
