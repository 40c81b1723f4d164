"""CPU oracle: a plain-Python/numpy restatement of the reference's hot path.

TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke() and
the cpu_baseline / --impl reference legs of bench.py, always as the checker
or the timed CPU baseline, never by the product package.

What it restates (reference = turnstile @ /root/reference/pkg/src):
  philox/stream/ziggurat  numpy Philox4x64-10 + Generator.random/standard_normal,
                          as used by turnstile/rng.py:36-73 (numpy is the
                          third-party dependency; its algorithm is restated
                          here and pinned against numpy itself)
  small-model kernels     turnstile/kernels.py:44-88 (numba loop order)
  logistic kernels        turnstile/kernels.py:90-123 via oracle/logistic_ref.c
  leapfrog / energy       turnstile/integrator.py:82-108, kernels.py:125-165
  iterative tree          turnstile/tree.py:344-453 (+ _merge 140-156,
                          merge_out 395-400), with trace and proposal leaf
  transition              turnstile/sampler.py:83-148
  step-size search, DA,   turnstile/adapt.py:28-236
  Welford, schedule
  run_chain / run         turnstile/chains.py:77-191
Arithmetic is written in the same association as the reference (Python
floats are IEEE doubles without FMA), so small-model results agree with the
reference's numba path bit for bit; tests/test_oracle.py pins this against
the golden fixtures generated from the reference (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

INF = math.inf
M64 = (1 << 64) - 1

# ----------------------------------------------------------------------------- rng


def philox4x64_10(ctr, key):
    """Ten Philox4x64 rounds (numpy/random/src/philox/philox.h)."""
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for _ in range(10):
        p0 = 0xD2E7470EE14C6C93 * c0
        p1 = 0xCA5A826395121157 * c2
        c0, c1, c2, c3 = ((p1 >> 64) ^ c1 ^ k0) & M64, p1 & M64, ((p0 >> 64) ^ c3 ^ k1) & M64, p0 & M64
        k0 = (k0 + 0x9E3779B97F4A7C15) & M64
        k1 = (k1 + 0xBB67AE8584CAA73B) & M64
    return (c0, c1, c2, c3)


def key_from_seed(seed):
    """RngKey.from_seed (rng.py:46-49): counter (seed >> 64, 0, 0, 0), pre-incremented."""
    w = philox4x64_10((((seed >> 64) & M64) + 1, 0, 0, 0), (0x9E3779B97F4A7C15, seed & M64))
    return (w[0], w[1])


def key_split(key):
    w = philox4x64_10((1, 0, 0, 2), key)
    return (w[0], w[1]), (w[2], w[3])


def key_fold(key, i):
    c0 = (i + 1) & M64
    c1 = ((i >> 64) + (1 if c0 == 0 else 0)) & M64
    w = philox4x64_10((c0, c1, 0, 3), key)
    return (w[0], w[1])


def chain_keys(seed, n):
    carry = key_from_seed(seed)
    out = []
    for _ in range(n):
        k, carry = key_split(carry)
        out.append(k)
    return out


_ZIG = None


def _zig_tables():
    """numpy's ziggurat tables, read out of numpy's own shared object."""
    global _ZIG
    if _ZIG is None:
        import importlib.util
        import sys

        here = os.path.dirname(os.path.abspath(__file__))
        gen = os.path.join(here, "..", "paper_1912_11554_b200", "csrc", "gen_ziggurat.py")
        spec = importlib.util.spec_from_file_location("_gen_zig", gen)
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        ki, wi, fi = mod.extract()
        _ZIG = (ki.tolist(), wi.tolist(), fi.tolist())
    return _ZIG


class Stream:
    """RngKey.generator(): numpy Philox stream starting at counter (0, 0, 0, 1)."""

    def __init__(self, key):
        self.key = key
        self.c0 = 0
        self.c1 = 0
        self.buf = (0, 0, 0, 0)
        self.pos = 4

    def u64(self):
        if self.pos < 4:
            v = self.buf[self.pos]
            self.pos += 1
            return v
        self.c0 = (self.c0 + 1) & M64
        if self.c0 == 0:
            self.c1 = (self.c1 + 1) & M64
        self.buf = philox4x64_10((self.c0, self.c1, 0, 1), self.key)
        self.pos = 1
        return self.buf[0]

    def random(self):
        return (self.u64() >> 11) * (1.0 / 9007199254740992.0)

    def normal(self):
        ki, wi, fi = _zig_tables()
        r_tail, inv_r = 3.6541528853610088, 0.27366123732975828
        while True:
            r = self.u64()
            idx = r & 0xFF
            r >>= 8
            sign = r & 1
            rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
            x = rabs * wi[idx]
            if sign:
                x = -x
            if rabs < ki[idx]:
                return x
            if idx == 0:
                while True:
                    xx = -inv_r * math.log1p(-self.random())
                    yy = -math.log1p(-self.random())
                    if yy + yy > xx * xx:
                        return -(r_tail + xx) if (rabs >> 8) & 1 else r_tail + xx
            elif (fi[idx - 1] - fi[idx]) * self.random() + fi[idx] < math.exp(-0.5 * x * x):
                return x


# ----------------------------------------------------------------------------- models


def _lib():
    here = os.path.dirname(os.path.abspath(__file__))
    so = os.path.join(here, "_ref", "liboracle.so")
    if not os.path.exists(so):
        build_c()
    lib = ctypes.CDLL(so)
    P, I64, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    lib.ts_oracle_logistic_potential_seq.restype = ctypes.c_double
    lib.ts_oracle_logistic_potential_seq.argtypes = [P, P, I64, I, P]
    lib.ts_oracle_logistic_gradient_seq.argtypes = [P, P, I64, I, P, P]
    lib.ts_oracle_logistic_omp.restype = I
    lib.ts_oracle_logistic_omp.argtypes = [P, P, I64, I, P, P]
    return lib


def build_c():
    """gcc the C restatement into oracle/_ref/liboracle.so (git-ignored)."""
    here = os.path.dirname(os.path.abspath(__file__))
    os.makedirs(os.path.join(here, "_ref"), exist_ok=True)
    subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
                           os.path.join(here, "logistic_ref.c"), "-o", os.path.join(here, "_ref", "liboracle.so"),
                           "-lm"])


def _exp(x):
    """exp with IEEE overflow to +inf (numba's math.exp; Python's raises)."""
    try:
        return math.exp(x)
    except OverflowError:
        return math.inf


@dataclass
class Model:
    """Oracle model: kind + parameters; potential/gradient restate kernels.py."""

    kind: str
    dim: int
    inv_var: list = None
    x: np.ndarray = None  # float64 (N, p), fp32-exact
    y: np.ndarray = None
    es_y: list = None
    es_s: list = None
    fused_omp: bool = False  # logistic: one OpenMP pass computes U and gradient (CPU baseline)
    dense_a: list = None  # dense_gaussian: A as a list of rows (U = x'Ax/2)
    _clib: object = field(default=None, repr=False)
    _cache: tuple = field(default=None, repr=False)
    threads: int = 0

    def _fused(self, q):
        """U and gradient from ts_oracle_logistic_omp, cached for the pair of calls
        integrator.leapfrog makes at the same point (integrator.py:98-101)."""
        key = tuple(q)
        if self._cache is None or self._cache[0] != key:
            if getattr(self, "_x32", None) is None:
                self._x32 = np.ascontiguousarray(self.x, dtype=np.float32)
                self._y8 = np.ascontiguousarray(self.y, dtype=np.uint8)
            th = np.ascontiguousarray(q, dtype=np.float64)
            out = np.empty(self.dim + 1)
            self.threads = self.clib().ts_oracle_logistic_omp(self._x32.ctypes.data, self._y8.ctypes.data,
                                                              self.x.shape[0], self.x.shape[1], th.ctypes.data,
                                                              out.ctypes.data)
            self._cache = (key, float(out[0]), out[1:].tolist())
        return self._cache[1], self._cache[2]

    def potential(self, q):
        if self.fused_omp:
            return self._fused(q)[0]
        k = self.kind
        if k == "std_normal":
            acc = 0.0
            for v in q:
                acc += 0.5 * v * v
            return acc
        if k == "gaussian":
            acc = 0.0
            for v, iv in zip(q, self.inv_var):
                acc += 0.5 * v * v * iv
            return acc
        if k == "funnel":
            v = q[0]
            ssq = 0.0
            for x in q[1:]:
                ssq += x * x
            return v * v / 18.0 + 0.5 * (len(q) - 1) * v + 0.5 * _exp(-v) * ssq
        if k == "eight_schools":
            return eight_schools_potential(q, self.es_y, self.es_s)
        if k == "dense_gaussian":
            return dense_potential(q, self.dense_a)
        if k == "logistic_regression":
            th = np.ascontiguousarray(q, dtype=np.float64)
            lib = self.clib()
            return lib.ts_oracle_logistic_potential_seq(self.x.ctypes.data, self.y.ctypes.data, self.x.shape[0],
                                                        self.x.shape[1], th.ctypes.data)
        raise ValueError(k)

    def gradient(self, q):
        if self.fused_omp:
            return list(self._fused(q)[1])
        k = self.kind
        if k == "std_normal":
            return list(q)
        if k == "gaussian":
            return [v * iv for v, iv in zip(q, self.inv_var)]
        if k == "funnel":
            v = q[0]
            inv_scale = _exp(-v)
            out = [0.0] * len(q)
            ssq = 0.0
            for i in range(1, len(q)):
                out[i] = inv_scale * q[i]
                ssq += q[i] * q[i]
            out[0] = v / 9.0 + 0.5 * (len(q) - 1) - 0.5 * inv_scale * ssq
            return out
        if k == "eight_schools":
            return eight_schools_gradient(q, self.es_y, self.es_s)
        if k == "dense_gaussian":
            return dense_gradient(q, self.dense_a)
        if k == "logistic_regression":
            th = np.ascontiguousarray(q, dtype=np.float64)
            out = np.empty(self.dim)
            self.clib().ts_oracle_logistic_gradient_seq(self.x.ctypes.data, self.y.ctypes.data, self.x.shape[0],
                                                        self.x.shape[1], th.ctypes.data, out.ctypes.data)
            return out.tolist()
        raise ValueError(k)

    def clib(self):
        if self._clib is None:
            self._clib = _lib()
        return self._clib


def dense_gradient(x, a):
    """Dense Gaussian (no reference built-in): g = A x,
    each row summed k = 0.. in order, multiply then add -- the device's SIMT
    fp64 GEMM policy (csrc/ts_k_dense.cu dense_tile_fp64)."""
    out = []
    for row in a:
        acc = 0.0
        for av, xv in zip(row, x):
            acc = acc + av * xv
        out.append(acc)
    return out


def dense_potential(x, a):
    """U = x.g / 2 with the device's order: lane-strided partial sums over 32
    lanes, then the warp shuffle-down tree (csrc/ts_k_dense.cu DenseW::wait)."""
    g = dense_gradient(x, a)
    part = [0.0] * 32
    for d in range(len(x)):
        part[d % 32] = part[d % 32] + x[d] * g[d]
    o = 16
    while o >= 1:
        part = [part[l] + part[l + o] if l + o < 32 else part[l] for l in range(32)]
        o //= 2
    return 0.5 * part[0]


def eight_schools_potential(q, y, s):
    """Non-centred eight schools (SURVEY.md 8(d) cfg 3); same op order as csrc/ts_models.cuh."""
    mu, lt = q[0], q[1]
    tau = math.exp(lt)
    sc = tau / 5.0
    s2 = sc * sc
    ulik = 0.0
    for j in range(len(y)):
        th = q[2 + j]
        z = ((y[j] - mu) - tau * th) / s[j]
        ulik += 0.5 * th * th
        ulik += 0.5 * z * z
    return ((mu * mu) / 50.0 + math.log1p(s2) - lt) + ulik


def eight_schools_gradient(q, y, s):
    mu, lt = q[0], q[1]
    tau = math.exp(lt)
    sc = tau / 5.0
    s2 = sc * sc
    out = [0.0] * len(q)
    smu = slt = 0.0
    for j in range(len(y)):
        th = q[2 + j]
        z = ((y[j] - mu) - tau * th) / s[j]
        zs = z / s[j]
        smu += zs
        slt += zs * tau * th
        out[2 + j] = th - zs * tau
    out[0] = mu / 25.0 - smu
    out[1] = ((2.0 * s2) / (1.0 + s2) - 1.0) - slt
    return out


def model_from_desc(d):
    n = d["name"]
    if n == "std_normal":
        return Model("std_normal", d["dim"])
    if n == "gaussian":
        cov = [float(v) for v in d["cov_diag"]]
        return Model("gaussian", len(cov), inv_var=(1.0 / np.asarray(cov)).tolist())
    if n == "funnel":
        return Model("funnel", d["dim"])
    if n == "eight_schools":
        y = d.get("y", [28.0, 8.0, -3.0, 7.0, -1.0, 1.0, 18.0, 12.0])
        s = d.get("sigma", [15.0, 10.0, 16.0, 11.0, 9.0, 11.0, 10.0, 18.0])
        return Model("eight_schools", len(y) + 2, es_y=list(y), es_s=list(s))
    if n == "logistic_regression":
        x = np.ascontiguousarray(np.asarray(d["x"], dtype=np.float64))
        y = np.ascontiguousarray(np.asarray(d["y"], dtype=np.float64))
        return Model("logistic_regression", x.shape[1] + 1, x=x, y=y)
    raise ValueError(n)


# ----------------------------------------------------------------------------- integrator


@dataclass
class Point:
    q: list
    r: list
    U: float
    g: list


def kinetic(r, inv):
    acc = 0.0
    for a, b in zip(r, inv):
        acc += 0.5 * a * a * b
    return acc


def hamiltonian(U, r, inv):
    if not math.isfinite(U):
        return INF
    h = U + kinetic(r, inv)
    return h if math.isfinite(h) else INF


def leapfrog(z: Point, eps, inv, model) -> Point:
    half = 0.5 * eps
    rh = [r - half * g for r, g in zip(z.r, z.g)]
    q = [q + eps * (iv * r) for q, iv, r in zip(z.q, inv, rh)]
    U = model.potential(q)
    if not math.isfinite(U):
        U = INF
    g = list(model.gradient(q))
    r = [r - half * gg for r, gg in zip(rh, g)]
    return Point(q, r, U, g)


def uturn(rho, inv, rl, rr):
    a = b = 0.0
    for x, iv, u, v in zip(rho, inv, rl, rr):
        a += x * iv * u
        b += x * iv * v
    return a < 0.0 or b < 0.0


def uturn_margin(rho, inv, rl, rr):
    """Relative distance of a U-turn check from flipping (test diagnostics,
    not on the reference path): min over the two dot products of
    |dot| / sum|terms|, i.e. how many relative rounding units separate the
    decision from the other outcome."""
    a = b = sa = sb = 0.0
    for x, iv, u, v in zip(rho, inv, rl, rr):
        a += x * iv * u
        b += x * iv * v
        sa += abs(x * iv * u)
        sb += abs(x * iv * v)
    return min(abs(a) / sa if sa else math.inf, abs(b) / sb if sb else math.inf)


# ----------------------------------------------------------------------------- tree


@dataclass
class Sub:
    """Completed-subtree summary (generation order), cf. tree.py:112-124."""

    first: Point
    last: Point
    prop: Point
    prop_h: float
    prop_leaf: int
    lw: float
    cum_first: list
    cum_last: list
    count: int
    metro: float


def lse_inner(a, b):
    if a == -INF:
        return b
    if b == -INF:
        return a
    hi, lo = (a, b) if a >= b else (b, a)
    return hi + math.log1p(math.exp(lo - hi))


def merge(left: Sub, right: Sub, u, margins=None) -> Sub:
    lw = lse_inner(left.lw, right.lw)
    p_right = 0.0 if right.lw == -INF else math.exp(right.lw - lw)
    take_right = u < p_right
    if margins is not None:
        margins.append(("merge", abs(u - p_right)))
    src = right if take_right else left
    return Sub(left.first, right.last, src.prop, src.prop_h, src.prop_leaf, lw, left.cum_first, right.cum_last,
               left.count + right.count, left.metro + right.metro)


def seg_sum(s: Sub):
    return [(a - b) + c for a, b, c in zip(s.cum_last, s.cum_first, s.first.r)]


@dataclass
class TreeResult:
    sub: Sub
    turning: bool
    diverging: bool
    msum: list
    writes: list
    checks: list
    leaf_lw: list
    max_occupied: int


def build_tree(z: Point, depth, eps, inv, model, key, h_ref, generalized=True, threshold=1000.0,
               margins=None) -> TreeResult:
    """Iterative builder (tree.py:344-453): slot s holds the latest even leaf
    with popcount s plus its completed subtree; odd leaf n merges and checks
    slots popcount(n)-1 down to popcount(n)-trailing_ones(n).

    ``margins`` (test diagnostics): a list that receives (kind, margin) for
    every floating-point decision - merges |u - p_right|, U-turn checks
    (uturn_margin), divergence |dH - threshold| / |threshold|."""
    st = Stream(key)
    D = len(z.q)
    cum = [0.0] * D
    cur = z
    slots: dict = {}
    slot_leaf: dict = {}
    writes, checks, lws = [], [], []
    forward = eps > 0

    def leaf(n):
        nonlocal cur, cum
        cur = leapfrog(cur, eps, inv, model)
        cum = [a + b for a, b in zip(cum, cur.r)]
        h = hamiltonian(cur.U, cur.r, inv)
        delta = h - h_ref
        div = not (math.isfinite(delta) and delta <= threshold)
        if margins is not None and math.isfinite(delta):
            margins.append(("divergence", abs(delta - threshold) / threshold))
        if div:
            lw = -INF
            metro = math.exp(-delta) if math.isfinite(delta) else 0.0
        else:
            lw = -h
            metro = math.exp(-delta) if delta > 0 else 1.0
        lws.append(lw)
        return Sub(cur, cur, cur, h, n, lw, cum, cum, 1, metro), div

    def fold_pending(start, part):
        for s in range(start - 1, -1, -1):
            part = merge(slots[s], part, st.random(), margins)
        return part

    def finish(sub, stop):
        return TreeResult(sub, stop == 1, stop == 2, seg_sum(sub), writes, checks, lws, len(slots))

    if depth == 0:
        sub, div = leaf(0)
        return finish(sub, 2 if div else 0)
    running = None
    for n in range(1 << depth):
        lf, div = leaf(n)
        pc = bin(n).count("1")
        if div:
            return finish(fold_pending(pc, lf), 2)
        if n % 2 == 0:
            slots[pc] = lf
            slot_leaf[pc] = n
            writes.append((n, pc))
            continue
        hi_slot = pc - 1
        lo_slot = hi_slot - bin(((n + 1) & ~n) - 1).count("1") + 1
        running = lf
        for s in range(hi_slot, lo_slot - 1, -1):
            checks.append((n, s, slot_leaf[s]))
            running = merge(slots[s], running, st.random(), margins)
            if generalized:
                args = (seg_sum(running), inv, running.first.r, running.last.r)
            elif forward:
                args = ([a - b for a, b in zip(running.last.q, running.first.q)], inv, running.first.r, running.last.r)
            else:
                args = ([a - b for a, b in zip(running.first.q, running.last.q)], inv, running.last.r, running.first.r)
            turned = uturn(*args)
            if margins is not None:
                margins.append(("uturn", uturn_margin(*args)))
            if turned:
                return finish(fold_pending(s, running), 1)
        slots[lo_slot] = running
    return finish(running, 0)


# ----------------------------------------------------------------------------- transition


@dataclass
class Stats:
    depth: int
    leapfrogs: int
    diverged: bool
    accept: float
    energy: float


def transition(z0: Point, step, inv, model, key, max_depth=10, generalized=True, threshold=1000.0, normals=None,
               margins=None):
    """nuts_transition_from (sampler.py:83-148); returns (point, Stats, decisions).

    ``margins`` (test diagnostics): a list that receives, per tree j, the list
    of (kind, margin) of every floating-point decision taken in it (see
    build_tree) plus the outer proposal draw and U-turn check."""
    D = len(z0.q)
    if normals is None:
        ns = Stream(key_fold(key, 0))
        normals = [ns.normal() for _ in range(D)]
    mstd = (1.0 / np.sqrt(np.asarray(inv, dtype=np.float64))).tolist()
    r0 = [a * b for a, b in zip(normals, mstd)]
    z = Point(list(z0.q), r0, z0.U, list(z0.g))
    h0 = hamiltonian(z.U, z.r, inv)
    gen = Stream(key_fold(key, 1))
    left = right = z
    prop, prop_h = z, h0
    prop_id = (-1, -1)
    lw = -h0
    rho = list(r0)
    lf, metro, diverged, depth = 0, 0.0, False, 0
    trees, outer = [], []
    for j in range(max_depth):
        go_right = gen.random() < 0.5
        eps = step if go_right else -step
        tm = None if margins is None else []
        if margins is not None:
            margins.append(tm)
        t = build_tree(right if go_right else left, j, eps, inv, model, key_fold(key, 2 + j), h0, generalized,
                       threshold, tm)
        lf += t.sub.count
        metro += t.sub.metro
        trees.append((j, int(go_right), t.sub.count, int(t.turning), int(t.diverging), t.sub.prop_leaf))
        if t.turning or t.diverging:
            diverged = diverged or t.diverging
            depth = j
            break
        u = gen.random()
        if tm is not None and t.sub.lw < lw:
            tm.append(("accept", abs(u - math.exp(t.sub.lw - lw))))
        if t.sub.lw >= lw or u < math.exp(t.sub.lw - lw):
            prop, prop_h, prop_id = t.sub.prop, t.sub.prop_h, (j, t.sub.prop_leaf)
        lw = float(np.logaddexp(lw, t.sub.lw))
        rho = [a + b for a, b in zip(rho, t.msum)]
        if go_right:
            right = t.sub.last
        else:
            left = t.sub.last
        depth = j + 1
        oargs = (rho, inv, left.r, right.r) if generalized else ([a - b for a, b in zip(right.q, left.q)], inv, left.r,
                                                                   right.r)
        turned = uturn(*oargs)
        if tm is not None:
            tm.append(("outer_uturn", uturn_margin(*oargs)))
        outer.append(int(turned))
        if turned:
            break
    st = Stats(depth, lf, diverged, metro / lf if lf else 0.0, prop_h)
    return Point(list(prop.q), [0.0] * D, prop.U, list(prop.g)), st, {"trees": trees, "outer": outer,
                                                                       "proposal": prop_id}


# ----------------------------------------------------------------------------- adaptation / run


def hmc_transition(q, step, inv, model, key, num_steps, threshold=1000.0, normals=None):
    """sampler.hmc_transition (sampler.py:163-203): returns (q, Stats, accepted)."""
    if num_steps < 1:
        raise ValueError("num_steps must be >= 1")
    D = len(q)
    if normals is None:
        ns = Stream(key_fold(key, 0))
        normals = [ns.normal() for _ in range(D)]
    mstd = (1.0 / np.sqrt(np.asarray(inv, dtype=np.float64))).tolist()
    r0 = [a * b for a, b in zip(normals, mstd)]
    z = Point(list(q), r0, model.potential(list(q)), model.gradient(list(q)))
    h0 = hamiltonian(z.U, z.r, inv)
    z_new = z
    steps = 0
    for _ in range(num_steps):
        z_new = leapfrog(z_new, step, inv, model)
        steps += 1
        if not math.isfinite(z_new.U):
            break
    h1 = hamiltonian(z_new.U, z_new.r, inv)
    delta = h1 - h0
    p_accept = math.exp(-delta) if math.isfinite(delta) and delta > 0 else (1.0 if math.isfinite(delta) else 0.0)
    accept = Stream(key_fold(key, 1)).random() < p_accept
    res = z_new if accept else z
    st = Stats(0, steps, (not math.isfinite(delta)) or delta > threshold, p_accept, hamiltonian(res.U, res.r, inv))
    return (list(z_new.q) if accept else list(q)), st, accept


def find_step_size(z: Point, inv, model, key, init=1.0, target=0.5, normals=None):
    """adapt.py:172-204 (momentum from key.generator() directly)."""
    D = len(z.q)
    if normals is None:
        ns = Stream(key)
        normals = [ns.normal() for _ in range(D)]
    mstd = (1.0 / np.sqrt(np.asarray(inv, dtype=np.float64))).tolist()
    zz = Point(list(z.q), [a * b for a, b in zip(normals, mstd)], z.U, list(z.g))
    h0 = hamiltonian(zz.U, zz.r, inv)

    def prob(eps):
        z1 = leapfrog(zz, eps, inv, model)
        h1 = hamiltonian(z1.U, z1.r, inv)
        return math.exp(min(0.0, h0 - h1)) if math.isfinite(h1) else 0.0

    eps = init
    direction = 1 if prob(eps) > target else -1
    for _ in range(64):
        nxt = eps * (2.0 ** direction)
        if not 1e-10 < nxt < 1e7:
            break
        p = prob(nxt)
        if (direction == 1 and p <= target) or (direction == -1 and p > target):
            return nxt if direction == -1 else eps
        eps = nxt
    return eps


def schedule_flags(W):
    """warmup_schedule + window_steps (adapt.py:111-169) as per-step flags."""
    init = round(0.15 * W)
    terminal = round(0.10 * W)
    middle = W - init - terminal
    reserve = middle // 10
    region = middle - reserve
    if region < 25:
        windows = [middle]
    else:
        windows, used, w = [], 0, 25
        while used + w <= region:
            windows.append(w)
            used += w
            w *= 2
        if used < region:
            windows.append(region - used)
        if reserve > 0:
            windows.append(reserve)
    flags = [0] * W
    at = init
    for w in windows:
        for i in range(at, at + w):
            flags[i] |= 1
        flags[at + w - 1] |= 2
        at += w
    return flags


class Adaptation:
    """Warmup adaptation of one chain (adapt.py:207-236): dual averaging on the
    log step size (DualAveragingState.init / da_update, adapt.py:44-70, gamma
    0.05, t0 10, kappa 0.75, clipped accept stat adapt.py:227) and the windowed
    Welford variance (welford_update adapt.py:86-94, regularized install
    adapt.py:104-108 at window ends, adapt.py:228-232)."""

    def __init__(self, eps0, W, D, target=0.8, inv0=None):
        self.mu, self.log_eps, self.log_bar, self.hbar = math.log(10.0 * eps0), math.log(eps0), 0.0, 0.0
        self.target = target
        self.flags = schedule_flags(W)
        self.D = D
        self.wc, self.mean, self.m2 = 0, [0.0] * D, [0.0] * D
        self.inv = list(inv0) if inv0 is not None else [1.0] * D
        self.installs = 0

    def step_size(self):
        return math.exp(self.log_eps)

    def final_step_size(self):
        return math.exp(self.log_bar)

    def update(self, i, accept, q):
        """After warmup transition i (0-based) with accept stat `accept` that
        moved the chain to position q."""
        a = min(1.0, max(0.0, accept))
        t = i + 1
        frac = 1.0 / (t + 10.0)
        self.hbar = (1.0 - frac) * self.hbar + frac * (self.target - a)
        self.log_eps = self.mu - math.sqrt(t) / 0.05 * self.hbar
        wgt = t ** (-0.75)
        self.log_bar = wgt * self.log_eps + (1.0 - wgt) * self.log_bar
        if self.flags[i] & 1:
            self.wc += 1
            for d in range(self.D):
                dl = q[d] - self.mean[d]
                self.mean[d] = self.mean[d] + dl / self.wc
                self.m2[d] = self.m2[d] + dl * (q[d] - self.mean[d])
        if self.flags[i] & 2 and self.wc >= 2:
            n = self.wc
            self.inv = [(n / (n + 5.0)) * (self.m2[d] / (self.wc - 1)) + (5.0 / (n + 5.0)) * 1e-3
                        for d in range(self.D)]
            self.wc, self.mean, self.m2 = 0, [0.0] * self.D, [0.0] * self.D
            self.installs += 1


def replay_adaptation(eps0, accepts, positions, target=0.8, inv0=None):
    """The adaptation recursion alone, fed another sampler's warmup accept
    stats and positions (e.g. the device's): step-size trace before each
    transition, final step size, inverse mass and the number of installs."""
    W, D = len(accepts), len(positions[0])
    ad = Adaptation(eps0, W, D, target, inv0)
    trace = []
    for i in range(W):
        trace.append(ad.step_size())
        ad.update(i, float(accepts[i]), [float(v) for v in positions[i]])
    return {"step_size_trace": trace, "final_step_size": ad.final_step_size(), "inv_mass_diag": ad.inv,
            "installs": ad.installs}


class Budget(Exception):
    """Raised by run_chain when max_leapfrogs is exhausted (bounded CPU samples)."""


def run_chain(model, key, W, S, step=1.0, inv0=None, has_sampler=False, target=0.8, max_depth=10, generalized=True,
              threshold=1000.0, max_leapfrogs=None):
    """chains.run_chain (chains.py:98-163); returns dict of samples/stats/adaptation.

    ``max_leapfrogs`` bounds the work for CPU timing samples: the run stops
    after the first transition that crosses the budget and returns what it has
    (``"truncated": True``)."""
    D = model.dim
    us = Stream(key_fold(key, 0))
    q0 = [-2.0 + 4.0 * us.random() for _ in range(D)]
    U = model.potential(q0)
    z = Point(q0, [0.0] * D, U if math.isfinite(U) else INF, list(model.gradient(q0)))
    inv = list(inv0) if inv0 is not None else [1.0] * D
    stats, trace, adaptation = [], [], {}
    if W > 0:
        eps0 = find_step_size(z, inv, model, key_fold(key, 1), init=step)
        ad = Adaptation(eps0, W, D, target, inv)
        for i in range(W):
            cur = ad.step_size()
            trace.append(cur)
            z, st, _ = transition(z, cur, inv, model, key_fold(key, 10 + i), max_depth, generalized, threshold)
            stats.append(st)
            if max_leapfrogs is not None and sum(s.leapfrogs for s in stats) >= max_leapfrogs:
                return {"samples": [], "stats": stats, "adaptation": {}, "truncated": True,
                        "total_leapfrogs": sum(s.leapfrogs for s in stats)}
            ad.update(i, st.accept, z.q)
            inv = ad.inv
        final = ad.final_step_size()
        adaptation = {"initial_step_size": eps0, "step_size_trace": trace, "final_step_size": final,
                      "inv_mass_diag": inv}
    else:
        final = step if has_sampler else find_step_size(z, inv, model, key_fold(key, 1))
        adaptation = {"final_step_size": final, "inv_mass_diag": inv}
    samples = []
    for i in range(S):
        z, st, _ = transition(z, final, inv, model, key_fold(key, 10 + W + i), max_depth, generalized, threshold)
        samples.append(list(z.q))
        stats.append(st)
        if max_leapfrogs is not None and sum(s.leapfrogs for s in stats) >= max_leapfrogs:
            break
    return {"samples": samples, "stats": stats, "adaptation": adaptation,
            "total_leapfrogs": sum(s.leapfrogs for s in stats)}


# ----------------------------------------------------------------------------- diagnostics


def ess(chains):
    """Split-chain ESS with Geyer monotone pairs (diagnostics.py:49-86)."""
    arr = np.asarray(chains, dtype=np.float64)
    if arr.ndim == 2:
        arr = arr[None]
    half = arr.shape[1] // 2
    seqs = np.concatenate([arr[:, :half], arr[:, half:2 * half]], axis=0)
    m, n, dim = seqs.shape
    out = np.empty(dim)
    for d in range(dim):
        x = seqs[:, :, d]
        c = x - x.mean(axis=1, keepdims=True)
        size = 2 ** int(np.ceil(np.log2(2 * n)))
        fx = np.fft.rfft(c, size, axis=1)
        acov = np.fft.irfft(fx * np.conj(fx), size, axis=1)[:, :n].real / n
        mean_var = float(np.mean(acov[:, 0] * n / (n - 1.0)))
        var_plus = mean_var * (n - 1.0) / n + (float(np.var(x.mean(axis=1), ddof=1)) if m > 1 else 0.0)
        rho = 1.0 - (mean_var - acov.mean(axis=0)) / var_plus
        rho[0] = 1.0
        tau, prev, k = 0.0, INF, 0
        while 2 * k + 1 < n:
            pair = rho[2 * k] + rho[2 * k + 1]
            if pair <= 0.0:
                break
            pair = min(pair, prev)
            tau += 2.0 * pair
            prev = pair
            k += 1
        tau -= 1.0
        out[d] = m * n if tau <= 0 else min(m * n / tau, m * n)
    return out
