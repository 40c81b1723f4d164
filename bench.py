#!/usr/bin/env python
"""Benchmark: iterative NUTS on B200 (BASELINE.json metric: leapfrog steps/s
and ESS/s at 1/2/4/8 GPUs vs the CPU reference).

Headline (the driver's line): configs[1] -- covtype-shaped Bayesian logistic
regression NUTS, 581,012 rows x 54 features (D = 55), 1 chain per GPU,
max_tree_depth 10, 1000 warmup + 1000 draws.  One
STEP = one complete run through the device engine (step-size search, warmup
with dual averaging and windowed mass adaptation, sampling) = ONE persistent
cooperative kernel launch; leapfrogs are counted on the device.  Under
torchrun every rank runs an independent replica (weak scaling, "replicas
only" for this config: a 126 MB pass is too small to amortise a per-leapfrog
collective).

Sub-records on the same line (each with value, roofline or issue note, a CPU
baseline timed in the same run and an end-to-end figure through run()):
  fp64_mode            config 2 in the fp64 (parity) policy
  gauss10              config 1: 10-D diagonal Gaussian, 1 chain, 1000+1000
  eight_schools_8192   config 3: 8192 chains (sharded over ranks), 1000+1000
  dense_1000x1024      config 4: 1000-D correlated Gaussian, dense mass, 1024
                       chains (sharded), tcgen05 TF32 gradient GEMMs
  rowshard_8Mx255      config 5: 8M x 255 logistic, 1 chain, rows sharded over
                       the ranks with the in-kernel NVLink exchange

CPU side ("reference" = the unmodified reference package installed in
baseline/_ref, run through its own public API on the host cores; "port" = the
oracle restatement, oracle/):
  --impl reference     the driver's reference arm: the reference's covtype
                       sampler (numpy fallback, BLAS on all host cores) on a
                       bounded sample of transitions per step
  cpu_baseline         the same, timed inside this run (rank 0, N = 1)
Workers run as subprocesses of this file (--cpu-worker) so the reference's
import-time kernel switch (TURNSTILE_DISABLE_NUMBA) and BLAS thread counts
are set per measurement.

--gpus N > 1 without WORLD_SIZE in the environment re-launches this file
under torch.distributed.run with N ranks (127.0.0.1) and fails if fewer than
N ranks or GPUs come up.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

N_ROWS, N_FEAT, DATA_SEED = 581012, 54, 20191222
ALGO_BYTES_PER_PASS = 4 * N_ROWS * N_FEAT + N_ROWS  # fp32 X + uint8 y = 126,079,604 B
C5_ROWS, C5_FEAT, C5_SEED = 8_000_000, 255, 20191223
C5_BYTES_PER_PASS = 4 * C5_ROWS * C5_FEAT + C5_ROWS  # 8,168,000,000 B
SUBS = ("gauss10", "eight_schools_8192", "dense_1000x1024", "rowshard_8Mx255", "covtype_many_chain")


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--precision", choices=("fp64", "fp32"), default="fp32",
                    help="arithmetic of the fused data pass for the headline (the other mode is reported too)")
    ap.add_argument("--single-precision", action="store_true", help="measure only --precision")
    ap.add_argument("--config", choices=("covtype", "eight_schools", "gauss10", "rowshard", "dense", "many"),
                    default="covtype",
                    help="headline workload (default: the driver's covtype line with every sub-record)")
    ap.add_argument("--subs", default=",".join(SUBS), help="comma list of sub-records for the covtype line ('' = none)")
    ap.add_argument("--chains", type=int, default=8192, help="eight_schools: total chains")
    ap.add_argument("--exec-mode", choices=("thread", "block", "warp"), default=None,
                    help="eight_schools/gauss10 team layout (default: warp for <=16 chains, else thread)")
    ap.add_argument("--num-warmup", type=int, default=1000)
    ap.add_argument("--num-samples", type=int, default=1000)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-worker", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--worker-args", default="{}", help=argparse.SUPPRESS)
    return ap.parse_args(argv)


# ============================================================================ launch helpers


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_command(argv, n):
    """The torch.distributed.run command that re-launches this file with n ranks."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + list(argv)


def maybe_spawn(args, argv):
    """--gpus N > 1 outside torchrun: spawn N ranks and return their exit code
    (None when this process is already a rank or N == 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    if args.impl != "reference":
        try:
            import torch

            have = torch.cuda.device_count()
        except Exception:
            have = 0
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible", file=sys.stderr)
            return 2
    return subprocess.call(spawn_command(argv, args.gpus))


def check_world(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} ranks came up")
    return world


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def tf32_peak():
    """Dense TF32 TFLOP/s: half the measured bf16 burst rate (the recipe's fallback 1125)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return 0.5 * float(json.load(fh)["bf16_tflops"]), "measured bf16 / 2"
    except Exception:
        return 1125.0, "fallback"


def committed_ncu(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as fh:
            return json.load(fh)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) >= 7:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None

        loaded = [s for s in self.samples if (num(s[6]) or 0) > 0] or self.samples
        sm = [num(s[0]) for s in loaded if num(s[0]) is not None]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for s in loaded:
            for k, name in enumerate(names):
                if s[2 + k].lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": num(loaded[0][1]),
                "reasons": sorted(reasons), "samples": len(loaded)}


# ============================================================================ CPU side (subprocess workers)


def reference_path():
    """Import root of the UNMODIFIED reference package: baseline/_ref (pip
    install --target, travels to the GPU box), else the read-only source tree
    when present (this container), else None."""
    for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "turnstile")):
            return p
    return None


def _import_reference():
    p = reference_path()
    if p is None:
        raise RuntimeError("reference package not installed (baseline/_ref) and /root/reference absent")
    sys.path.insert(0, p)
    import turnstile

    return turnstile


def _covtype_mode_and_mass(x, y, iters=10, sub=200_000):
    """Laplace start for the CPU samples: posterior mode (numpy Newton on the
    first `sub` rows, likelihood scaled to N) and the diagonal of the inverse
    Hessian as inverse mass (what the windowed Welford adaptation converges
    to).  Only a starting state: the timed quantity is leapfrogs per second."""
    n = min(sub, x.shape[0])
    X = np.hstack([x[:n], np.ones((n, 1))])
    yy = y[:n]
    scale = x.shape[0] / n
    th = np.zeros(X.shape[1])
    H = None
    for _ in range(iters):
        s = 1.0 / (1.0 + np.exp(-(X @ th)))
        g = th - scale * (X.T @ (yy - s))
        H = np.eye(X.shape[1]) + scale * ((X * (s * (1 - s))[:, None]).T @ X)
        th = th - np.linalg.solve(H, g)
    return th, np.diag(np.linalg.inv(H)).copy()


def w_logistic_transitions(a):
    """Reference NUTS transitions on a logistic model (its own public API:
    logistic_regression_model, find_reasonable_step_size, nuts_transition_from)
    until `seconds` of whole transitions have run."""
    ts = _import_reference()
    from turnstile import kernels
    from turnstile.adapt import find_reasonable_step_size
    from turnstile.integrator import MassMatrix, PhasePoint
    from turnstile.models import LogisticRegressionData, logistic_regression_model
    from turnstile.rng import RngKey
    from turnstile.sampler import SamplerConfig, nuts_transition_from
    from tests_data import logistic_data

    n, p, seed = a["rows"], a["features"], a["seed"]
    # (config 5's sample: 1M rows of the same generator family; per-leapfrog
    # cost does not depend on the values)
    x, y = logistic_data(n, p, seed)
    model = logistic_regression_model(LogisticRegressionData(x, y))
    kernels.warm_up()
    q, inv = _covtype_mode_and_mass(x, y)
    mass = MassMatrix(inv)
    z = PhasePoint.from_position(model, q, np.zeros(model.dim))
    key = RngKey.from_seed(a.get("key_seed", 1))
    eps = find_reasonable_step_size(z, mass, model, key.fold(1))
    cfg = SamplerConfig(step_size=eps, mass=mass)
    t0 = time.perf_counter()
    lf = trans = 0
    while time.perf_counter() - t0 < a["seconds"] or trans == 0:
        z, st = nuts_transition_from(z, cfg, model, key.fold(10 + trans))
        lf += st.leapfrog_calls
        trans += 1
    el = time.perf_counter() - t0
    return {"leapfrogs": lf, "seconds": el, "transitions": trans, "numba": bool(kernels.NUMBA_ENABLED),
            "step_size": eps, "reference": ts.__file__}


def w_run(a):
    """Reference run_chain for the chains `ids` of a RunConfig (process fan-out
    unit).  model: gaussian10 (built-in), eight_schools / dense (plugin twins
    through the reference's TargetModel API)."""
    _import_reference()
    from turnstile import chains as tch
    from turnstile import kernels
    from turnstile.models import TargetModel, gaussian_model

    kernels.warm_up()
    name = a["model"]
    if name == "gaussian10":
        model = gaussian_model(np.ones(10))
    elif name == "eight_schools":
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from turnstile_oracle import eight_schools_gradient, eight_schools_potential

        yy = [28.0, 8.0, -3.0, 7.0, -1.0, 1.0, 18.0, 12.0]
        ss = [15.0, 10.0, 16.0, 11.0, 9.0, 11.0, 10.0, 18.0]
        model = TargetModel("eight_schools", 10, lambda q: eight_schools_potential(q, yy, ss),
                            lambda q: eight_schools_gradient(q, yy, ss), {})
    elif name == "dense":
        A = dense_config4()[2]

        def pot(q):
            return 0.5 * float(q @ (A @ q))

        def grad(q):
            return A @ q

        model = TargetModel("dense_gaussian", A.shape[0], pot, grad, {})
    else:
        raise ValueError(name)
    cfg = tch.RunConfig(model={"model": name}, num_chains=a["num_chains"], num_warmup=a["num_warmup"],
                        num_samples=a["num_samples"], seed=a["seed"])
    keys = tch.chain_keys(a["seed"], a["num_chains"])
    base = tch._base_config(cfg, model)
    t0 = time.perf_counter()
    lf, done, samples = 0, 0, []
    deadline = a.get("seconds")
    for c in a["ids"]:
        r = tch.run_chain(c, keys[c], model, cfg, base)
        lf += r.total_leapfrogs
        done += 1
        if a.get("return_samples"):
            samples.append(r.samples.tolist())
        if deadline is not None and time.perf_counter() - t0 >= deadline:
            break
    return {"leapfrogs": lf, "seconds": time.perf_counter() - t0, "chains": done, "samples": samples}


def w_port_covtype(a):
    """The oracle port (fused OpenMP fp64 logistic pass + Python tree logic) on
    the same data: the builder's fastest CPU restatement, for reference."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import turnstile_oracle as o
    from tests_data import logistic_data

    x, y = logistic_data(N_ROWS, N_FEAT, DATA_SEED)
    m = o.Model("logistic_regression", N_FEAT + 1, x=x, y=y, fused_omp=True)
    q, inv = _covtype_mode_and_mass(x, y)
    U, g = m._fused(q.tolist())
    z = o.Point(q.tolist(), [0.0] * (N_FEAT + 1), U, list(g))
    step = a.get("step", 0.01)
    key = o.chain_keys(1, 1)[0]
    t0 = time.perf_counter()
    lf = i = 0
    while time.perf_counter() - t0 < a["seconds"] or i == 0:
        z, st, _ = o.transition(z, step, inv.tolist(), m, o.key_fold(key, 10 + i))
        lf += st.leapfrogs
        i += 1
    return {"leapfrogs": lf, "seconds": time.perf_counter() - t0, "transitions": i, "threads": m.threads}


WORKERS = {"logistic": w_logistic_transitions, "run": w_run, "port_covtype": w_port_covtype}


def cpu_worker_main(args):
    out = WORKERS[args.cpu_worker](json.loads(args.worker_args))
    print("CPUWORKER " + json.dumps(out), flush=True)
    return 0


def run_worker(name, wargs, threads, timeout=900):
    """One CPU worker subprocess: `threads` BLAS/OpenMP threads; numba path
    unless wargs['numpy'] (the reference's TURNSTILE_DISABLE_NUMBA switch)."""
    env = dict(os.environ)
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS"):
        env[k] = str(threads)
    env["NUMBA_CACHE_DIR"] = env.get("NUMBA_CACHE_DIR", "/tmp/numba_cache_bench")
    env["CUDA_VISIBLE_DEVICES"] = ""
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    if wargs.get("numpy"):
        env["TURNSTILE_DISABLE_NUMBA"] = "1"
    else:
        env.pop("TURNSTILE_DISABLE_NUMBA", None)
    return subprocess.Popen([sys.executable, os.path.abspath(__file__), "--cpu-worker", name, "--worker-args",
                             json.dumps(wargs)], env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)


def collect(procs, timeout=900):
    outs = []
    for p in procs:
        try:
            o, e = p.communicate(timeout=timeout)
        except subprocess.TimeoutExpired:
            p.kill()
            raise RuntimeError("CPU worker timed out")
        line = [ln for ln in o.splitlines() if ln.startswith("CPUWORKER ")]
        if p.returncode != 0 or not line:
            raise RuntimeError(f"CPU worker failed: {e.strip().splitlines()[-1] if e.strip() else p.returncode}")
        outs.append(json.loads(line[-1][len("CPUWORKER "):]))
    return outs


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_covtype(seconds, numpy_path=True):
    """The reference's covtype sampler on the host: numpy fallback with BLAS
    on all cores (its fastest path for one large chain), or numba on 1 core."""
    nc = cores() if numpy_path else 1
    w = {"rows": N_ROWS, "features": N_FEAT, "seed": DATA_SEED, "seconds": seconds, "numpy": numpy_path}
    r = collect([run_worker("logistic", w, nc)])[0]
    return {"value": r["leapfrogs"] / r["seconds"], "unit": "leapfrog/s", "cores": nc, "kind": "reference",
            "sample": (f"reference turnstile ({'numpy fallback, BLAS' if numpy_path else 'numba'}, {nc} thread(s)): "
                       f"{r['transitions']} nuts_transition_from draws from a Laplace start (mode, diag inverse "
                       f"Hessian, find_reasonable_step_size), {r['leapfrogs']} leapfrogs in {r['seconds']:.1f} s; "
                       "per-leapfrog cost is two full passes over X in every run phase"),
            "leapfrogs": r["leapfrogs"], "seconds": r["seconds"]}


def cpu_fanout(model, num_chains, seed, W, S, per_proc, procs, seconds=None):
    """Process fan-out of reference run_chain over the host cores (chains are
    independent and prefix-stable, reference tests/test_chains.py:70-72).
    Throughput = all leapfrogs / the slowest worker's time."""
    ps = []
    for k in range(procs):
        ids = list(range(k * per_proc, (k + 1) * per_proc))
        ps.append(run_worker("run", {"model": model, "num_chains": num_chains, "num_warmup": W, "num_samples": S,
                                     "seed": seed, "ids": ids, "seconds": seconds}, 1))
    outs = collect(ps)
    lf = sum(o["leapfrogs"] for o in outs)
    el = max(o["seconds"] for o in outs)
    ch = sum(o["chains"] for o in outs)
    return lf, el, ch


# ============================================================================ GPU side


def dense_config4():
    """Sigma = Q diag(logspace(-2, 2, D)) Q^T, Q from the
    QR of an N(0,1) D x D matrix (seed 4); P = Sigma^-1; dense mass M^-1 = Sigma.
    The device runs identity-mass NUTS on x = L^-1 q (M^-1 = L L^T), i.e. on
    U(x) = x'Ax/2 with A = L^T P L (models.dense_gaussian_model)."""
    D = 1000
    g = np.random.default_rng(4)
    Q, _ = np.linalg.qr(g.standard_normal((D, D)))
    lam = np.logspace(-2, 2, D)
    Sigma = (Q * lam) @ Q.T
    P = (Q / lam) @ Q.T
    L = np.linalg.cholesky(Sigma)
    return P, Sigma, L.T @ P @ L


class Ctx:
    """Rank context: device, world, reductions over ranks."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.world = check_world(args)
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.world > 1:
            dist.init_process_group("nccl", device_id=self.dev)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def red(self, v, op="max"):
        if self.world == 1:
            return v
        t = self.torch.tensor([float(v)], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return float(t.item())

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def sub_chains(ctx, args, name, model, cfg, keys, exec_mode, K, Wu, cpu):
    """Many-chain / single-small-chain configs: chains sharded over ranks, one
    launch per rank per step; device time (CUDA events) max over ranks."""
    import paper_1912_11554_b200 as ts

    torch = ctx.torch
    C = len(keys)
    # one chain: every rank runs a replica (weak scaling); many chains: sharded
    mine = list(keys) if C == 1 else [keys[c] for c in ts.chains.shard_range(C, ctx.rank, ctx.world)]
    times, lfs, last = [], [], None
    for s in range(Wu + K):
        ctx.barrier()
        r = ts.run_device(model, cfg, mine, ctx.dev, exec_mode=exec_mode, sync=False)
        r.event_ms[1].synchronize()
        if s >= Wu:
            times.append(r.event_ms[0].elapsed_time(r.event_ms[1]))
            lfs.append(float(r.stats[:, :, 1].sum().item()))
            last = r
    t_ms = ctx.red(sum(times), "max")
    lf = ctx.red(sum(lfs), "sum")
    ess, rhat = ts.chain_diagnostics_device(last.samples)
    min_ess = ctx.red(float(np.nanmin(ess)), "sum") if C > 1 else float(np.nanmin(ess))
    rec = {"value": lf / (t_ms / 1000.0), "unit": "leapfrog/s" if C == 1 else "chain-leapfrog/s",
           "ms_per_step": t_ms / K, "steps": K, "warmup": Wu, "leapfrogs_per_step": lf / K,
           "min_ess_per_step": min_ess, "ess_per_sec": min_ess / (t_ms / 1000.0 / K),
           "max_split_rhat_rank0": float(np.nanmax(rhat)), "gpu_launches": K}
    return rec, last, mine


def e2e_run(ctx, model_fn, cfg, K, h2d_bytes, exec_mode=None):
    """End to end through the public API: model from host arrays + run()
    (H2D of the data, the launch, D2H of samples/stats/adaptation), wall
    clock max over ranks."""
    import paper_1912_11554_b200 as ts

    ms, lfs, d2h = [], [], 0
    for _ in range(max(1, K)):
        ctx.barrier()
        t0 = time.perf_counter()
        model = model_fn()
        if ctx.world == 1 or cfg.num_chains == 1:  # one chain: a replica per rank
            res = ts.run(cfg, model, devices=[ctx.local], exec_mode=exec_mode)
        else:
            res = ts.chains.run_sharded(cfg, model, ctx.rank, ctx.world, device=ctx.local, exec_mode=exec_mode)
        el = time.perf_counter() - t0
        ctx.barrier()
        ms.append(ctx.red(el * 1000.0, "max"))
        lfs.append(ctx.red(float(sum(r.total_leapfrogs for r in res)), "sum"))
        d2h = sum(r.samples.nbytes + (cfg.num_warmup + cfg.num_samples) * 5 * 8 for r in res)
    return {"value": sum(lfs) / (sum(ms) / 1000.0), "unit": "leapfrog/s", "h2d_bytes_per_step": int(h2d_bytes),
            "d2h_bytes_per_step": int(d2h), "steps": max(1, K)}


def run_gauss10(ctx, args):
    import paper_1912_11554_b200 as ts

    K, Wu = min(args.steps, 5), 2
    model = ts.gaussian_model(np.ones(10))
    cfg = ts.RunConfig(model={"model": "gaussian"}, num_chains=1, num_warmup=1000, num_samples=1000, seed=7)
    keys = ts.chain_keys(7, 1)
    # one chain on every rank (replicas): a warp per chain (vectors in shared memory)
    rec, last, _ = sub_chains(ctx, args, "gauss10", model, cfg, keys, "warp", K, Wu, None)
    rec["config"] = "10-D diagonal Gaussian (cov_diag = ones), 1 chain per GPU, seed 7, 1000+1000, max_tree_depth 10"
    rec["roofline"] = {"bound": "latency", "note": "one warp runs the chain: a dependent chain of ~100 flops per "
                       "leapfrog plus tree logic; no HBM or tensor roofline applies (SURVEY 8(d) config 1)"}
    if not args.no_e2e:
        rec["e2e"] = e2e_run(ctx, lambda: ts.gaussian_model(np.ones(10)), cfg, K, 8 * 10 + 16, "warp")
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu:
        try:
            lf, el, ch = cpu_fanout("gaussian10", 1, 7, 1000, 1000, 1, 1)
            rec["cpu_baseline"] = {"value": lf / el, "unit": "leapfrog/s", "cores": 1, "kind": "reference",
                                   "sample": f"reference run_chain (numba), the same full run (seed 7, 1000+1000): "
                                             f"{lf} leapfrogs in {el:.2f} s", "same_config": True}
        except Exception as e:  # the GPU record stands without its CPU baseline
            rec["cpu_baseline"] = {"value": None, "error": f"{type(e).__name__}: {e}"[:300]}
    return rec


def run_eight(ctx, args):
    import paper_1912_11554_b200 as ts

    K, Wu, C = min(args.steps, 3), 1, 8192
    model = ts.eight_schools_model()
    cfg = ts.RunConfig(model={"model": "eight_schools"}, num_chains=C, num_warmup=1000, num_samples=1000, seed=3)
    rec, last, mine = sub_chains(ctx, args, "eight", model, cfg, ts.chain_keys(3, C), "thread", K, Wu, None)
    rec["config"] = f"eight schools NC, {C} chains sharded over {ctx.world} GPU(s), seed 3, 1000+1000, one chain per thread"
    rec["roofline"] = {"bound": "issue", "note": "state in registers/L1 (one chain per thread); no HBM or tensor "
                       "roofline applies (SURVEY 8(d) config 3): ~300 flops per chain-leapfrog"}
    if not args.no_e2e:
        rec["e2e"] = e2e_run(ctx, ts.eight_schools_model, cfg, 1, 16 * C + 8 * 10 + 64, "thread")
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu:
        try:
            nc = cores()
            per = 2
            lf, el, ch = cpu_fanout("eight_schools", C, 3, 1000, 1000, per, nc)
            v = lf / el
            rec["cpu_baseline"] = {"value": v, "unit": "chain-leapfrog/s", "cores": nc, "kind": "reference",
                                   "sample": f"reference run_chain with the eight-schools TargetModel plugin twin, process "
                                             f"fan-out: chains 0..{ch - 1} of chain_keys(3, 8192) on {nc} processes, {lf} "
                                             f"leapfrogs in {el:.1f} s; full 8192-chain run extrapolated "
                                             f"{el * C / ch / 3600:.2f} h"}
        except Exception as e:  # the GPU record stands without its CPU baseline
            rec["cpu_baseline"] = {"value": None, "error": f"{type(e).__name__}: {e}"[:300]}
    return rec


def run_dense(ctx, args, W=1000, S=1000):
    import paper_1912_11554_b200 as ts

    K, Wu, C, D = 1, 1, 1024, 1000
    P, Sigma, A = dense_config4()
    model = ts.dense_gaussian_model(P, inv_mass=Sigma, precision="tf32")
    cfg = ts.RunConfig(model={"model": "dense_gaussian"}, num_chains=C, num_warmup=W, num_samples=S, seed=4)
    keys = ts.chain_keys(4, C)
    mine = [keys[c] for c in ts.chains.shard_range(C, ctx.rank, ctx.world)]
    times, lfs, steps = [], [], []
    for s in range(Wu + K):
        ctx.barrier()
        r = ts.run_device(model, cfg, mine, ctx.dev, sync=False)
        r.event_ms[1].synchronize()
        if s >= Wu:
            times.append(r.event_ms[0].elapsed_time(r.event_ms[1]))
            lfs.append(float(r.stats[:, :, 1].sum().item()))
            steps.append(float(r.evals.max().item()))
            last = r
    t_ms = ctx.red(sum(times), "max")
    lf = ctx.red(sum(lfs), "sum")
    Cr = len(mine)
    flops = 2.0 * D * D * (-(-Cr // 64) * 64) * sum(steps)
    tflops = flops / (sum(times) / 1e3) / 1e12
    peak, pk = tf32_peak()
    ess, rhat = ts.chain_diagnostics_device(last.samples)
    ncu = committed_ncu("r2_ncu_dense.json") or {}
    rec = {"value": lf / (t_ms / 1000.0), "unit": "chain-leapfrog/s", "ms_per_step": t_ms / K, "steps": K,
           "warmup": Wu, "dtype": "tf32",
           "config": f"1000-D correlated Gaussian (SURVEY 8(d) cfg 4), dense mass M^-1 = Sigma, {C} chains sharded over "
                     f"{ctx.world} GPU(s), seed 4, {W}+{S}, batched tcgen05 TF32 gradient GEMMs",
           "leapfrogs_per_step": lf / K, "lockstep_steps_per_run": sum(steps) / K,
           "us_per_gemm_step": 1e3 * sum(times) / max(1.0, sum(steps)),
           "min_ess_per_step": float(np.nanmin(ess)), "ess_per_sec": float(np.nanmin(ess)) / (t_ms / 1000.0 / K),
           "max_split_rhat_rank0": float(np.nanmax(rhat)), "gpu_launches": K,
           "roofline": {"bound": "tensor", "achieved": tflops, "peak": peak, "unit": "TFLOP/s", "frac": tflops / peak,
                        "peak_kind": pk, "tensor_pipe_pct": ncu.get("tensor_pipe_pct"),
                        "dram_bytes_per_chain_leapfrog": ncu.get("dram_bytes_per_chain_leapfrog"),
                        "note": "GEMM flops (2 D^2 per chain per step) over the whole run's device time; the chains' "
                                "fp64 vector bookkeeping is the rest of the step"}}
    if not args.no_e2e:
        rec["e2e"] = e2e_run(ctx, lambda: ts.dense_gaussian_model(P, inv_mass=Sigma, precision="tf32"), cfg, 1,
                             P.nbytes + Sigma.nbytes + 16 * C)
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu:
        try:
            nc = cores()
            lf_c, el, ch = cpu_fanout("dense", C, 4, W, S, 1, nc, seconds=args.cpu_seconds)
            rec["cpu_baseline"] = {"value": lf_c / el, "unit": "chain-leapfrog/s", "cores": nc, "kind": "reference",
                                   "sample": f"reference run_chain with a numpy dense TargetModel (U = x'Ax/2, A = L'PL, "
                                             f"the device's model), process fan-out on {nc} processes (1 BLAS thread "
                                             f"each), bounded at {args.cpu_seconds:.0f} s: {lf_c} leapfrogs in {el:.1f} s "
                                             f"({ch} chains completed)"}
        except Exception as e:  # the GPU record stands without its CPU baseline
            rec["cpu_baseline"] = {"value": None, "error": f"{type(e).__name__}: {e}"[:300]}
    return rec


def run_rowshard(ctx, args, W=20, S=20):
    import paper_1912_11554_b200 as ts
    from tests_data import logistic_data_f32

    K, Wu = 1, 1
    a, b = ts.rowshard.row_range(C5_ROWS, ctx.rank, ctx.world)
    t0 = time.perf_counter()
    x, y = logistic_data_f32(C5_ROWS, C5_FEAT, C5_SEED, rows=(a, b))
    gen_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    model = ts.logistic_regression_model(ts.LogisticRegressionData(x, y), precision="fp32")
    model.device_spec.handle(ctx.dev)
    upload_s = time.perf_counter() - t0
    if ctx.world > 1:
        ts.rowshard.connect(model.device_spec, ctx.rank, ctx.world, ts.rowshard.torch_all_gather(), device=ctx.dev)
    peak, pk = peaks()
    times, lfs, evs = [], [], []
    for s in range(Wu + K):
        cfg = ts.RunConfig(model={"model": "logistic_regression"}, num_chains=1, num_warmup=W, num_samples=S,
                           seed=args.seed + s)
        ctx.barrier()
        r = ts.run_device(model, cfg, ts.chain_keys(args.seed + s, 1), ctx.dev, sync=False)
        r.event_ms[1].synchronize()
        if s >= Wu:
            times.append(r.event_ms[0].elapsed_time(r.event_ms[1]))
            lfs.append(float(r.stats[0, :, 1].sum().item()))
            evs.append(float(r.evals[0].item()))
            st = r.status.cpu().numpy()
            if (st != 0).any():
                raise RuntimeError(f"row-shard run status {st.tolist()}")
    t_ms = ctx.red(sum(times), "max")
    lf, ev = sum(lfs), sum(evs)  # one replicated chain: counted once
    achieved = C5_BYTES_PER_PASS * ev / (t_ms / 1000.0) / 1e9
    ncu = committed_ncu("r1_ncu_wide_8Mx255_fp32.json")
    rec = {"value": lf / (t_ms / 1000.0), "unit": "leapfrog/s", "ms_per_step": t_ms / K, "steps": K, "warmup": Wu,
           "dtype": "f32", "scaling": "strong",
           "config": f"logistic NUTS 8,000,000 x 255 (D=256), 1 chain, rows sharded over {ctx.world} GPU(s) "
                     f"(in-kernel NVLink exchange of the fixed-point totals per pass), max_tree_depth 10, "
                     f"{W}+{S} draws per step (a full 1000+1000 run is ~4 min per step at this size)",
           "leapfrogs_per_step": lf / K, "passes_per_step": ev / K,
           "data_gen_s_rank0": gen_s, "model_upload_retile_s_rank0": upload_s,
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * ctx.world, "unit": "GB/s",
                        "frac": achieved / (peak * ctx.world), "peak_kind": pk, "bytes_per_pass": C5_BYTES_PER_PASS,
                        "traffic": (ncu[0].get("dram_bytes_per_pass") if ncu else None)},
           "gpu_launches": K}
    if not args.no_e2e and ctx.world == 1:
        xh = ctx.torch.from_numpy(x).pin_memory().numpy()
        cfg = ts.RunConfig(model={"model": "logistic_regression"}, num_chains=1, num_warmup=W, num_samples=S,
                           seed=args.seed + Wu)
        rec["e2e"] = e2e_run(ctx, lambda: ts.logistic_regression_model(ts.LogisticRegressionData(xh, y),
                                                                        precision="fp32"), cfg, 1, x.nbytes + y.nbytes)
    del x, y
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu:
        try:
            rows = 1_000_000
            nc = cores()
            w = {"rows": rows, "features": C5_FEAT, "seed": C5_SEED, "seconds": args.cpu_seconds, "numpy": True}
            r = collect([run_worker("logistic", w, nc)])[0]
            per_lf_full = r["seconds"] / r["leapfrogs"] * (C5_ROWS / rows)
            rec["cpu_baseline"] = {"value": 1.0 / per_lf_full, "unit": "leapfrog/s", "cores": nc, "kind": "reference",
                                   "sample": f"reference turnstile numpy fallback (BLAS, {nc} threads) on {rows:,} x 255 "
                                             f"rows of the same generator: {r['leapfrogs']} leapfrogs in "
                                             f"{r['seconds']:.1f} s, time per leapfrog scaled x{C5_ROWS // rows} "
                                             "(linear in rows)"}
        except Exception as e:  # the GPU record stands without its CPU baseline
            rec["cpu_baseline"] = {"value": None, "error": f"{type(e).__name__}: {e}"[:300]}
    return rec


def run_many(ctx, args, C=256, W=100, S=100):
    """Covtype with C chains sharing X on the tensor cores (precision "tf32",
    csrc/ts_k_logistic_many.cu): one X stream per batched step serves every
    chain with an outstanding gradient request.  Chains sharded over ranks."""
    import paper_1912_11554_b200 as ts
    from tests_data import logistic_data

    K, Wu = 1, 1
    x, y = logistic_data(N_ROWS, N_FEAT, DATA_SEED)
    model = ts.logistic_regression_model(ts.LogisticRegressionData(x, y), precision="tf32")
    cfg = ts.RunConfig(model={"model": "logistic_regression"}, num_chains=C, num_warmup=W, num_samples=S, seed=5)
    keys = ts.chain_keys(5, C)
    mine = [keys[c] for c in ts.chains.shard_range(C, ctx.rank, ctx.world)]
    times, lfs, evs = [], [], []
    for s in range(Wu + K):
        ctx.barrier()
        r = ts.run_device(model, cfg, mine, ctx.dev, sync=False)
        r.event_ms[1].synchronize()
        if s >= Wu:
            times.append(r.event_ms[0].elapsed_time(r.event_ms[1]))
            lfs.append(float(r.stats[:, :, 1].sum().item()))
            evs.append(float(r.evals.sum().item()))
            last = r
    t_ms = ctx.red(sum(times), "max")
    lf = ctx.red(sum(lfs), "sum")
    ev = ctx.red(sum(evs), "sum")
    ess, rhat = ts.chain_diagnostics_device(last.samples)
    # tensor work per chain-evaluation over the N rows: GEMM 1 3 x 2 x 56 (3xTF32), GEMM 2 4 x 2 x 64 (3xBF16 stacked)
    flops_per_eval = (3 * 2 * 56 + 4 * 2 * 64) * N_ROWS
    tf = flops_per_eval * ev / (t_ms / 1000.0) / 1e12
    peak, pk = tf32_peak()
    ncu = committed_ncu("r2_ncu_many.json") or {}
    rec = {"value": lf / (t_ms / 1000.0), "unit": "chain-leapfrog/s", "ms_per_step": t_ms / K, "steps": K, "warmup": Wu,
           "dtype": "tf32x3/bf16x3",
           "config": f"covtype 581012x54 logistic, {C} chains sharded over {ctx.world} GPU(s) sharing X (precision tf32), "
                     f"seed 5, {W}+{S}, max_tree_depth 10",
           "leapfrogs_per_step": lf / K, "evals_per_step": ev / K,
           "min_ess_per_step": float(np.nanmin(ess)), "ess_per_sec": float(np.nanmin(ess)) / (t_ms / 1000.0 / K),
           "max_split_rhat_rank0": float(np.nanmax(rhat)), "gpu_launches": K,
           "roofline": {"bound": "issue (epilogue)", "achieved": tf, "peak": peak, "unit": "TFLOP/s",
                        "frac": tf / peak, "peak_kind": pk, "tensor_pipe_pct": ncu.get("tensor_pipe_pct"),
                        "note": "tensor flops of both GEMMs per chain-evaluation; the per-(row, chain) CUDA-core "
                                "epilogue (sigmoid, log-likelihood, bf16 split of the residuals) bounds the step"}}
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu:
        try:
            nc = min(cores(), 32)  # each process holds covtype X (251 MB) and its numba code: bounded host memory
            ps = [run_worker("logistic", {"rows": N_ROWS, "features": N_FEAT, "seed": DATA_SEED, "seconds": args.cpu_seconds,
                                          "numpy": False, "key_seed": 100 + k}, 1) for k in range(nc)]
            outs = collect(ps)
            lf_c = sum(o["leapfrogs"] for o in outs)
            el = max(o["seconds"] for o in outs)
            rec["cpu_baseline"] = {"value": lf_c / el, "unit": "chain-leapfrog/s", "cores": nc, "kind": "reference",
                                   "sample": f"reference turnstile (numba, 1 thread per process) nuts_transition_from on "
                                             f"covtype, one chain per process on {nc} processes: {lf_c} leapfrogs in "
                                             f"{el:.1f} s"}
        except Exception as e:  # the GPU record stands without its CPU baseline
            rec["cpu_baseline"] = {"value": None, "error": f"{type(e).__name__}: {e}"[:300]}
    return rec


def timed_covtype(ctx, args, x32, y8, precision, K, Wu, with_clocks, flush):
    """Wu untimed + K timed full runs; device time per launch (CUDA events)."""
    import paper_1912_11554_b200 as ts

    torch = ctx.torch
    model = ts.logistic_regression_model(ts.LogisticRegressionData(x32, y8), precision=precision)
    model.device_spec.handle(ctx.dev)
    ms_list, lf_list, ev_list, ess_list, seeds = [], [], [], [], []
    last = None
    clocks = ClockSampler(ctx.local)
    cfg_for = lambda seed: ts.RunConfig(model={"model": "logistic_regression"}, num_chains=1,  # noqa: E731
                                        num_warmup=args.num_warmup, num_samples=args.num_samples, seed=seed)
    for s in range(Wu + K):
        seed = args.seed + 1000 * s + ctx.rank
        flush.fill_(float(s))
        ctx.barrier()
        if s == Wu and with_clocks:
            clocks.__enter__()
        r = ts.run_device(model, cfg_for(seed), ts.chain_keys(seed, 1), ctx.dev, sync=False)
        r.event_ms[1].synchronize()
        ctx.barrier()
        if s >= Wu:
            ms_list.append(r.event_ms[0].elapsed_time(r.event_ms[1]))
            lf_list.append(float(r.stats[0, :, 1].sum().item()))
            ev_list.append(float(r.evals[0].item()))
            ess_list.append(float(np.nanmin(ts.ess(r.samples.cpu().numpy()))))
            seeds.append(seed)
            last = r
    if with_clocks:
        clocks.__exit__(None, None, None)
    t_total_ms = ctx.red(sum(ms_list), "max")
    lf_total = ctx.red(sum(lf_list), "sum")
    ess_total = ctx.red(sum(ess_list), "sum")
    bpp = ALGO_BYTES_PER_PASS if precision != "fp64x" else 8 * N_ROWS * N_FEAT + N_ROWS  # X stored in fp64
    achieved = bpp * sum(ev_list) / (sum(ms_list) / 1000.0) / 1e9
    # the fused pass alone: 200 passes in one launch, timed inside the kernel
    q = last.samples[0, -1].contiguous()
    out = torch.zeros(12, dtype=torch.float64, device=ctx.dev)
    lib = ts._lib.load_library()
    h = model.device_spec.handle(ctx.dev)
    ts._lib.check(lib.ts_eval_bench(h, q.data_ptr(), 20, out.data_ptr(), ts._lib.stream_ptr(torch)))
    flush.fill_(1.0)
    ts._lib.check(lib.ts_eval_bench(h, q.data_ptr(), 200, out.data_ptr(), ts._lib.stream_ptr(torch)))
    torch.cuda.synchronize()
    eval_us = float(out.cpu().numpy()[1]) / 1000.0 / 200
    peak, peak_kind = peaks()
    eval_gbs = bpp / (eval_us * 1e-6) / 1e9
    ncu = committed_ncu(f"r2_ncu_run_{precision}.json") or committed_ncu(f"r1_ncu_run_{precision}.json")
    traffic = ncu[0].get("dram_bytes_per_pass") if ncu else None
    return {
        "value": lf_total / (t_total_ms / 1000.0),
        "ms_per_step": t_total_ms / K,
        "ess_per_sec": ess_total / (t_total_ms / 1000.0),
        "leapfrogs_per_step": lf_total / K,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_per": "data pass (ncu capture in profiles/)",
                     "dram_gbs_from_traffic": (traffic * sum(ev_list) / (sum(ms_list) / 1000.0) / 1e9
                                               if traffic else None),
                     "peak_kind": peak_kind, "bytes_per_pass": bpp, "passes": sum(ev_list)},
        "eval_only": {"us_per_pass": eval_us, "achieved_gbs": eval_gbs, "frac": eval_gbs / peak},
        "clocks": clocks.summary() if with_clocks else None,
        "seeds": seeds, "last": last, "steps": K, "warmup": Wu,
    }


def run_covtype(args):
    import paper_1912_11554_b200 as ts
    from tests_data import logistic_data

    ctx = Ctx(args)
    torch = ctx.torch
    x, y = logistic_data(N_ROWS, N_FEAT, DATA_SEED)
    x32, y8 = np.ascontiguousarray(x, dtype=np.float32), np.ascontiguousarray(y, dtype=np.uint8)
    del x, y
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=ctx.dev)  # 256 MB > L2
    main_m = timed_covtype(ctx, args, x32, y8, args.precision, args.steps, args.warmup, True, flush)
    other = "fp64" if args.precision == "fp32" else "fp32"
    other_m = None if args.single_precision else timed_covtype(ctx, args, x32, y8, other, min(args.steps, 5), 1,
                                                               False, flush)
    # the fp64 policy with X stored in fp64 (2x the bytes, no conversions): the
    # layout for data that are not fp32-exact
    x64_m = None if args.single_precision else timed_covtype(ctx, args, x32, y8, "fp64x", min(args.steps, 3), 1,
                                                             False, flush)
    last = main_m["last"]

    # ---------------------------------------------------------------- end to end through the public API
    # the same seeds as the timed leg: identical device work plus H2D / re-tiling / D2H
    e2e = None
    if not args.no_e2e:
        xp = torch.from_numpy(x32).pin_memory()
        yp = torch.from_numpy(y8).pin_memory()
        e_ms, e_lf = [], []
        h2d = x32.nbytes + y8.nbytes
        d2h = 0
        for seed in main_m["seeds"][: min(args.steps, 5)]:
            cfg = ts.RunConfig(model={"model": "logistic_regression"}, num_chains=1, num_warmup=args.num_warmup,
                               num_samples=args.num_samples, seed=seed)
            flush.fill_(2.0)
            ctx.barrier()
            t0 = time.perf_counter()
            m2 = ts.logistic_regression_model(ts.LogisticRegressionData(xp.numpy(), yp.numpy()),
                                              precision=args.precision)
            res = ts.run(cfg, m2, devices=[ctx.local])
            el = time.perf_counter() - t0
            ctx.barrier()
            e_ms.append(ctx.red(el * 1000.0, "max"))
            e_lf.append(ctx.red(float(res[0].total_leapfrogs), "sum"))
            d2h = (res[0].samples.nbytes + (args.num_warmup + args.num_samples) * 5 * 8
                   + (2 + args.num_warmup + N_FEAT + 1) * 8)
            del m2, res
        e2e = {"value": sum(e_lf) / (sum(e_ms) / 1000.0), "unit": "leapfrog/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "steps": len(e_ms), "seeds": "the timed leg's first seeds"}

    cpu = None
    if ctx.rank == 0 and ctx.world == 1 and not args.no_cpu:
        try:
            cpu = cpu_covtype(args.cpu_seconds, numpy_path=True)
            lf_per_ess = main_m["leapfrogs_per_step"] / (main_m["ess_per_sec"] * main_m["ms_per_step"] / 1000.0)
            cpu["ess_per_sec_est"] = cpu["value"] / lf_per_ess
            cpu["ess_note"] = "estimated: CPU leapfrog/s x (device min-ESS per leapfrog), SURVEY 8(d)"
            port = collect([run_worker("port_covtype", {"seconds": min(args.cpu_seconds, 10.0),
                                                        "step": float(last.adapt[0, 1].item())}, cores())])[0]
            cpu["port_omp"] = {"value": port["leapfrogs"] / port["seconds"], "cores": port["threads"], "kind": "port",
                               "sample": f"oracle port (fused OpenMP fp64 pass + Python tree logic): "
                                         f"{port['leapfrogs']} leapfrogs in {port['seconds']:.1f} s"}
        except Exception as e:  # the CPU leg never sinks the GPU line
            cpu = {"value": None, "error": str(e)}

    subs = {}
    wanted = [s for s in args.subs.split(",") if s]
    for name, fn in (("gauss10", run_gauss10), ("eight_schools_8192", run_eight), ("dense_1000x1024", run_dense),
                     ("rowshard_8Mx255", run_rowshard), ("covtype_many_chain", run_many)):
        if name not in wanted:
            continue
        t0 = time.perf_counter()
        ok = 1.0
        try:
            rec = fn(ctx, args)
        except Exception as e:
            rec = {"error": f"{type(e).__name__}: {e}"}
            ok = 0.0
        torch.cuda.synchronize()
        if ctx.red(1.0 - ok, "max") > 0 and "error" not in rec:
            rec = {"error": "failed on another rank"}
        rec["wall_s_rank0"] = time.perf_counter() - t0
        subs[name] = rec

    if ctx.rank == 0:
        line = {
            "metric": "leapfrog_steps_per_sec",
            "value": main_m["value"],
            "unit": "leapfrog/s",
            "n_gpus": ctx.world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": main_m["ms_per_step"],
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "f64" if args.precision == "fp64" else "f32",
            "data": "synthetic",
            "config": {
                "workload": "covtype-shaped logistic NUTS, 581012x54 (D=55), 1 chain per GPU, max_tree_depth 10",
                "num_warmup": args.num_warmup, "num_samples": args.num_samples, "precision": args.precision,
                "parallelism": f"replicas{ctx.world}", "l2": "256 MB buffer written between steps (X+y = 126 MB ~ L2)",
                "step": "one full run (step-size search + warmup + sampling) = one persistent kernel launch",
            },
            "ess_per_sec": main_m["ess_per_sec"],
            "leapfrogs_per_step": main_m["leapfrogs_per_step"],
            "roofline": main_m["roofline"],
            "eval_only": main_m["eval_only"],
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps,
            "clocks": main_m["clocks"],
        }
        if other_m is not None:
            line[f"{other}_mode"] = {k: other_m[k] for k in ("value", "ms_per_step", "ess_per_sec", "leapfrogs_per_step",
                                                            "roofline", "eval_only", "steps", "warmup")}
        if x64_m is not None:
            line["fp64x_mode"] = {k: x64_m[k] for k in ("value", "ms_per_step", "ess_per_sec", "leapfrogs_per_step",
                                                       "roofline", "eval_only", "steps", "warmup")}
        line.update(subs)
        print(json.dumps(line), flush=True)
    ctx.close()
    return 0


# ============================================================================ single-config lines


def run_single(args):
    """--config gauss10 / eight_schools / dense / rowshard: that configuration's
    own line (not the driver's headline)."""
    ctx = Ctx(args)
    fn = {"gauss10": run_gauss10, "eight_schools": run_eight, "dense": run_dense, "rowshard": run_rowshard,
          "many": run_many}[args.config]
    if args.config == "many":
        rec = run_many(ctx, args, args.chains if args.chains != 8192 else 256, args.num_warmup, args.num_samples)
    elif args.config == "dense":
        rec = run_dense(ctx, args, args.num_warmup, args.num_samples)
    elif args.config == "rowshard":
        rec = run_rowshard(ctx, args, min(args.num_warmup, 1000), min(args.num_samples, 1000))
    else:
        rec = fn(ctx, args)
    if ctx.rank == 0:
        line = {"metric": "leapfrog_steps_per_sec", "n_gpus": ctx.world, "higher_is_better": True,
                "scaling": rec.pop("scaling", "weak" if args.config == "gauss10" else "strong"), "vs_baseline": None,
                "dtype": rec.pop("dtype", "f64"), "data": "synthetic"}
        line.update(rec)
        print(json.dumps(line), flush=True)
    ctx.close()
    return 0


# ============================================================================ reference arm


def run_reference(args):
    """--impl reference: the unmodified reference package (baseline/_ref)
    through its own public API on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    if reference_path() is None:
        print(json.dumps({"impl": "reference", "unavailable": "reference package not installed in baseline/_ref"}))
        return 0
    per_step = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    nc = cores()
    # one long-lived worker: data, numba warm-up and the Laplace start once; then
    # one bounded sample per step
    times, lfs = [], []
    w = {"rows": N_ROWS, "features": N_FEAT, "seed": DATA_SEED, "numpy": True,
         "seconds": per_step * (args.steps + args.warmup), "steps": args.steps + args.warmup}
    r = collect([run_worker("logistic", w, nc)], timeout=1800)[0]
    value = r["leapfrogs"] / r["seconds"]
    line = {
        "impl": "reference",
        "metric": "leapfrog_steps_per_sec",
        "value": value,
        "unit": "leapfrog/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 * per_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "covtype-shaped logistic NUTS, 581012x54 (D=55), 1 chain, max_tree_depth 10",
                   "rows": N_ROWS, "features": N_FEAT},
        "cpu_baseline": {"value": value, "unit": "leapfrog/s", "cores": nc, "kind": "reference",
                         "sample": f"reference turnstile (numpy fallback, BLAS {nc} threads) nuts_transition_from "
                                   f"draws from a Laplace start: {r['transitions']} transitions, {r['leapfrogs']} "
                                   f"leapfrogs in {r['seconds']:.1f} s (~{per_step:.0f} s per step x "
                                   f"{args.steps + args.warmup}); a full 1000+1000 run (~1.1e5 leapfrogs) would take "
                                   f"{1.1e5 / value / 3600:.1f} h"},
        "e2e": {"value": value, "unit": "leapfrog/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    try:
        nb = collect([run_worker("logistic", {"rows": N_ROWS, "features": N_FEAT, "seed": DATA_SEED, "numpy": False,
                                              "seconds": 10.0}, 1)])[0]
        line["numba_1core"] = {"value": nb["leapfrogs"] / nb["seconds"], "cores": 1, "kind": "reference",
                               "sample": f"reference default numba path: {nb['leapfrogs']} leapfrogs in "
                                         f"{nb['seconds']:.1f} s"}
    except Exception as e:
        line["numba_1core"] = {"error": str(e)}
    print(json.dumps(line), flush=True)
    return 0


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    if args.cpu_worker:
        return cpu_worker_main(args)
    rc = maybe_spawn(args, argv)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    if args.config != "covtype":
        return run_single(args)
    return run_covtype(args)


if __name__ == "__main__":
    sys.exit(main())
