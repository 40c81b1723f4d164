#!/usr/bin/env python
"""Benchmark: covtype-shaped Bayesian logistic regression NUTS on B200.

BASELINE.json metric: leapfrog steps/s (and ESS/s) of NUTS on synthetic
covtype-shaped logistic regression (581,012 rows x 54 features, D = 55),
1 chain per GPU, max_tree_depth 10 (configs[1]).

One benchmark STEP = one complete run of that configuration through the
device engine: step-size search, 1000 warmup draws with dual averaging and
windowed mass adaptation, 1000 sampling draws.  All of it is ONE persistent
cooperative kernel launch (ts_run_chains); the step's leapfrogs are counted
on the device.  Multi-GPU (torchrun, one rank per GPU) runs independent
replicas with different seeds (weak scaling, "replicas only": a 126 MB data
pass is too small to amortise a per-leapfrog collective).

Keys of the JSON line beyond the driver contract:
  roofline     achieved GB/s of the persistent kernel = algorithmic bytes per
               data pass (4*N*p + N) x passes / kernel time (CUDA events on
               the launching stream); peak = MEASURED_PEAKS.json hbm_gbs
  eval_only    the fused potential+gradient pass alone (ts_eval_bench)
  cpu_baseline the oracle port (oracle/, fused OpenMP pass + Python tree
               logic) on the host cores for a bounded sample
  e2e          the public API (logistic_regression_model + run) from host
               numpy data: H2D of X and y, re-tiling, run, D2H of results
"""

from __future__ import annotations

import argparse
import json
import math
import os
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--precision", choices=("fp64", "fp32"), default="fp32",
                    help="arithmetic of the fused data pass for the headline (the other mode is reported too)")
    ap.add_argument("--single-precision", action="store_true", help="measure only --precision")
    ap.add_argument("--config", choices=("covtype", "eight_schools", "gauss10", "rowshard", "dense"), default="covtype")
    ap.add_argument("--chains", type=int, default=8192, help="eight_schools: total chains")
    ap.add_argument("--exec-mode", choices=("thread", "block", "warp"), default=None,
                    help="eight_schools/gauss10 team layout (default: warp for <=16 chains, else thread)")
    ap.add_argument("--num-warmup", type=int, default=1000)
    ap.add_argument("--num-samples", type=int, default=1000)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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


def make_data():
    from tests_data import logistic_data

    x, y = logistic_data(N_ROWS, N_FEAT, DATA_SEED)
    return np.ascontiguousarray(x, dtype=np.float32), np.ascontiguousarray(y, dtype=np.uint8)


def cpu_baseline(x32, y8, seconds, start=None, step=None, inv=None, seed=1):
    """Oracle port on the host cores: NUTS transitions of the same model
    (fused OpenMP logistic pass + Python tree logic), bounded by `seconds`."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import turnstile_oracle as o

    m = o.Model("logistic_regression", N_FEAT + 1, x=x32.astype(np.float64), y=y8.astype(np.float64), fused_omp=True)
    m._x32, m._y8 = x32, y8
    key = o.chain_keys(seed, 1)[0]
    if start is None:
        # bounded sample of the run itself: q0 ~ U(-2,2), step-size search, warmup draws
        t0 = time.perf_counter()
        lf = 0
        out = None
        budget = 64
        while time.perf_counter() - t0 < seconds:
            out = o.run_chain(m, key, 1000, 1, max_leapfrogs=budget)
            lf += out["total_leapfrogs"]
            budget *= 2
        el = time.perf_counter() - t0
        return lf, el, m.threads, "oracle run_chain warmup draws from q0 (leapfrog budget doubling)"
    z = o.Point(list(start), [0.0] * (N_FEAT + 1), m.potential(list(start)), m.gradient(list(start)))
    t0 = time.perf_counter()
    lf = 0
    i = 0
    while time.perf_counter() - t0 < seconds:
        z, st, _ = o.transition(z, step, inv, m, o.key_fold(key, 10 + i))
        lf += st.leapfrogs
        i += 1
    el = time.perf_counter() - t0
    return lf, el, m.threads, f"{i} oracle NUTS transitions from the device's adapted state"


def run_reference(args):
    """--impl reference: the CPU implementation of the path (oracle port), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    x32, y8 = make_data()
    times, lfs = [], []
    threads = 1
    per_step = max(1.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    for s in range(args.warmup + args.steps):
        lf, el, threads, sample = cpu_baseline(x32, y8, per_step, seed=args.seed + s)
        if s >= args.warmup:
            times.append(el)
            lfs.append(lf)
    value = sum(lfs) / sum(times)
    line = {
        "impl": "reference",
        "metric": "leapfrog_steps_per_sec",
        "value": value,
        "unit": "leapfrog/s",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1000.0 * sum(times) / len(times),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "covtype-shaped logistic NUTS, 581012x54 (D=55), 1 chain, max_tree_depth 10",
                   "rows": N_ROWS, "features": N_FEAT},
        "cpu_baseline": {"value": value, "unit": "leapfrog/s", "cores": threads, "kind": "port",
                         "sample": f"{per_step:.0f} s per step: {sample}"},
        "e2e": {"value": value, "unit": "leapfrog/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_eight_schools(args):
    """Secondary workload: 8192 eight-schools chains,
    1000+1000, sharded across ranks (one chain per thread, one launch per GPU).
    Not the driver's headline line; run with --config eight_schools."""
    import torch
    import torch.distributed as dist

    import paper_1912_11554_b200 as ts

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.config == "gauss10":  # 10-D diagonal Gaussian, 1 chain
        C = 1
        model = ts.gaussian_model(np.ones(10))
        cfg = ts.RunConfig(model={"model": "gaussian"}, num_chains=1, num_warmup=args.num_warmup,
                           num_samples=args.num_samples, seed=7)
        keys = ts.chain_keys(7, 1)
    else:
        C = args.chains
        model = ts.eight_schools_model()
        cfg = ts.RunConfig(model={"model": "eight_schools"}, num_chains=C, num_warmup=args.num_warmup,
                           num_samples=args.num_samples, seed=3)
        keys = ts.chain_keys(3, C)
    mine = [keys[c] for c in ts.chains.shard_range(C, rank, world)]
    # one chain: a warp per chain (vectors in shared memory) is ~2x faster than
    # the one-thread-per-chain layout built for thousands of chains
    mode = args.exec_mode or ("warp" if len(mine) <= 16 else "thread")
    times, lfs = [], []
    last = None
    for s in range(args.warmup + args.steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        r = ts.run_device(model, cfg, mine, dev, exec_mode=mode)
        if s >= args.warmup:
            times.append(r.event_ms)
            lfs.append(float(r.stats.cpu().numpy()[:, :, 1].sum()))
            last = r
    t = torch.tensor([sum(times), sum(lfs)], dtype=torch.float64, device=dev)
    if world > 1:
        tm = t[:1].clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        tl = t[1:].clone()
        dist.all_reduce(tl, op=dist.ReduceOp.SUM)
        t = torch.cat([tm, tl])
    t_ms, lf = float(t[0]), float(t[1])
    ess = ts.ess_device(last.samples)  # on the GPU: no host copy of the 8192-chain samples
    if rank == 0:
        print(json.dumps({
            "metric": "leapfrog_steps_per_sec", "value": lf / (t_ms / 1000.0), "unit": "leapfrog/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "dtype": "f64", "data": "synthetic",
            "config": {"workload": (f"eight schools NC, {C} chains" if args.config == "eight_schools"
                                    else "10-D diagonal Gaussian, 1 chain")
                                   + f" x ({args.num_warmup}+{args.num_samples}), "
                                   + {"block": "one CTA per chain", "warp": "one warp per chain",
                                      "thread": "one chain per thread"}[mode]},
            "min_ess_rank0_shard": float(np.nanmin(ess)),
            "ess_per_sec_rank0_shard": float(np.nanmin(ess)) / (t_ms / 1000.0 / args.steps),
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


C5_ROWS, C5_FEAT, C5_SEED = 8_000_000, 255, 20191223
C5_BYTES_PER_PASS = 4 * C5_ROWS * C5_FEAT + C5_ROWS  # 8,168,000,000 B


def run_row_sharded(args):
    """ONE logistic chain over 8M x 255 rows, rows
    sharded over the ranks (world 1 = one GPU holds all rows).  Each data
    pass ends with the in-kernel NVLink peer exchange of the fixed-point
    totals (paper_1912_11554_b200/rowshard.py); every rank runs the same
    chain.  Not the driver's headline line; run with --config rowshard."""
    import torch
    import torch.distributed as dist

    import paper_1912_11554_b200 as ts
    from tests_data import logistic_data_f32

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    a, b = ts.rowshard.row_range(C5_ROWS, rank, world)
    x, y = logistic_data_f32(C5_ROWS, C5_FEAT, C5_SEED, rows=(a, b))
    model = ts.logistic_regression_model(ts.LogisticRegressionData(x, y), precision=args.precision)
    del x, y
    model.device_spec.handle(dev)
    if world > 1:
        ts.rowshard.connect(model.device_spec, rank, world, ts.rowshard.torch_all_gather(), device=dev)
    W, S = args.num_warmup, args.num_samples
    peak, peak_kind = peaks()
    times, lfs, evs = [], [], []
    clocks = ClockSampler(local)
    for s in range(args.warmup + args.steps):
        cfg = ts.RunConfig(model={"model": "logistic_regression"}, num_chains=1, num_warmup=W, num_samples=S,
                           seed=args.seed + s)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if s == args.warmup:
            clocks.__enter__()
        r = ts.run_device(model, cfg, ts.chain_keys(args.seed + s, 1), dev, sync=False)
        r.event_ms[1].synchronize()
        if s >= args.warmup:
            times.append(r.event_ms[0].elapsed_time(r.event_ms[1]))
            lfs.append(float(r.stats.cpu().numpy()[0][:, 1].sum()))
            evs.append(float(r.evals.cpu().numpy()[0]))
    clocks.__exit__(None, None, None)
    t_ms = sum(times)
    if world > 1:
        t = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())
    lf, ev = sum(lfs), sum(evs)  # one replicated chain: counted once
    achieved = C5_BYTES_PER_PASS * ev / (t_ms / 1000.0) / 1e9
    if rank == 0:
        print(json.dumps({
            "metric": "leapfrog_steps_per_sec", "value": lf / (t_ms / 1000.0), "unit": "leapfrog/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64" if args.precision == "fp64" else "f32", "data": "synthetic",
            "config": {"workload": f"logistic NUTS 8,000,000 x 255 (D=256), 1 chain, rows sharded over {world} GPU(s),"
                                   f" max_tree_depth 10, {W}+{S} draws per step",
                       "precision": args.precision, "parallelism": f"rows{world}",
                       "l2": "X (8.2 GB) >> L2: every pass streams from HBM"},
            "leapfrogs_per_step": lf / args.steps, "passes_per_step": ev / args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * world, "unit": "GB/s",
                         "frac": achieved / (peak * world), "traffic": None, "peak_kind": peak_kind,
                         "bytes_per_pass": C5_BYTES_PER_PASS},
            "gpu_launches": args.steps, "clocks": clocks.summary(),
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_dense(args):
    """1000-D correlated Gaussian (Sigma = Q diag(logspace(-2,2)) Q^T,
    Q from the QR of an N(0,1) matrix, seed 4), dense mass M^-1 = Sigma, --chains chains
    (default 1024), --num-warmup/--num-samples draws; chains sharded over ranks (weak: each
    rank runs its shard in one lockstep launch).  One lockstep step = one tcgen05 TF32 GEMM
    of 2*D*D*C flops for all chains' gradients.  Not the driver's headline line."""
    import torch
    import torch.distributed as dist

    import paper_1912_11554_b200 as ts

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    D = 1000
    C = args.chains if args.chains != 8192 else 1024
    g = np.random.default_rng(4)
    Q, _ = np.linalg.qr(g.standard_normal((D, D)))
    lam = np.logspace(-2, 2, D)
    Sigma = (Q * lam) @ Q.T
    P = (Q / lam) @ Q.T
    prec = "fp64" if args.precision == "fp64" else "tf32"
    model = ts.dense_gaussian_model(P, inv_mass=Sigma, precision=prec)
    keys = ts.chain_keys(4, C)
    mine = [keys[c] for c in ts.chains.shard_range(C, rank, world)]
    cfg = ts.RunConfig(model={"model": "dense_gaussian"}, num_chains=C, num_warmup=args.num_warmup,
                       num_samples=args.num_samples, seed=4)
    times, lfs, steps = [], [], []
    clocks = ClockSampler(local)
    last = None
    for s in range(args.warmup + args.steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if s == args.warmup:
            clocks.__enter__()
        r = ts.run_device(model, cfg, mine, dev)
        if s >= args.warmup:
            times.append(r.event_ms)
            lfs.append(float(r.stats.cpu().numpy()[:, :, 1].sum()))
            steps.append(float(r.evals.cpu().numpy().max()))
            last = r
    clocks.__exit__(None, None, None)
    t = torch.tensor([sum(times), sum(lfs)], dtype=torch.float64, device=dev)
    if world > 1:
        tm = t[:1].clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        tl = t[1:].clone()
        dist.all_reduce(tl, op=dist.ReduceOp.SUM)
        t = torch.cat([tm, tl])
    t_ms, lf = float(t[0]), float(t[1])
    Cr = len(mine)
    flops = 2.0 * D * D * (-(-Cr // 64) * 64) * sum(steps)
    tflops = flops / (sum(times) / 1e3) / 1e12
    peak = None
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peak = 0.5 * float(json.load(fh)["bf16_tflops"])  # dense TF32 = half the bf16 rate
    except Exception:
        peak = 1125.0
    if rank == 0:
        samples = last.samples.cpu().numpy()
        print(json.dumps({
            "metric": "leapfrog_steps_per_sec", "value": lf / (t_ms / 1000.0), "unit": "chain-leapfrog/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": prec, "data": "synthetic",
            "config": {"workload": f"1000-D correlated Gaussian, dense mass, {C} chains, batched tcgen05 gradient steps, "
                                   f"{args.num_warmup}+{args.num_samples} draws", "parallelism": f"chains{world}"},
            "lockstep_steps_per_run": sum(steps) / args.steps, "us_per_lockstep_step": 1e3 * sum(times) / sum(steps),
            "roofline": {"bound": "tensor", "achieved": tflops, "peak": peak, "unit": "TFLOP/s", "frac": tflops / peak,
                         "traffic": None, "note": "GEMM flops only; the step is bound by the chains' vector work"},
            "min_ess_rank0": float(np.nanmin(ts.ess(samples))), "gpu_launches": args.steps,
            "clocks": clocks.summary(),
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "dense":
        return run_dense(args)
    if args.config in ("eight_schools", "gauss10"):
        return run_eight_schools(args)
    if args.config == "rowshard":
        return run_row_sharded(args)

    import torch
    import torch.distributed as dist

    import paper_1912_11554_b200 as ts

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    x32, y8 = make_data()
    cfg_for = lambda seed: ts.RunConfig(model={"model": "logistic_regression"}, num_chains=1,  # noqa: E731
                                        num_warmup=args.num_warmup, num_samples=args.num_samples, seed=seed)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > L2
    peak, peak_kind = peaks()

    def timed_runs(precision, with_clocks):
        """W untimed + K timed full runs; device time per launch (CUDA events)."""
        model = ts.logistic_regression_model(ts.LogisticRegressionData(x32, y8), precision=precision)
        model.device_spec.handle(dev)
        ms_list, lf_list, ev_list, ess_list = [], [], [], []
        last = None
        clocks = ClockSampler(local)
        for s in range(args.warmup + args.steps):
            seed = args.seed + 1000 * s + rank
            keys = ts.chain_keys(seed, 1)
            flush.fill_(float(s))
            barrier()
            if s == args.warmup and with_clocks:
                clocks.__enter__()
            r = ts.run_device(model, cfg_for(seed), keys, dev, sync=False)
            r.event_ms[1].synchronize()
            barrier()
            if s >= args.warmup:
                ms_list.append(r.event_ms[0].elapsed_time(r.event_ms[1]))
                st = r.stats.cpu().numpy()[0]
                lf_list.append(float(st[:, 1].sum()))
                ev_list.append(float(r.evals.cpu().numpy()[0]))
                samples = r.samples.cpu().numpy()[0]
                ess_list.append(float(np.nanmin(ts.ess(samples[None]))))
                last = r
        if with_clocks:
            clocks.__exit__(None, None, None)
        t_total_ms = max_over_ranks(sum(ms_list))
        lf_total = sum_over_ranks(sum(lf_list))
        ess_total = sum_over_ranks(sum(ess_list))
        # roofline of the persistent kernel (this rank's own launches and clock)
        achieved = ALGO_BYTES_PER_PASS * sum(ev_list) / (sum(ms_list) / 1000.0) / 1e9
        # the fused pass alone: 200 passes in one launch, timed inside the kernel
        q = torch.from_numpy(np.asarray(last.samples.cpu().numpy()[0, -1])).to(dev)
        out = torch.zeros(12, dtype=torch.float64, device=dev)
        lib = ts._lib.load_library()
        h = model.device_spec.handle(dev)
        ts._lib.check(lib.ts_eval_bench(h, q.data_ptr(), 20, out.data_ptr(), ts._lib.stream_ptr(torch)))
        flush.fill_(1.0)
        ts._lib.check(lib.ts_eval_bench(h, q.data_ptr(), 200, out.data_ptr(), ts._lib.stream_ptr(torch)))
        torch.cuda.synchronize()
        eval_us = float(out.cpu().numpy()[1]) / 1000.0 / 200
        eval_gbs = ALGO_BYTES_PER_PASS / (eval_us * 1e-6) / 1e9
        # DRAM traffic per data pass from the committed ncu capture of this kernel
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", f"r1_ncu_run_{precision}.json")) as fh:
                rec = json.load(fh)[0]
            traffic = rec["dram_bytes_per_pass"]
        except Exception:
            pass
        return {
            "value": lf_total / (t_total_ms / 1000.0),
            "ms_per_step": t_total_ms / args.steps,
            "ess_per_sec": ess_total / (t_total_ms / 1000.0),
            "leapfrogs_per_step": lf_total / args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_per": "data pass (ncu, profiles/)",
                         "peak_kind": peak_kind, "bytes_per_pass": ALGO_BYTES_PER_PASS, "passes": sum(ev_list)},
            "eval_only": {"us_per_pass": eval_us, "achieved_gbs": eval_gbs, "frac": eval_gbs / peak},
            "clocks": clocks.summary() if with_clocks else None,
            "last": last,
        }

    main_m = timed_runs(args.precision, True)
    other = "fp64" if args.precision == "fp32" else "fp32"
    other_m = None if args.single_precision else timed_runs(other, False)
    last = main_m["last"]

    # ---------------------------------------------------------------- end to end through the public API
    e2e = None
    if not args.no_e2e:
        xp = torch.from_numpy(x32).pin_memory()
        yp = torch.from_numpy(y8).pin_memory()
        e_ms, e_lf = [], []
        h2d = x32.nbytes + y8.nbytes
        d2h = 0
        for s in range(max(1, args.steps)):
            seed = args.seed + 7777 + 1000 * s + rank
            barrier()
            t0 = time.perf_counter()
            # the user's calls: model from host arrays (pinned), then run()
            m2 = ts.logistic_regression_model(ts.LogisticRegressionData(xp.numpy(), yp.numpy()),
                                              precision=args.precision)
            res = ts.run(cfg_for(seed), m2, devices=[local])
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            barrier()
            e_ms.append(max_over_ranks(el * 1000.0))
            e_lf.append(sum_over_ranks(float(res[0].total_leapfrogs)))
            d2h = (res[0].samples.nbytes + (args.num_warmup + args.num_samples) * 5 * 8
                   + (2 + args.num_warmup + N_FEAT + 1) * 8)
            del m2, res
        e2e = {"value": sum(e_lf) / (sum(e_ms) / 1000.0), "unit": "leapfrog/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        samples = last.samples.cpu().numpy()[0]
        adapt = last.adapt.cpu().numpy()[0]
        W = args.num_warmup
        lf, el, threads, sample = cpu_baseline(x32, y8, args.cpu_seconds, start=samples[-1], step=float(adapt[1]),
                                               inv=adapt[2 + W:].tolist(), seed=args.seed)
        cpu = {"value": lf / el, "unit": "leapfrog/s", "cores": threads, "kind": "port",
               "sample": f"{sample}: {lf} leapfrogs in {el:.1f} s (fused OpenMP fp64 pass, {threads} threads)"}

    if rank == 0:
        line = {
            "metric": "leapfrog_steps_per_sec",
            "value": main_m["value"],
            "unit": "leapfrog/s",
            "n_gpus": world,
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
                "parallelism": f"replicas{world}", "l2": "256 MB buffer written between steps (X+y = 126 MB ~ L2)",
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
            line[f"{other}_mode"] = {k: other_m[k] for k in ("value", "ms_per_step", "ess_per_sec",
                                                            "leapfrogs_per_step", "roofline", "eval_only")}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
