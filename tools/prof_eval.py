"""Profiling driver: fused potential+gradient passes inside one persistent
launch (ts_eval_bench).
Usage: python tools/prof_eval.py [fp64|fp32] [repeats] [N] [p] [seed]
Default shape: covtype (581012 x 54, seed 20191222); config 5: 8000000 255 20191223."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_1912_11554_b200 as ts
from tests_data import logistic_data_f32

prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
N = int(sys.argv[3]) if len(sys.argv) > 3 else 581012
P = int(sys.argv[4]) if len(sys.argv) > 4 else 54
seed = int(sys.argv[5]) if len(sys.argv) > 5 else 20191222
t0 = time.time()
x, y = logistic_data_f32(N, P, seed)
print(f"data {N}x{P} in {time.time() - t0:.1f} s", flush=True)
m = ts.logistic_regression_model(ts.LogisticRegressionData(x, y), precision=prec)
h = m.device_spec.handle(0)
lib = ts._lib.load_library()
q = torch.from_numpy(np.random.default_rng(0).standard_normal(P + 1) * 0.05).cuda()
out = torch.zeros(12, dtype=torch.float64, device="cuda")
algo = 4 * N * P + N
for r in (5, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ts._lib.check(lib.ts_eval_bench(h, q.data_ptr(), r, out.data_ptr(), 0))
    e1.record(); e1.synchronize()
    us = e0.elapsed_time(e1) * 1000 / r
    ins = float(out.cpu().numpy()[1]) / 1000.0 / r
    print(f"{prec} {N}x{P} repeats={r}: {us:.2f} us/pass (launch)  {ins:.2f} us/pass (in-kernel)  "
          f"{algo/ins/1e3:.1f} GB/s", flush=True)
