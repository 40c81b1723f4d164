"""Profiling driver: covtype-shaped fused potential+gradient passes inside one
persistent launch (ts_eval_bench).  Usage: python tools/prof_eval.py [fp64|fp32] [repeats]"""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_1912_11554_b200 as ts
from tests_data import logistic_data

prec = sys.argv[1] if len(sys.argv) > 1 else "fp64"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
x, y = logistic_data(581012, 54, 20191222)
m = ts.logistic_regression_model(ts.LogisticRegressionData(x.astype(np.float32), y), precision=prec)
h = m.device_spec.handle(0)
lib = ts._lib.load_library()
q = torch.from_numpy(np.random.default_rng(0).standard_normal(55) * 0.05).cuda()
out = torch.empty(1, dtype=torch.float64, device="cuda")
for r in (5, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ts._lib.check(lib.ts_eval_bench(h, q.data_ptr(), r, out.data_ptr(), 0))
    e1.record(); e1.synchronize()
    us = e0.elapsed_time(e1) * 1000 / r
    print(f"{prec} repeats={r}: {us:.2f} us/pass  {126079604/us/1e3:.1f} GB/s")
