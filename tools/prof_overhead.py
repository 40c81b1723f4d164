"""Per-pass time of the fused logistic pass vs N and grid size, timed inside the
kernel (globaltimer) with CTA-0 phase cycle counters.  Scratch profiling tool."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_1912_11554_b200 as ts
from tests_data import logistic_data

lib = ts._lib.load_library()
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
sizes = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [148 * 32, 148 * 32 * 10, 581012]
grids = [int(v) for v in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0]
clk = torch.cuda.get_device_properties(0).clock_rate if hasattr(torch.cuda.get_device_properties(0), "clock_rate") else 1.965e6
for n in sizes:
    x, y = logistic_data(n, 54, 1)
    m = ts.logistic_regression_model(ts.LogisticRegressionData(x.astype(np.float32), y), precision=prec)
    for grid in grids:
        m.device_spec.set_grid(grid)
        h = m.device_spec.handle(0)
        q = torch.from_numpy(np.random.default_rng(0).standard_normal(55) * 0.05).cuda()
        out = torch.zeros(12, dtype=torch.float64, device="cuda")
        R = 100
        ts._lib.check(lib.ts_eval_bench(h, q.data_ptr(), 5, out.data_ptr(), 0))
        ts._lib.check(lib.ts_eval_bench(h, q.data_ptr(), R, out.data_ptr(), 0))
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        cyc = o[2:10].view(np.uint64).astype(float) / R
        per = o[1] / R / 1000.0
        print(f"{prec} n={n} grid={grid or 'all'}: {per:.2f} us/pass {n*(54*4+1)/per/1e3:.0f} GB/s | CTA0 cycles/pass "
              f"prior {cyc[0]:.0f} pass {cyc[1]:.0f} [entry {cyc[4]:.0f} loop {cyc[5]:.0f} warpred {cyc[6]:.0f} ctared {cyc[7]:.0f}] barrier {cyc[2]:.0f} reduce {cyc[3]:.0f}", flush=True)
