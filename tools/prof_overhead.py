"""Per-pass time of the fused logistic pass vs N and grid size (scratch profiling)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_1912_11554_b200 as ts
from tests_data import logistic_data

lib = ts._lib.load_library()
prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
for n in (148 * 32, 148 * 32 * 10, 148 * 32 * 40, 581012):
    x, y = logistic_data(n, 54, 1)
    m = ts.logistic_regression_model(ts.LogisticRegressionData(x.astype(np.float32), y), precision=prec)
    for grid in (0, 74, 16, 1):
        if grid == 1 and n > 148 * 32 * 10:
            continue
        m.device_spec.set_grid(grid)
        h = m.device_spec.handle(0)
        q = torch.from_numpy(np.random.default_rng(0).standard_normal(55) * 0.05).cuda()
        out = torch.empty(1, dtype=torch.float64, device="cuda")
        res = []
        for r in (10, 110):
            ts._lib.check(lib.ts_eval_bench(h, q.data_ptr(), 2, out.data_ptr(), 0))
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ts._lib.check(lib.ts_eval_bench(h, q.data_ptr(), r, out.data_ptr(), 0))
            e1.record(); e1.synchronize()
            res.append(e0.elapsed_time(e1) * 1000)
        per = (res[1] - res[0]) / 100
        print(f"{prec} n={n} tiles={(n+31)//32} grid={grid or 148}: {per:.2f} us/pass (launch overhead {res[0]-10*per:.1f} us)  {n*(54*4+1)/per/1e3:.0f} GB/s", flush=True)
