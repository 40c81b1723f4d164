"""Diagnostic (not collected by pytest): fp32 covtype pass vs the fp64 oracle,
per log-likelihood precision mode (TS_LLMODE), with the pass time.
Usage: python tests/diag_fp32_error.py"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

if len(sys.argv) > 2 and sys.argv[1] == "child":
    sys.path.insert(0, ROOT)
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import torch

    import paper_1912_11554_b200 as ts
    import turnstile_oracle as o
    from tests_data import logistic_data

    x, y = logistic_data(581012, 54, 20191222)
    X = np.hstack([x, np.ones((x.shape[0], 1))])
    th = np.zeros(55)
    for _ in range(12):
        s = 1 / (1 + np.exp(-(X @ th)))
        g = th - X.T @ (y - s)
        H = np.eye(55) + (X * (s * (1 - s))[:, None]).T @ X
        th = th - np.linalg.solve(H, g)
    om = o.Model("logistic_regression", 55, x=x, y=y, fused_omp=True)
    for prec in sys.argv[2].split(","):
        m = ts.logistic_regression_model(ts.LogisticRegressionData(x, y), precision=prec)
        res = []
        for name, q in (("zero", np.zeros(55)), ("mode", th), ("mode+0.01", th + 0.01), ("rand", np.random.default_rng(1).standard_normal(55) * 0.1)):
            got = ts.models.potential_and_gradient(m.device_spec, q[None, :])[0]
            U, gg = om._fused(q.tolist())
            res.append(f"{name}: dU={got[0] - U:+.3e} max|dg|={np.abs(got[1:] - np.asarray(gg)).max():.2e}")
        h = m.device_spec.handle(0)
        lib = ts._lib.load_library()
        qd = torch.from_numpy(th).cuda()
        out = torch.zeros(12, dtype=torch.float64, device="cuda")
        ts._lib.check(lib.ts_eval_bench(h, qd.data_ptr(), 20, out.data_ptr(), 0))
        ts._lib.check(lib.ts_eval_bench(h, qd.data_ptr(), 400, out.data_ptr(), 0))
        torch.cuda.synchronize()
        us = float(out.cpu().numpy()[1]) / 1000.0 / 400
        print(f"LL={os.environ.get('TS_LLMODE', 'default')} {prec}: pass {us:.2f} us | " + " | ".join(res), flush=True)
else:
    for ll in sys.argv[1:] or ("0", "1", "2", "3", "4"):
        env = dict(os.environ, TS_LLMODE=ll)
        subprocess.call([sys.executable, __file__, "child", "fp32" if ll != "1" else "fp32,fp64"], env=env)
