"""Time ts_pooled_covariance at the config-4 shape: C chains x S draws x D.

python tools/cov_bench.py [C S D]   (prints one JSON line)
FP64-pipe bound: the lower triangle costs n*D*(D+1) flops (FMA = 2).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1912_11554_b200 as t  # noqa: E402

C, S, D = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (1024, 200, 1000)
x = torch.randn((C, S, D), dtype=torch.float64, device="cuda")
for _ in range(3):
    t.pooled_covariance(x)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    t.pooled_covariance(x)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / reps
n = C * S
tiles = -(-D // 64)
flops = n * (tiles * (tiles + 1) // 2) * 64 * 64 * 2
print(json.dumps({"C": C, "S": S, "D": D, "ms": ms, "useful_tflops": n * D * (D + 1) / ms / 1e9,
                  "issued_tflops": flops / ms / 1e9, "input_gb": n * D * 8 / 1e9}))
