"""Phase split of the batched step (C5): NS_BATCH_TRACE stamps of each CTA's
first path -> median microseconds per phase.  usage: python scripts/trace_batch.py [K]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["NS_BATCH_TRACE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_12659_b200 as P  # noqa: E402
import synth  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 2
base = synth.triangular_system(32, 15, K, seed=12665, name="C5")
B = 4096
X0 = torch.tensor(np.stack([synth.make_x(base, "near", seed=100)] * B), device="cuda:0")
R = torch.tensor(np.stack([base.rhs] * B), device="cuda:0")
h = P.NewtonSystem.from_system(base, max_batch=B)
X = X0.clone()
for _ in range(3):
    X.copy_(X0)
    h.step_batched(X, R)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
X.copy_(X0)
a.record()
h.step_batched(X, R)
b.record()
torch.cuda.synchronize()
t = h.batch_trace().astype(np.float64)
ph = np.diff(t[:, :6], axis=1) / 1e3
names = ["evaldiff", "qr", "tiles", "stages", "residual"]
out = {"K": K, "ctas": len(t), "step_ms": a.elapsed_time(b),
       "first_path_us_median": {n: float(np.median(ph[:, i])) for i, n in enumerate(names)},
       "first_path_total_us": float(np.median(t[:, 5] - t[:, 0]) / 1e3)}
print(json.dumps(out))
