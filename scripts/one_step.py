"""Run `steps` Newton steps of a BASELINE config on cuda:0 after one warm-up
step (for ncu / compute-sanitizer runs: no timing, no oracle).
usage: python scripts/one_step.py C3 [steps] [precision] [batch (C5)]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2301_12659_b200 as P  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
K = int(sys.argv[3]) if len(sys.argv) > 3 else None
if cfg == "C5":
    import numpy as np
    base = synth.triangular_system(32, 15, K or 2, seed=12665, name="C5")
    B = int(sys.argv[4]) if len(sys.argv) > 4 else 4096
    xs = synth.make_x(base, "near", seed=100)
    X0 = torch.tensor(np.stack([xs] * B), device="cuda:0")
    R = torch.tensor(np.stack([base.rhs] * B), device="cuda:0")
    h = P.NewtonSystem.from_system(base, max_batch=B)
    X = X0.clone()
    for _ in range(steps + 1):
        X.copy_(X0)
        h.step_batched(X, R)
else:
    sys_ = synth.build_config(cfg, K=K)
    h = P.NewtonSystem.from_system(sys_)
    x0 = torch.tensor(synth.make_x(sys_, "near", seed=1), device="cuda:0")
    x = x0.clone()
    res = torch.zeros((sys_.K, 3), dtype=torch.float64, device="cuda:0")
    for _ in range(steps + 1):
        x.copy_(x0)
        h.step(x, res)
torch.cuda.synchronize()
print("status", h.status().status_bits)
