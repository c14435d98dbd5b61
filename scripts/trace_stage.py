"""Per-stage stamps of the split stage loop's critical chain (NS_STAGE_TRACE=1)."""
import json
import os
import sys

os.environ["NS_STAGE_TRACE"] = "1"
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2301_12659_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
s = synth.build_config(cfg)
h = P.NewtonSystem.from_system(s)
x = torch.tensor(synth.make_x(s, "near"), device="cuda")
for _ in range(3):
    xx = x.clone()
    h.step(xx)
torch.cuda.synchronize()
t, pd = h.stage_trace()
t = t.astype(float)
pd = pd.astype(float)
# bulk latency: dx_{k-2} published (t[k-2, 3]) -> last row of pend_k (pd[k])
lat = [(pd[k] - t[k - 2, 3]) / 1e3 for k in range(2, len(pd)) if pd[k] > 0]
d = np.diff(t, axis=1) / 1e3
per = np.diff(t[:, 0]) / 1e3
out = {"config": cfg, "us_mean": {"wait_pend": float(d[:, 0].mean()), "rowdot_b'": float(d[:, 1].mean()),
                                  "matvec_dx": float(d[:, 2].mean())},
       "stage_period_us": float(per.mean()), "span_us": float((t[-1, 3] - t[0, 0]) / 1e3),
       "bulk_latency_us": [round(v, 2) for v in lat],
       "per_stage_us": [[round(v, 2) for v in row] for row in d.tolist()]}
print(json.dumps(out))
