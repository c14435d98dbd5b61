"""Per-step stamps of the cluster QR look-ahead warp (NS_CQR_TRACE=1)."""
import json
import os
import sys

os.environ["NS_CQR_TRACE"] = "1"
import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2301_12659_b200 as P

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
s = synth.build_config(cfg)
h = P.NewtonSystem.from_system(s)
x = torch.tensor(synth.make_x(s, "near"), device="cuda")
res = torch.zeros((s.K, 3), dtype=torch.float64, device="cuda")
for _ in range(3):
    xx = x.clone()
    h.step(xx, res)
torch.cuda.synchronize()
buf = np.zeros((s.n, 8), np.int64)
import ctypes
fn = P.lib().ns_get_qr_trace
fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
fn.restype = ctypes.c_int32
m = fn(h._h, buf.ctypes.data, s.n)
phs = buf[m - 1, :5].astype(float)
phases = {"prologue_us": (phs[1] - phs[0]) / 1e3, "steps_us": (phs[2] - phs[1]) / 1e3,
          "out_RQt_us": (phs[3] - phs[2]) / 1e3, "form_M_us": (phs[4] - phs[3]) / 1e3}
t = buf[: m - 1].astype(float)
ok = t[:, 0] > 0
t = t[ok]
names = ["wait_A", "partial_dot", "wait_B", "v0dot_wait_C", "update", "publish_A", "reflector"]
d = np.diff(t, axis=1)
out = {"config": cfg, "steps": int(ok.sum()), "us_per_step_mean": {k: float(d[:, i].mean() / 1e3) for i, k in enumerate(names)},
       "step_period_us": float(np.diff(t[:, 7]).mean() / 1e3) if len(t) > 1 else 0.0,
       "span_us": float((t[-1, 7] - t[0, 0]) / 1e3), "phases": phases}
print(json.dumps(out, indent=1))
