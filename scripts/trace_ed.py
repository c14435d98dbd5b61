"""Trace the eval/diff job queue of one step (NS_TRACE=1) and summarise it."""
import json
import os
import sys

os.environ["NS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2301_12659_b200 as P
import synth

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
if cfg.startswith("single"):
    # one long monomial alone (no contention): eq 0 = x_0 ... x_{n-1}, eq i = x_i
    K = 4 if cfg == "single4" else 8
    n, D = (64, 31) if K == 4 else (128, 63)
    eqs = [[list(range(n))]] + [[[i]] for i in range(1, n)]
    s = synth.custom_system(eqs, [1.0] * n, D, K, synth.draw_alphas(n, 5))
else:
    s = synth.build_config(cfg)
h = P.NewtonSystem.from_system(s)
x0 = torch.tensor(synth.make_x(s, "near", seed=1), device="cuda")
for _ in range(3):
    x = x0.clone()
    h.step(x)
torch.cuda.synchronize()
t, jb = h.trace()
import ctypes
cap = 1 << 22
raw = np.zeros((cap, 3), np.int64)
jbr = np.zeros((cap, 4), np.int32)
nj = P.lib().ns_get_trace(h._h, raw.ctypes.data, cap, jbr.ctypes.data)
steps = raw.reshape(-1)[3 * nj: 3 * nj + 4 * 256].reshape(256, 4)
inner = raw.reshape(-1)[3 * nj + 4 * 256: 3 * nj + 6 * 256].reshape(256, 2)
L = int(jbr[0, 2]) if jbr[0, 0] <= 1 else 0
if L:
    st = steps[:L]
    conv = (st[:, 1] - st[:, 0]).astype(float)
    sync = (st[:, 2] - st[:, 1]).astype(float)
    gap = (st[1:, 0] - st[:-1, 2]).astype(float)
    step_stats = {"job0_len": L, "conv_cycles_mean": float(conv.mean()), "conv_cycles_min": float(conv.min()),
                  "wait_sync_cycles_mean": float(sync.mean()),
                  "terms_cycles_mean": float((inner[:L, 0] - st[:, 0]).mean()),
                  "butterfly_cycles_mean": float((inner[:L, 1] - inner[:L, 0]).mean()),
                  "store_cycles_mean": float((st[:, 1] - inner[:L, 1]).mean()), "gap_cycles_mean": float(gap.mean()) if L > 1 else 0.0}
else:
    step_stats = {}
t0 = t[:, 0].min()
t = (t - t0) / 1e3  # us
out = {"config": cfg, "njobs": int(len(t)), "span_us": float(t[:, 2].max())}
for ty, name in ((0, "fwd_chain"), (1, "bwd_chain"), (2, "cross"), (3, "equation")):
    sel = jb[:, 0] == ty
    if sel.any():
        dur = t[sel, 2] - np.where(t[sel, 1] > 0, t[sel, 1], t[sel, 0])
        out[name] = {"count": int(sel.sum()), "first_pop": float(t[sel, 0].min()), "last_done": float(t[sel, 2].max()),
                     "mean_run_us": float(dur.mean()), "max_run_us": float(dur.max())}
# the longest chain: per-step time
sel = (jb[:, 0] == 0)
i = np.argmax(jb[:, 2] * sel)
out["longest_fwd_chain"] = {"len": int(jb[i, 2]), "start": float(t[i, 0]), "done": float(t[i, 2]),
                            "us_per_step": float((t[i, 2] - t[i, 0]) / max(1, jb[i, 2]))}
out["job0_steps"] = step_stats
print(json.dumps(out, indent=1))
