"""Compare the grid QR with the critical-chain variant (NS_QR_CRIT) on a small
system: R diagonal and the solve's dx, NaN positions.  usage: python scripts/debug_crit.py [K] [n] [wy]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2301_12659_b200 as P  # noqa: E402
import synth  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
wy = sys.argv[3] if len(sys.argv) > 3 else "0"
sys_ = synth.triangular_system(n, 6, K, seed=53)
x = torch.tensor(synth.make_x(sys_, "rough", seed=54), device="cuda:0")
out = {}
for crit in ("0", "1"):
    os.environ["NS_QR_CRIT"] = crit
    os.environ["NS_WY"] = wy
    os.environ["NS_WY_BW"] = "16"
    h = P.NewtonSystem.from_system(sys_)
    b, A, A0 = h.eval_diff(x)
    dx = h.toeplitz_solve(b, A, A0)
    rd = h.r_diag()
    torch.cuda.synchronize()
    out[crit] = (rd.cpu().numpy(), dx.cpu().numpy(), h.status().status_bits)
rd0, dx0, s0 = out["0"]
rd1, dx1, s1 = out["1"]
print("status", s0, s1)
print("rdiag grid", rd0[0])
print("rdiag crit", rd1[0])
print("rdiag rel diff", np.abs(rd1[0] - rd0[0]) / np.abs(rd0[0]))
print("dx nan (k, i):", [tuple(v) for v in np.argwhere(~np.isfinite(dx1[0]))][:20])
print("dx rel diff per k", [float(np.max(np.abs(dx1[0, k] - dx0[0, k]) / (np.abs(dx0[0, k]) + 1e-300))) for k in range(dx0.shape[1])])
