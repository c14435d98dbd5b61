"""C4 step variants on one GPU (device time, CUDA events, L2 flushed):
full QR with M = R^-1 Q^T (default), full QR with the per-stage tiled back
substitution (NS_TILED_BS), QR reused (NS_REUSE_QR).  Env knobs are read at
handle creation (NS_QR_SMALLREGS ...).  usage: python scripts/time_c4.py [K]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2301_12659_b200 as P  # noqa: E402
import synth  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 4
sys_ = synth.build_config("C4", K=K)
x0 = torch.tensor(synth.make_x(sys_, "near", seed=1), device="cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
out = {"K": K, "env": {k: v for k, v in os.environ.items() if k.startswith("NS_")}}
h = P.NewtonSystem.from_system(sys_)
for name, fl in (("full_M", P.NS_LEDGER), ("full_tiled_bs", P.NS_TILED_BS | P.NS_LEDGER),
                 ("reuse", P.NS_REUSE_QR | P.NS_LEDGER)):
    x = x0.clone()
    for _ in range(2):
        x.copy_(x0)
        h.step(x, flags=fl & ~P.NS_LEDGER if name != "reuse" else fl & ~P.NS_LEDGER)
    torch.cuda.synchronize()
    h.reset_ledger()
    ts = []
    for _ in range(3):
        x.copy_(x0)
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        h.step(x, flags=fl)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    led = h.ledger()
    out[name] = {"ms": sorted(ts)[1], "ledger": {k: led[k] / max(1, led["steps"]) for k in
                                                 ("ms_convolution", "ms_qr", "ms_stage", "ms_residual", "ms_total")}}
print(json.dumps(out))
