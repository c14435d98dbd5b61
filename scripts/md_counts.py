"""ns_md_op over n elements for every K and op, to count the FP64 instructions
of one md operation with ncu (sm__sass_thread_inst_executed_op_{dadd,dmul,dfma}
/ n): the static mix of perfmodel.MD_FMA_MIX against the hardware.
usage: ncu --metrics ... python scripts/md_counts.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2301_12659_b200 as P  # noqa: E402

n = 1 << 16
for K in (2, 4, 8):
    a = torch.rand((K, n), dtype=torch.float64, device="cuda:0") + 1.0
    a[1:] *= 1e-17
    b = a.flip(1).contiguous()
    for op in ("add", "mul", "fma"):
        c = torch.zeros_like(a)
        P.md_op(K, op, a, b, c)
torch.cuda.synchronize()
print("n", n)
