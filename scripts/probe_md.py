"""Print md-op latencies (cycles, dependent chain on one warp) and the FP64 peaks."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2301_12659_b200 as P

out = {"fp64_dfma": P.fp64_peak_probe(0, "dfma"), "fp64_dadd": P.fp64_peak_probe(0, "dadd")}
for K in (2, 4, 8):
    out[f"K{K}"] = {op: P.md_latency_probe(K, op) for op in ("fma", "add", "mul", "recip", "sqrt")}
out["barrier_us"] = {b: P.barrier_probe(b) for b in (16, 32, 64, 148)}
print(json.dumps(out))
