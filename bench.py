#!/usr/bin/env python
"""bench.py -- one Newton step on truncated power series (arxiv 2301.12659) on B200.

Workload at N = 1: BASELINE.json configs[1] (C2): dim 64 one-column monomial
system (Eq.(5)), degree 31, quad double, one full Newton step
(eval/diff + Householder QR + staged updates / Q^T b / back substitution +
residual + x += dx) through the C ABI.  N > 1 (torchrun): C2 replicas, one
per GPU ("replicas only": one C2 system does not shard), weak
scaling.  --config picks another BASELINE config (C3, C1).

Prints ONE JSON line (rank 0).  value = FP64 GFLOP/s (whole job), the flop
numerator being the algorithmic md multiply-adds of the step (perfmodel.py:
triangular convolutions, the QR of [A0|I], updates, Q^T b, back substitution,
residual) times the FP64 flops of one md multiply-add of this library (FMA = 2).
ms_per_step is the Newton step time.  --impl reference times the CPU oracle
(the base contract's reference arm for this tier) on a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Newton step ms and FP64 GFLOPS (% of peak) per 2d/4d/8d at 1/2/4/8 B200"
UNIT = "GFLOP/s (FP64, FMA=2; algorithmic md multiply-adds x flops per md multiply-add)"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    p.add_argument("--reuse-qr", action="store_true", help="C4: NS_REUSE_QR in the timed steps (QR once)")
    p.add_argument("--batch", type=int, default=4096, help="C5: total paths (partitioned over ranks)")
    p.add_argument("--driver", action="store_true",
                   help="NEXT-1: time whole staggered Newton runs (ns_run_newton) from 'start' to convergence")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of oracle work for cpu_baseline")
    return p.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload_desc(name, sys_):
    prec = {2: "double double", 4: "quad double", 8: "octo double"}[sys_.K]
    return (f"{name}: dim={sys_.n} one-column lower-triangular monomial system (Eq.(5)), "
            f"degree {sys_.D}, {prec}, one Newton step")


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        cmd = ["nvidia-smi", "-i", str(self.gpu),
               "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
               "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
               "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
               "--format=csv,noheader,nounits", "-lms", "100"]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        med = sm[len(sm) // 2] if sm else None
        return {"sm_mhz": med, "sm_max_mhz": smax, "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------------ work model
def work(sys_, nnz):
    from paper_2301_12659_b200 import perfmodel as PM
    c = PM.step_counts(sys_.eq_ptr, sys_.mono_ptr, nnz, sys_.n, sys_.d)
    per_class = {"convolution": c["convolution"], "qr": c["qr"], "stage": c["stage"], "residual": c["residual"]}
    total = sum(per_class.values())
    return c, per_class, total


# ------------------------------------------------------------------ CPU oracle (bounded sample)
def oracle_sample(sys_, x_np, budget_s: float, rotate: int = 0):
    """Time the oracle (O-hp tier) on a bounded sample of the step: the
    evaluation/differentiation of a subset of equations plus the block solve
    of the first stages.  Returns (seconds, fraction of the full step's oracle
    work the sample covers, description).  Work is counted in oracle
    multiply-adds: eval/diff of row i with m variables = (m-1) + (3m-2)
    convolutions of d(d+1)/2 terms (value + before/after partial products);
    solve = n^3/3 (LU) + sum_k (k nnz + n^2)."""
    from oracle import newton as O
    n, d = sys_.n, sys_.d
    F = O.field_for(sys_.K)
    tri = d * (d + 1) // 2
    rows_cost = []
    for i in range(n):
        m = sum(int(sys_.mono_ptr[t + 1] - sys_.mono_ptr[t]) for t in O.eq_monomials(sys_, i))
        rows_cost.append(((m - 1) + (3 * m - 2)) * tri)
    nnz = sum(len(r) for r in O.jacobian_pattern(sys_))
    stage_cost = [k * nnz + n * n for k in range(d)]
    full = sum(rows_cost) + n ** 3 // 3 + sum(stage_cost)
    # calibrate: ~5 us per multiply-add at 256-1024 bits (mpmath, pure Python)
    target = max(budget_s / 6e-6, 1.0)
    frac = min(1.0, target / full)
    # equations: every r-th row, rotating start
    stride = max(1, int(round(1.0 / frac)))
    rows = list(range(rotate % stride, n, stride))
    # stages: first ks stages with cost ~ frac of the solve
    ks, acc = 1, stage_cost[0]
    solve_full = n ** 3 // 3 + sum(stage_cost)
    while ks < d and n ** 3 // 3 + acc < frac * solve_full:
        acc += stage_cost[ks]
        ks += 1
    t0 = time.perf_counter()
    if frac >= 0.999:
        # the budget covers the whole step: run it (no extrapolation)
        O.step(sys_, x_np, F, split=True)
        dt = time.perf_counter() - t0
        return dt, 1.0, f"oracle (mpmath {F.name}) full step (eval/diff of all {n} equations + block solve of all {d} stages)"
    xs = O.read_x(x_np, F)
    b_s, A_s = O.evaluate(sys_, xs, F, split=True, rows=rows)
    # the solve needs every row of A_0..A_{ks-1}: evaluate the solve's inputs on a
    # truncated series (first ks coefficients)
    import copy
    sub = copy.copy(sys_)
    sub.D = ks - 1
    sub.rhs = sys_.rhs[:, :, :ks]
    xs_k = [ser[:ks] for ser in xs]
    b_k, A_k = O.evaluate(sub, xs_k, F, split=True)
    O.solve(A_k, b_k, n, ks, F)
    dt = time.perf_counter() - t0
    tri_k = ks * (ks + 1) // 2
    done = sum(rows_cost[i] for i in rows) + sum(c // tri * tri_k for c in rows_cost) + n ** 3 // 3 + acc
    frac_done = min(1.0, done / full)
    desc = (f"oracle (mpmath {F.name}) on {len(rows)}/{n} equations for eval/diff plus the block solve "
            f"of stages 0..{ks - 1} (with their truncated eval/diff); {frac_done:.3f} of the step's "
            f"oracle multiply-adds, extrapolated by that count")
    return dt, frac_done, desc


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    ws, rank, local = dist_env()
    if ws > 1 and rank != 0:
        return
    import synth
    from paper_2301_12659_b200 import perfmodel as PM
    sys_ = synth.build_config(args.config)
    x_np = synth.make_x(sys_, "near", seed=1)
    from oracle import newton as O
    nnz = sum(len(r) for r in O.jacobian_pattern(sys_))
    _, per_class, total = work(sys_, nnz)
    flops = PM.flops(total, sys_.K)
    budget = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    for w in range(args.warmup):
        oracle_sample(sys_, x_np, budget, rotate=w)
    per_step = []
    descs = None
    for s in range(args.steps):
        dt, frac, descs = oracle_sample(sys_, x_np, budget, rotate=args.warmup + s)
        per_step.append(dt / frac)
    ms = 1e3 * sum(per_step) / len(per_step)
    value = flops / (ms * 1e-3) * 1e-9
    cores = 1
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, synth.py)",
        "config": {"workload": workload_desc(args.config, sys_)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": descs},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ C5: batch of paths
def _c5_path(p):
    import synth
    sys_ = synth.triangular_system(32, 15, 2, seed=12665 + p, name="C5")
    return synth.make_x(sys_, "near", seed=100 + p), sys_.rhs


def run_c5(args):
    """BASELINE configs[4]: 4096 independent paths (dim 32, degree 15, double
    double), paths partitioned across ranks (dist.partition), one
    ns_newton_series_step_batched per rank per step; no collective in the step.
    Strong scaling: the total batch is fixed."""
    import multiprocessing as mp

    import numpy as np
    import torch

    import paper_2301_12659_b200 as P
    import synth
    from paper_2301_12659_b200 import perfmodel as PM
    from paper_2301_12659_b200.dist import max_over_ranks, partition

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    lo, hi = partition(args.batch, ws, rank)
    with mp.Pool(min(16, os.cpu_count() or 1)) as pool:
        data = pool.map(_c5_path, range(lo, hi), chunksize=16)
    base = synth.triangular_system(32, 15, 2, seed=12665, name="C5")
    dev = torch.device(f"cuda:{local}")
    X0 = torch.tensor(np.stack([d[0] for d in data]), device=dev)
    R = torch.tensor(np.stack([d[1] for d in data]), device=dev)
    X = X0.clone()
    B = hi - lo
    res = torch.zeros((B, 2, 3), dtype=torch.float64, device=dev)
    h = P.NewtonSystem.from_system(base, max_batch=max(1, B), device=local)
    c, per_class, total = work(base, h.nnz)
    flops_path = PM.flops(total, 2)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(max(args.warmup, 3)):
        X.copy_(X0)
        h.step_batched(X, R, res)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        X.copy_(X0)
        flush.zero_()
        ev[i][0].record(stream)
        h.step_batched(X, R, res)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    ms_total = sum(a.elapsed_time(b) for a, b in ev)
    # e2e: pinned host x and rhs in, x and residuals out, every step
    Xh = X0.cpu().pin_memory(); Rh = R.cpu().pin_memory()
    Xo = torch.empty_like(Xh).pin_memory(); Ro = torch.empty((B, 2, 3), dtype=torch.float64).pin_memory()
    ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        ee[i][0].record(stream)
        X.copy_(Xh, non_blocking=True)
        R.copy_(Rh, non_blocking=True)
        h.step_batched(X, R, res)
        Xo.copy_(X, non_blocking=True)
        Ro.copy_(res, non_blocking=True)
        ee[i][1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    e2e_ms = sum(a.elapsed_time(b) for a, b in ee)
    ms_total = max_over_ranks(ms_total, dev)
    e2e_ms = max_over_ranks(e2e_ms, dev)
    ms_step = ms_total / args.steps
    value = args.batch * flops_path / (ms_step * 1e-3) * 1e-9
    probe = P.fp64_peak_probe(local, "dfma")
    peak = 2.0 * probe["ginstr_per_s"]
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded per path, synth.py; 'near' start series)",
        "config": {"workload": f"C5: batch of {args.batch} independent paths, dim=32 one-column monomial "
                               f"system, degree 15, double double, one Newton step per path",
                   "batch": args.batch, "parallelism": f"paths partitioned x{ws}",
                   "l2": "flushed (256 MiB memset) before every timed step"},
        "paths_per_s": args.batch / (ms_step * 1e-3),
        "pct_of_peak": 100.0 * value / (ws * peak),
        "e2e": {"value": args.batch * flops_path / (e2e_ms / args.steps * 1e-3) * 1e-9, "unit": UNIT,
                "h2d_bytes_per_step": (Xh.numel() + Rh.numel()) * 8 * ws,
                "d2h_bytes_per_step": (Xo.numel() + Ro.numel()) * 8 * ws, "ms_per_step": e2e_ms / args.steps},
        "roofline": {"bound": "alu", "kernel_class": "batched_step", "achieved": value / ws, "peak": peak,
                     "unit": "GFLOP/s", "frac": value / ws / peak, "traffic": None,
                     "peak_source": "measured DFMA-chain probe x2"},
        "gpu_launches": args.steps,
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


# ------------------------------------------------------------------ C4: one large system, sharded eval/diff
def run_c4(args):
    """BASELINE configs[3]: dim 1024 2-column banded (w = 32) system, degree 31,
    quad double.  Equation-owner sharding of eval/diff over the ranks
    (dist.equation_partition), row replication by all-gather over NVLink
    (torch.distributed NCCL), then the QR + stage loop + residual replicated on
    every rank (ns_newton_series_step_from).  Strong scaling (one system)."""
    import numpy as np
    import torch

    import paper_2301_12659_b200 as P
    import synth
    from paper_2301_12659_b200 import perfmodel as PM
    from paper_2301_12659_b200.dist import equation_partition, max_over_ranks, replicate_rows

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    sys_ = synth.build_config("C4")
    x_np = synth.make_x(sys_, "near", seed=1)
    dev = torch.device(f"cuda:{local}")
    h = P.NewtonSystem.from_system(sys_, device=local)
    ranges = equation_partition(sys_.eq_ptr, sys_.mono_ptr, sys_.d, ws)
    lo, hi = ranges[rank]
    if ws > 1:
        h.set_partition(lo, hi)
    rp, _ = h.pattern()
    x0 = torch.tensor(x_np, device=dev)
    x = x0.clone()
    res = torch.zeros((4, 3), dtype=torch.float64, device=dev)
    c, per_class, total = work(sys_, h.nnz)
    flops_step = PM.flops(total, sys_.K)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def one(flags):
        b, A, A0 = h.eval_diff(x)
        replicate_rows(b, A, A0, rp, ranges, rank)
        h.step_from(x, b, A, A0, res, flags=flags)

    for _ in range(max(args.warmup, 3)):
        x.copy_(x0)
        one(0)
    torch.cuda.synchronize()
    flags = P.NS_REUSE_QR if args.reuse_qr else 0
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        x.copy_(x0)
        flush.zero_()
        ev[i][0].record(stream)
        one(flags)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms_total = max_over_ranks(sum(a.elapsed_time(b) for a, b in ev), dev)
    ms_step = ms_total / args.steps
    probe = P.fp64_peak_probe(local, "dfma")
    peak = 2.0 * probe["ginstr_per_s"]
    fl = flops_step - (PM.flops(per_class["qr"], sys_.K) if args.reuse_qr else 0)
    value = fl / (ms_step * 1e-3) * 1e-9
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded, synth.py; 'near' start series)",
        "config": {"workload": "C4: dim=1024 2-column banded (w=32) monomial system, degree 31, quad double, "
                               "eval/diff sharded by equations + all-gather row replication, solve replicated",
                   "ranges": ranges, "reuse_qr": bool(args.reuse_qr),
                   "l2": "flushed (256 MiB memset) before every timed step"},
        "pct_of_peak": 100.0 * value / (ws * peak),
        "roofline": {"bound": "alu", "achieved": value, "peak": peak, "unit": "GFLOP/s", "frac": value / peak,
                     "traffic": None, "peak_source": "measured DFMA-chain probe x2"},
        "clocks": clk,
    }
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import numpy as np
    import torch

    import paper_2301_12659_b200 as P
    import synth
    from paper_2301_12659_b200 import perfmodel as PM

    ws, rank, local = dist_env()
    if args.gpus > 1 and ws == 1:
        raise SystemExit("--gpus N > 1 must be launched with torchrun (one process per GPU)")
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))

    sys_ = synth.build_config(args.config)
    x_np = synth.make_x(sys_, "near", seed=1)
    h = P.NewtonSystem.from_system(sys_, device=local)
    dev = torch.device(f"cuda:{local}")
    x0 = torch.tensor(x_np, device=dev)
    x = x0.clone()
    res = torch.zeros((sys_.K, 3), dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream()
    c, per_class, total = work(sys_, h.nnz)
    flops_step = PM.flops(total, sys_.K)

    # warm-up
    for _ in range(max(args.warmup, 3)):
        x.copy_(x0)
        h.step(x, res)
    torch.cuda.synchronize()
    h.reset_ledger()

    # timed region: each step bracketed by events on the launching stream,
    # L2 flushed (256 MiB memset) before every step, outside the events
    clocks = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[0])
                          if os.environ.get("CUDA_VISIBLE_DEVICES", "").isdigit() else local)
    clocks.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches = 0
    for i in range(args.steps):
        x.copy_(x0)
        flush.zero_()
        ev[i][0].record(stream)
        h.step(x, res, flags=P.NS_LEDGER)
        ev[i][1].record(stream)
        launches += h.last_launch_count()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms_steps = [a.elapsed_time(b) for a, b in ev]
    ms_total = sum(ms_steps)
    led = h.ledger()
    # e2e through the public API with host buffers: pinned H2D of x, step, D2H of x and the residual
    xh = torch.tensor(x_np).pin_memory()
    xo = torch.empty_like(xh).pin_memory()
    rh = torch.empty((sys_.K, 3), dtype=torch.float64).pin_memory()
    ee = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        flush.zero_()
        ee[i][0].record(stream)
        x.copy_(xh, non_blocking=True)
        h.step(x, res)
        xo.copy_(x, non_blocking=True)
        rh.copy_(res, non_blocking=True)
        ee[i][1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    e2e_ms = sum(a.elapsed_time(b) for a, b in ee)

    if dist:
        t = torch.tensor([ms_total, e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total, e2e_ms = float(t[0]), float(t[1])
    n_gpus = ws
    ms_step = ms_total / args.steps
    value = n_gpus * flops_step / (ms_step * 1e-3) * 1e-9
    e2e_value = n_gpus * flops_step / (e2e_ms / args.steps * 1e-3) * 1e-9

    # roofline of the dominant kernel class (ledger events on the launching stream)
    cls_ms = {"convolution": led["ms_convolution"], "qr": led["ms_qr"], "stage": led["ms_stage"],
              "residual": led["ms_residual"]}
    dom = max(cls_ms, key=cls_ms.get)
    dom_ms = cls_ms[dom] / max(1, led["steps"])
    dom_gflops = PM.flops(per_class[dom], sys_.K) / (dom_ms * 1e-3) * 1e-9
    peaks = PM.fp64_peak_gflops(torch.cuda.get_device_properties(dev).multi_processor_count, 1965.0)
    probe = P.fp64_peak_probe(local, "dfma")
    measured_peak_gflops = 2.0 * probe["ginstr_per_s"]
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"{args.config}:{dom}")
        except Exception:
            traffic = None
    roofline = {
        "bound": "alu", "kernel_class": dom, "achieved": dom_gflops, "peak": measured_peak_gflops,
        "unit": "GFLOP/s", "frac": dom_gflops / measured_peak_gflops, "traffic": traffic,
        "peak_source": "measured DFMA-chain probe (ns_fp64_peak_probe), x2 flops per DFMA",
        "peak_derived_gflops": peaks["gflops"],
        "fp64_pipe_frac": PM.instr(per_class[dom], sys_.K) / (dom_ms * 1e-3) * 1e-9 / probe["ginstr_per_s"],
        "class_ms_per_step": {k: v / max(1, led["steps"]) for k, v in cls_ms.items()},
        "ledger_step_ms": led["ms_total"] / max(1, led["steps"]),
        "note": "eval/diff runs on a side stream concurrently with A0 + QR; class times overlap",
    }
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, synth.py; 'near' start series)",
        "config": {"workload": workload_desc(args.config, sys_), "dim": sys_.n, "degree": sys_.D,
                   "precision": {2: "2d", 4: "4d", 8: "8d"}[sys_.K],
                   "parallelism": f"replicas x{n_gpus}" if n_gpus > 1 else "1 GPU",
                   "l2": "flushed (256 MiB memset) before every timed step"},
        "pct_of_peak": 100.0 * value / (n_gpus * measured_peak_gflops),
        "md_fma_per_step": total, "fp64_flops_per_step": flops_step,
        "paper_equivalent_gflops": n_gpus * PM.T2_MUL[sys_.K] * total / (ms_step * 1e-3) * 1e-9,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": xh.numel() * 8,
                "d2h_bytes_per_step": (xo.numel() + rh.numel()) * 8, "ms_per_step": e2e_ms / args.steps},
        "roofline": roofline,
        "gpu_launches": launches,
        "clocks": clk,
    }
    if rank == 0 and n_gpus == 1 and not args.no_cpu_baseline:
        dt, frac, desc = oracle_sample(sys_, x_np, args.cpu_budget)
        cpu_ms = dt / frac * 1e3
        out["cpu_baseline"] = {"value": flops_step / (cpu_ms * 1e-3) * 1e-9, "unit": UNIT, "cores": 1,
                               "kind": "oracle", "sample": desc, "ms_per_step": cpu_ms}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


def run_driver(args):
    """NEXT-1: one 'step' = one whole staggered Newton run
    (ns_run_newton) from the 'start' series (x_0 correct to half
    precision) until every stage is retired, against the same run
    with all orders in every iteration (NS_NO_STAGGER).  Device time from
    CUDA events around each run (the driver synchronises once per iteration
    to read the norms; that host time is inside the events)."""
    import torch

    import paper_2301_12659_b200 as P
    import synth

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    sys_ = synth.build_config(args.config)
    h = P.NewtonSystem.from_system(sys_, device=local)
    xs = torch.tensor(synth.make_x(sys_, "start", seed=1), device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {}
    clocks = ClockSampler(local)
    for name, fl in (("staggered", 0), ("staggered_qr_once", P.NS_QR_ONCE), ("full_orders", P.NS_NO_STAGGER)):
        for _ in range(max(1, args.warmup)):
            x = xs.clone()
            h.run_newton(x, max_iter=24, flags=fl)
        if name == "staggered":
            clocks.start()
        times, info, log = [], None, None
        for _ in range(args.steps):
            x = xs.clone()
            flush.zero_()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            info, log = h.run_newton(x, max_iter=24, flags=fl)
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        if name == "staggered":
            clk = clocks.stop()
        times.sort()
        out[name] = {"ms_median": times[len(times) // 2], "ms_min": times[0], "iterations": info["iterations"],
                     "converged": info["converged"], "qr_count": info["qr_count"],
                     "log": [{k: (round(v, 4) if isinstance(v, float) else v) for k, v in e.items()} for e in log]}
    line = {"metric": "staggered Newton run ms (ns_run_newton, 'start' to convergence)",
            "value": out["staggered"]["ms_median"], "unit": "ms", "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": False, "dtype": "f64", "data": "synthetic (seeded, synth.py)",
            "config": {"workload": workload_desc(args.config, sys_).replace("one Newton step", "staggered run"),
                       "l2": "flushed (256 MiB memset) before every timed run"},
            "runs": out, "clocks": clk}
    if rank == 0:
        print(json.dumps(line))


def main():
    args = parse()
    if args.driver and args.impl == "ours":
        run_driver(args)
        return
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "C5":
        run_c5(args)
    elif args.config == "C4":
        run_c4(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
