#!/usr/bin/env python
"""bench.py -- the Newton step on truncated power series (arxiv 2301.12659) on B200.

Headline workload (N = 1, no flags): BASELINE.json configs[2] (C3), the
largest single-GPU config and the paper's own precision: dim 128 one-column
lower-triangular monomial system (Eq.(5)), degree 63, octo double,
one full Newton step (eval/diff + Householder QR of A0 + staged updates /
Q^T b / back substitution + residual + x += dx) through the C ABI.

One "step" = one ns_newton_series_step on one system.  value = FP64 GFLOP/s
of the whole job: algorithmic md multiply-adds of the step (SURVEY 8(d) d.4,
perfmodel.algorithmic_counts) x the FP64 flops of one md multiply-add of
md.cuh (FMA = 2; perfmodel.MD_FMA_MIX, cross-checked against ncu dadd/dmul/dfma
counts in profiles/) / device time.

N > 1 (torchrun, one process per GPU): one C3 system does not shard (the
stage loop is sequential in k), so the headline is
N independent C3 replicas (weak scaling).  The workloads that DO shard ride
on the same line at every N (also N = 1, the scaling anchor):
  "c5": 4096 independent paths (configs[4]) partitioned over the ranks, no
        collective in the step (strong scaling: the batch is fixed);
  "c4": the dim 1024 system (configs[3]) with its eval/diff sharded by
        equations over the ranks and the rows replicated over NVLink, the
        solve replicated (strong scaling).
"c2" (configs[1], 4d) is also reported.  --impl reference times the CPU
oracle (this tier's reference arm) on a bounded sample on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os

# single-threaded BLAS (the oracle's pools + OpenBLAS threads deadlocked a test process)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Newton step ms and FP64 GFLOPS (% of peak) per 2d/4d/8d at 1/2/4/8 B200"
UNIT = "GFLOP/s (FP64, FMA=2: algorithmic md multiply-adds x FP64 flops per md multiply-add)"
PREC = {2: "2d", 4: "4d", 8: "8d"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C3", choices=["C1", "C2", "C3", "C4", "C5"],
                   help="headline workload (default C3); C4/C5 make the sharded workload the headline")
    p.add_argument("--precision", type=int, default=0, choices=[0, 2, 4, 8],
                   help="run the workload at another precision (SURVEY d.2 'precision-swapped')")
    p.add_argument("--reuse-qr", action="store_true", help="C4: NS_REUSE_QR in the timed steps (QR once)")
    p.add_argument("--batch", type=int, default=4096, help="C5: total paths (partitioned over ranks)")
    p.add_argument("--no-extras", action="store_true", help="skip the c2/c4/c5 keys")
    p.add_argument("--driver", action="store_true",
                   help="NEXT-1: time whole staggered Newton runs (ns_run_newton) from 'start' to convergence")
    p.add_argument("--sweep", action="store_true", help="NEXT-3: T6-style eval/diff order sweep (dim 1024, 8d)")
    p.add_argument("--sweep-dim", type=int, default=1024)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-budget", type=float, default=12.0, help="seconds per oracle sample (1 and N processes)")
    return p.parse_args()


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def workload_desc(name, sys_):
    prec = {2: "double double", 4: "quad double", 8: "octo double"}[sys_.K]
    if name.startswith("C4"):
        return (f"{name}: dim={sys_.n} 2-column banded (w={sys_.meta.get('w')}) monomial system (Eq.(8)-(9)), "
                f"degree {sys_.D}, {prec}, one Newton step")
    return (f"{name}: dim={sys_.n} one-column lower-triangular monomial system (Eq.(5)), "
            f"degree {sys_.D}, {prec}, one Newton step")


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi sampled every 100 ms during the timed region (B200_PROFILING.md clocks line)."""

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


def smi_index(local):
    cvd = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    ids = [c for c in cvd.split(",") if c.strip()]
    return int(ids[local]) if local < len(ids) and ids[local].isdigit() else local


# ------------------------------------------------------------------ work model
def counts_for(sys_, nnz):
    from paper_2301_12659_b200 import perfmodel as PM
    return PM.algorithmic_counts(sys_.eq_ptr, sys_.mono_ptr, nnz, sys_.n, sys_.d)


def fp64_peak(local):
    """Measured FP64 rate (DFMA chains on every SM, ns_fp64_peak_probe) and the
    derived figure (148 SMs x 64 FP64 lanes x 2 x sm_max_mhz)."""
    import torch

    import paper_2301_12659_b200 as P
    from paper_2301_12659_b200 import perfmodel as PM
    probe = P.fp64_peak_probe(local, "dfma")
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    mhz = 1965.0
    try:
        mhz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"])
    except Exception:
        pass
    der = PM.fp64_peak_gflops(sms, mhz)
    return {"gflops": 2.0 * probe["ginstr_per_s"], "ginstr": probe["ginstr_per_s"], "derived_gflops": der["gflops"],
            "source": f"measured: ns_fp64_peak_probe DFMA chains on all SMs x 2 flops (derived {der['gflops']:.0f} "
                      f"= {sms} SMs x 64 FP64 lanes x 2 x {mhz:.0f} MHz; MEASURED_PEAKS.json has no FP64 entry)"}


def class_roofline(counts, cls_ms, K, peak):
    """Per kernel class: algorithmic md multiply-adds, achieved FP64 GFLOP/s,
    fraction of the FP64 peak and of the FP64 pipe (instructions)."""
    from paper_2301_12659_b200 import perfmodel as PM
    out = {}
    for c, ms in cls_ms.items():
        if ms is None or ms <= 0:
            continue
        f = PM.flops(counts[c], K)
        g = f / (ms * 1e-3) * 1e-9
        out[c] = {"ms": ms, "md_fma": counts[c], "achieved": g, "frac": g / peak["gflops"],
                  "fp64_pipe_frac": PM.instr(counts[c], K) / (ms * 1e-3) * 1e-9 / peak["ginstr"]}
    return out


def traffic_of(key):
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(tf)).get(key)
    except Exception:
        return None


# ------------------------------------------------------------------ CPU oracle (bounded sample)
def _oracle_rows(args):
    sys_, x_np, rows = args
    from oracle import newton as O
    F = O.field_for(sys_.K)
    xs = O.read_x(x_np, F)   # input conversion, not timed
    t0 = time.perf_counter()
    O.evaluate(sys_, xs, F, split=True, rows=rows)
    return time.perf_counter() - t0


def oracle_sample(sys_, x_np, budget_s: float, procs: int = 1, rotate: int = 0):
    """Time the oracle (O-hp tier, as it stands) on a bounded sample of one
    step: eval/diff of a subset of the equations (over `procs` worker
    processes) plus the block solve of the first stages (one process; the
    stage recursion is sequential).  Work is counted in oracle multiply-adds:
    row i with m variables = (m-1) + (3m-2) convolutions of d(d+1)/2 terms;
    solve = n^3/3 (LU) + sum_k (k nnz + n^2).  Returns (seconds extrapolated
    to the whole step by that count, fraction sampled, description)."""
    import copy
    import multiprocessing as mp

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
    ed_full = sum(rows_cost)
    solve_full = n ** 3 // 3 + sum(stage_cost)
    rate = 6e-6  # seconds per multiply-add (mpmath, pure Python) -- only sizes the sample
    # eval/diff sample: every stride-th row, sized to ~budget/2 per process
    target_rows = max(1.0, 0.5 * budget_s / rate * procs)
    stride = max(1, int(round(ed_full / target_rows)))
    rows = list(range((stride // 2 + rotate) % stride, n, stride))
    # solve sample: stages 0..ks-1 (with the truncated eval/diff they need), ~budget/2
    ks, acc = 1, stage_cost[0]
    sub_cost = lambda k: sum(c // tri * (k * (k + 1) // 2) for c in rows_cost)
    while ks < d and (n ** 3 // 3 + acc + stage_cost[ks] + sub_cost(ks + 1)) * rate < 0.5 * budget_s:
        acc += stage_cost[ks]
        ks += 1
    if procs > 1 and len(rows) > 1:
        # rows dealt to the processes by decreasing cost (LPT); the wall time of the slowest counts
        order = sorted(rows, key=lambda i: -rows_cost[i])
        chunks = [order[p::procs] for p in range(procs) if order[p::procs]]
        with mp.get_context("forkserver").Pool(len(chunks)) as pool:
            t_ed = max(pool.map(_oracle_rows, [(sys_, x_np, c) for c in chunks]))
    else:
        t_ed = _oracle_rows((sys_, x_np, rows))
    sub = copy.copy(sys_)
    sub.D = ks - 1
    sub.rhs = sys_.rhs[:, :, :ks]
    t1 = time.perf_counter()
    xs_k = [ser[:ks] for ser in O.read_x(x_np, F)]
    b_k, A_k = O.evaluate(sub, xs_k, F, split=True)
    O.solve(A_k, b_k, n, ks, F)
    t_solve = time.perf_counter() - t1
    ed_done = sum(rows_cost[i] for i in rows)
    solve_done = n ** 3 // 3 + acc + sub_cost(ks)
    # extrapolate each part by its own count (the parts run at different rates)
    secs = t_ed * ed_full / ed_done + t_solve * (solve_full + 0.0) / solve_done
    frac = (ed_done + solve_done) / (ed_full + solve_full)
    desc = (f"oracle (mpmath {F.name}) eval/diff of {len(rows)}/{n} equations on {procs} process(es) "
            f"({t_ed:.1f} s) + block solve of stages 0..{ks - 1} with their truncated eval/diff on 1 process "
            f"({t_solve:.1f} s); each part extrapolated to the whole step by its oracle multiply-add count")
    return secs, frac, desc


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(sys_, x_np, flops_step, budget):
    cores = host_cores()
    s1, f1, d1 = oracle_sample(sys_, x_np, budget, procs=1)
    sN, fN, dN = oracle_sample(sys_, x_np, budget, procs=cores, rotate=1)
    g = lambda s: flops_step / s * 1e-9
    return {"value": g(sN), "unit": UNIT, "cores": cores, "kind": "oracle", "sample": dN,
            "ms_per_step": sN * 1e3, "one_process": {"value": g(s1), "cores": 1, "ms_per_step": s1 * 1e3,
                                                       "sample": d1},
            "host_cores": cores}


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    ws, rank, local = dist_env()
    if ws > 1 and rank != 0:
        return
    import synth
    from oracle import newton as O
    from paper_2301_12659_b200 import perfmodel as PM
    sys_ = synth.build_config(args.config, K=args.precision or None)
    x_np = synth.make_x(sys_, "near", seed=1)
    nnz = sum(len(r) for r in O.jacobian_pattern(sys_))
    counts = counts_for(sys_, nnz)
    flops = PM.flops(counts["total"], sys_.K)
    cores = host_cores()
    budget = max(2.0, 120.0 / max(1, args.steps + args.warmup))
    for w in range(args.warmup):
        oracle_sample(sys_, x_np, budget, procs=cores, rotate=w)
    per_step, desc = [], None
    for s in range(args.steps):
        secs, frac, desc = oracle_sample(sys_, x_np, budget, procs=cores, rotate=args.warmup + s)
        per_step.append(secs)
    ms = 1e3 * sum(per_step) / len(per_step)
    value = flops / (ms * 1e-3) * 1e-9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, synth.py; 'near' series)",
        "config": {"workload": workload_desc(args.config, sys_)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ one system per rank
def bench_single(sys_, args, local, dev, flush, ledger=True):
    """Timed steps of one system (device time, CUDA events on the launching
    stream, L2 flushed before every step), the ledger's class times, and the
    e2e steps with pinned host buffers."""
    import torch

    import paper_2301_12659_b200 as P
    import synth
    x_np = synth.make_x(sys_, "near", seed=1)
    h = P.NewtonSystem.from_system(sys_, device=local)
    x0 = torch.tensor(x_np, device=dev)
    x = x0.clone()
    res = torch.zeros((sys_.K, 3), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(max(args.warmup, 3)):
        x.copy_(x0)
        h.step(x, res)
    torch.cuda.synchronize()
    h.reset_ledger()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches = 0
    for i in range(args.steps):
        x.copy_(x0)
        flush.zero_()
        ev[i][0].record(stream)
        h.step(x, res, flags=P.NS_LEDGER if ledger else 0)
        ev[i][1].record(stream)
        launches += h.last_launch_count()
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in ev]
    led = h.ledger()
    # e2e through the public API with host buffers: pinned H2D of x, the step,
    # D2H of the new x and the residual norms, every step
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
    e2e = [a.elapsed_time(b) for a, b in ee]
    nst = max(1, led["steps"])
    cls = {"evaldiff": led["ms_convolution"] / nst, "qr": led["ms_qr"] / nst, "stage": led["ms_stage"] / nst,
           "residual": led["ms_residual"] / nst}
    return {"h": h, "x_np": x_np, "ms": ms, "e2e_ms": e2e, "cls": cls, "ledger_step_ms": led["ms_total"] / nst,
            "launches": launches, "h2d": xh.numel() * 8, "d2h": (xo.numel() + rh.numel()) * 8}


def max_ranks(v, dev):
    from paper_2301_12659_b200.dist import max_over_ranks
    return max_over_ranks(v, dev)


def extra_c2(args, local, dev, flush, peak):
    import synth
    from paper_2301_12659_b200 import perfmodel as PM
    sys_ = synth.build_config("C2")
    r = bench_single(sys_, args, local, dev, flush)
    counts = counts_for(sys_, r["h"].nnz)
    ms = max_ranks(sum(r["ms"]) / len(r["ms"]), dev)
    g = PM.flops(counts["total"], 4) / (ms * 1e-3) * 1e-9
    return {"workload": workload_desc("C2", sys_), "ms_per_step": ms, "gflops_per_gpu": g,
            "pct_of_peak": 100 * g / peak["gflops"], "classes": class_roofline(counts, r["cls"], 4, peak)}


def _c5_path(args):
    p, K = args
    import synth
    sys_ = synth.triangular_system(32, 15, K, seed=12665 + p, name="C5")
    return synth.make_x(sys_, "near", seed=100 + p), sys_.rhs


def extra_c5(args, local, dev, flush, peak, K=2, batch=4096):
    """configs[4]: `batch` paths partitioned over the ranks, one
    ns_newton_series_step_batched per rank per step, no collective."""
    import multiprocessing as mp

    import numpy as np
    import torch

    import paper_2301_12659_b200 as P
    import synth
    from paper_2301_12659_b200 import perfmodel as PM
    from paper_2301_12659_b200.dist import partition
    ws, rank, _ = dist_env()
    lo, hi = partition(batch, ws, rank)
    with mp.get_context("forkserver").Pool(min(16, host_cores())) as pool:
        data = pool.map(_c5_path, [(p, K) for p in range(lo, hi)], chunksize=16)
    base = synth.triangular_system(32, 15, K, seed=12665, name="C5")
    X0 = torch.tensor(np.stack([d[0] for d in data]), device=dev)
    R = torch.tensor(np.stack([d[1] for d in data]), device=dev)
    X = X0.clone()
    B = hi - lo
    res = torch.zeros((B, K, 3), dtype=torch.float64, device=dev)
    h = P.NewtonSystem.from_system(base, max_batch=max(1, B), device=local)
    counts = counts_for(base, h.nnz)
    stream = torch.cuda.current_stream()
    for _ in range(max(args.warmup, 3)):
        X.copy_(X0)
        h.step_batched(X, R, res)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(args.steps):
        X.copy_(X0)
        flush.zero_()
        ev[i][0].record(stream)
        h.step_batched(X, R, res)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    ms = max_ranks(sum(a.elapsed_time(b) for a, b in ev) / args.steps, dev)
    g = batch * PM.flops(counts["total"], K) / (ms * 1e-3) * 1e-9
    return {"workload": f"C5: batch of {batch} independent paths, dim=32, degree 15, {PREC[K]}, paths "
                        f"partitioned over {ws} GPU(s), no collective in the step",
            "ms_per_step": ms, "paths_per_s": batch / (ms * 1e-3), "gflops": g,
            "pct_of_peak": 100 * g / (ws * peak["gflops"]), "scaling": "strong", "launches_per_step": 1}


def extra_c4(args, local, dev, flush, peak, K=4, reuse=False):
    """configs[3]: eval/diff sharded by equations (equation-owner, no
    arithmetic reduction), rows replicated over NVLink, solve replicated."""
    import torch

    import paper_2301_12659_b200 as P
    import synth
    from paper_2301_12659_b200 import perfmodel as PM
    ws, rank, _ = dist_env()
    sys_ = synth.build_config("C4", K=K)
    x_np = synth.make_x(sys_, "near", seed=1)
    h = P.NewtonSystem.from_system(sys_, device=local)
    if ws > 1:
        # the library owns the communicator: rank 0's NCCL id goes to every rank
        # (torch.distributed is the bootstrap only); from then on the step
        # shards eval/diff and replicates the rows inside the library
        import torch.distributed as tdist
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(P.nccl_unique_id()), dtype=torch.uint8))
        tdist.broadcast(uid, src=0)
        h.comm_init(ws, rank, bytes(uid.cpu().numpy().tobytes()))
    bounds, _ = P.exchange_plan(sys_.eq_ptr, sys_.mono_ptr, sys_.var_idx, sys_.n,
                                                                    sys_.D, sys_.K, ws)
    ranges = [(int(bounds[r]), int(bounds[r + 1])) for r in range(ws)]
    x0 = torch.tensor(x_np, device=dev)
    x = x0.clone()
    res = torch.zeros((K, 3), dtype=torch.float64, device=dev)
    counts = counts_for(sys_, h.nnz)
    stream = torch.cuda.current_stream()

    def one(flags):
        h.step(x, res, flags=flags)

    for _ in range(max(args.warmup, 2)):
        x.copy_(x0)
        one(0)
    torch.cuda.synchronize()
    steps = max(3, args.steps // 2)

    def timed(flags):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for i in range(steps):
            x.copy_(x0)
            flush.zero_()
            ev[i][0].record(stream)
            one(flags)
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        return max_ranks(sum(a.elapsed_time(b) for a, b in ev) / steps, dev)

    ms = timed(P.NS_REUSE_QR if reuse else 0)
    tot = counts["total"] - (counts["qr"] if reuse else 0)
    g = PM.flops(tot, K) / (ms * 1e-3) * 1e-9
    out = {"workload": workload_desc("C4", sys_) + f"; eval/diff sharded by equations over {ws} GPU(s), rows "
                       "replicated by the library's grouped ncclBroadcast, solve replicated",
           "ranges": ranges, "reuse_qr": reuse, "ms_per_step": ms, "gflops": g,
           "pct_of_peak": 100 * g / (ws * peak["gflops"]), "scaling": "strong"}
    if not reuse:
        # the paper's "QR only once" (what ns_run_newton does after stage 0
        # retires): the step without the replicated QR, where the sharding shows
        ms_r = timed(P.NS_REUSE_QR)
        out["reuse_qr_step"] = {"ms_per_step": ms_r,
                                "gflops": PM.flops(counts["total"] - counts["qr"], K) / (ms_r * 1e-3) * 1e-9}
    return out


def run_ours(args):
    import torch

    import synth
    from paper_2301_12659_b200 import perfmodel as PM

    ws, rank, local = dist_env()
    if args.gpus > 1 and ws == 1:
        raise SystemExit("--gpus N > 1 must be launched with torchrun (one process per GPU)")
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    peak = fp64_peak(local)
    name = args.config
    sys_ = synth.build_config(name, K=args.precision or None)
    clocks = ClockSampler(smi_index(local))
    clocks.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    r = bench_single(sys_, args, local, dev, flush)
    ms_total = max_ranks(sum(r["ms"]), dev)
    e2e_total = max_ranks(sum(r["e2e_ms"]), dev)
    clk = clocks.stop()
    K = sys_.K
    counts = counts_for(sys_, r["h"].nnz)
    flops_step = PM.flops(counts["total"], K)
    ms_step = ms_total / args.steps
    value = ws * flops_step / (ms_step * 1e-3) * 1e-9
    e2e_value = ws * flops_step / (e2e_total / args.steps * 1e-3) * 1e-9
    classes = class_roofline(counts, r["cls"], K, peak)
    dom = max(classes, key=lambda c: classes[c]["ms"])
    roofline = {
        "bound": "alu", "kernel_class": dom, "achieved": classes[dom]["achieved"], "peak": peak["gflops"],
        "unit": "GFLOP/s", "frac": classes[dom]["frac"], "traffic": traffic_of(f"{name}:{dom}"),
        "peak_source": peak["source"], "peak_derived_gflops": peak["derived_gflops"],
        "fp64_pipe_frac": classes[dom]["fp64_pipe_frac"], "classes": classes,
        "numerator": "SURVEY 8(d) d.4 algorithmic md multiply-adds (triangular convolutions, QR (2/3)n^3, "
                     "updates nnz d(d-1)/2 + Q^T b 2n^2 d + back substitution n^2 d/2, residual nnz d) x "
                     f"{PM.mix_flops(PM.MD_FMA_MIX[K])} FP64 flops per {PREC[K]} md multiply-add (md.cuh static "
                     "count; ncu dadd/dmul/dfma cross-check in profiles/)",
        "ledger_step_ms": r["ledger_step_ms"],
        "note": "class times from CUDA events on the launching streams (NS_LEDGER); eval/diff runs on a side "
                "stream concurrently with A0 + QR, so those two overlap",
    }
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, synth.py; 'near' series)",
        "config": {"workload": workload_desc(name, sys_), "dim": sys_.n, "degree": sys_.D, "precision": PREC[K],
                   "parallelism": (f"replicas x{ws} (one system per GPU: the step of one system does not shard, "
                                   "DESIGN.md 7)") if ws > 1 else "1 GPU",
                   "l2": "flushed (256 MiB memset) before every timed step"},
        "pct_of_peak": 100.0 * value / (ws * peak["gflops"]),
        "ms_min": min(r["ms"]), "ms_median": sorted(r["ms"])[len(r["ms"]) // 2],
        "md_fma_per_step": counts["total"], "md_fma_by_class": {c: counts[c] for c in ("evaldiff", "qr", "stage",
                                                                                        "residual")},
        "fp64_flops_per_step": flops_step,
        "paper_equivalent_gflops": ws * PM.T2_MUL[K] * counts["total"] / (ms_step * 1e-3) * 1e-9,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": r["h2d"] * ws,
                "d2h_bytes_per_step": r["d2h"] * ws, "ms_per_step": e2e_total / args.steps},
        "roofline": roofline,
        "gpu_launches": r["launches"],
        "clocks": clk,
    }
    if not args.no_extras:
        # the extra workloads must not cost the headline line: an exception is
        # recorded in its key (the ranks keep the same collective sequence: every
        # rank runs the same extras in the same order)
        def guarded(fn, *a, **kw):
            try:
                return fn(*a, **kw)
            except Exception as e:  # noqa: BLE001
                return {"error": f"{type(e).__name__}: {e}"[:300]}
        if name != "C2":
            out["c2"] = guarded(extra_c2, args, local, dev, flush, peak)
        out["c5"] = guarded(extra_c5, args, local, dev, flush, peak)
        out["c4"] = guarded(extra_c4, args, local, dev, flush, peak)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(sys_, r["x_np"], flops_step, args.cpu_budget)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


def run_sharded_headline(args):
    """--config C4 / C5: the sharded workload as the headline line."""
    import torch

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    peak = fp64_peak(local)
    clocks = ClockSampler(smi_index(local))
    clocks.start()
    time.sleep(0.3)
    if args.config == "C5":
        r = extra_c5(args, local, dev, flush, peak, K=args.precision or 2, batch=args.batch)
    else:
        r = extra_c4(args, local, dev, flush, peak, K=args.precision or 4, reuse=args.reuse_qr)
    clk = clocks.stop()
    out = {"metric": METRIC, "value": r["gflops"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": r["ms_per_step"], "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, synth.py)",
           "config": {"workload": r["workload"], "l2": "flushed (256 MiB memset) before every timed step"},
           "pct_of_peak": r["pct_of_peak"], "detail": r, "clocks": clk}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if dist:
        dist.destroy_process_group()


def run_driver(args):
    """NEXT-1: one 'step' = one whole staggered Newton run
    (ns_run_newton) from the 'start' series (x_0 correct to half
    precision) until every stage is retired, against the same run
    with all orders in every iteration (NS_NO_STAGGER)."""
    import torch

    import paper_2301_12659_b200 as P
    import synth

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    sys_ = synth.build_config(args.config, K=args.precision or None)
    h = P.NewtonSystem.from_system(sys_, device=local)
    xs = torch.tensor(synth.make_x(sys_, "start", seed=1), device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = {}
    clocks = ClockSampler(smi_index(local))
    clk = None
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


def run_sweep(args):
    """NEXT-3 order sweep in the style of T6: the paper's shape
    (one-column system of Eq.(5), dim 1024, octo double) evaluated and
    differentiated at the orders 1, 2, 3, 5, 8, 12, 18, 27, 41, 62, 64 (the
    window [0, dc) of ns_set_window truncates every convolution at t^dc,
    P:495-497); device time of ns_eval_diff per order.  FP64 GFLOPS = the
    algorithmic md multiply-adds of the truncated convolutions (triangular,
    S dc(dc+1)/2 + scalings) x FP64 flops per md multiply-add; the paper's
    own counting (md multiplications x 1742, padded dc^2 products, T2/P:574)
    beside it as context."""
    import ctypes

    import torch

    import paper_2301_12659_b200 as P
    import synth
    from paper_2301_12659_b200 import perfmodel as PM
    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    n = args.sweep_dim
    K = args.precision or 8
    sys_ = synth.triangular_system(n, 63, K, seed=12667, name="T6")
    x = torch.tensor(synth.make_x(sys_, "near", seed=1), device=dev)
    h = P.NewtonSystem.from_system(sys_, device=local)
    M = sys_.M
    ms_ = [int(sys_.mono_ptr[t + 1] - sys_.mono_ptr[t]) for t in range(M)]
    S = sum(PM.products(m) for m in ms_)
    L = P.lib()
    stream = torch.cuda.current_stream()
    clocks = ClockSampler(smi_index(local))
    clocks.start()
    rows = []
    for dc in (1, 2, 3, 5, 8, 12, 18, 27, 41, 62, 64):
        h.set_window(0, dc)
        for _ in range(2):
            L.ns_eval_diff(h._h, ctypes.c_void_p(x.data_ptr()), None, None, None, ctypes.c_void_p(stream.cuda_stream))
        reps = 3
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            L.ns_eval_diff(h._h, ctypes.c_void_p(x.data_ptr()), None, None, None, ctypes.c_void_p(stream.cuda_stream))
        b.record(stream)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        md_fma = S * dc * (dc + 1) // 2 + (M + sum(ms_)) * dc
        g = PM.flops(md_fma, K) / (ms * 1e-3) * 1e-9
        paper = S * dc * dc * PM.T2_MUL[K] / (ms * 1e-3) * 1e-9
        rows.append({"order": dc, "ms": ms, "gflops": g, "paper_convention_gflops": paper})
    h.set_window(0, sys_.d)
    clk = clocks.stop()
    line = {"metric": "eval/diff ms and FP64 GFLOPS per order (T6 sweep)", "value": rows[-1]["gflops"],
            "unit": "GFLOP/s (FP64, FMA=2)", "n_gpus": 1, "higher_is_better": True, "dtype": "f64",
            "data": "synthetic (seeded, synth.py; 'near' series)",
            "config": {"workload": f"T6 shape: dim={n} one-column system (Eq.(5)), {PREC[K]}, eval/diff at orders "
                                   "1..64 (ns_set_window)", "series_products": S},
            "orders": rows, "clocks": clk,
            "paper_T6_context": "V100 1658.4, A100 2568.0, P100 554.7 GFLOPS at order 64, 8d, dim 1024 (paper's "
                                "convention: md-mul x 1742, padded products)"}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.sweep:
        run_sweep(args)
        return
    if args.impl == "reference":
        run_reference(args)
    elif args.driver:
        run_driver(args)
    elif args.config in ("C4", "C5"):
        run_sharded_headline(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
