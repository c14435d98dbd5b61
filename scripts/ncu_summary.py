"""Summarise .ncu-rep captures (ncu --set full) into a small JSON for profiles/.

usage: python scripts/ncu_summary.py out.json rep1.ncu-rep [rep2 ...]
Keeps per kernel: duration, FP64 pipe utilisation, issue activity, occupancy,
registers, DRAM bytes (read + write = `traffic`), FP64 instruction counts and
the warp-stall breakdown from the details page."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "sm__sass_thread_inst_executed_op_dmul_pred_on.sum", "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
        "l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum"]


def page(rep, name):
    r = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv"], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(r.stdout)))


def summarise(rep):
    rows = page(rep, "raw")
    hdr, units = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        d = {"kernel": v[hdr.index("Kernel Name")][:120]}
        for k in KEYS:
            if k in hdr:
                d[k] = f"{v[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        out.append(d)
    det = page(rep, "details")
    stalls = {}
    for r in det:
        if len(r) > 14 and r[11] in ("Warp State Statistics", "Scheduler Statistics", "Occupancy",
                                     "Compute Workload Analysis"):
            stalls[r[12]] = f"{r[14]} {r[13]}".strip()
        if len(r) > 18 and r[11] == "WarpStateStats" and r[15] == "CPIStall":
            stalls.setdefault("stall_notes", []).append(r[17][:200])
    if out:
        out[0]["details"] = stalls
    return out


if __name__ == "__main__":
    res = {}
    for rep in sys.argv[2:]:
        res[rep.split("/")[-1]] = summarise(rep)
    json.dump(res, open(sys.argv[1], "w"), indent=1)
    print(sys.argv[1])
