"""Summarise an `ncu --metrics ... --csv --log-file X.csv` launch list: per
kernel launch the metric values, plus FP64 flops (dadd + dmul + 2 dfma) and the
FP64 instructions.  usage: python scripts/ncu_metrics.py X.csv [--json out.json]"""
import csv
import io
import json
import sys


def load(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    launches = {}
    for r in rows:
        key = int(r["ID"])
        d = launches.setdefault(key, {"id": key, "kernel": r["Kernel Name"], "grid": r["Grid Size"],
                                      "block": r["Block Size"]})
        v = r["Metric Value"].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            pass
        d[r["Metric Name"]] = v
    out = []
    for k in sorted(launches):
        d = launches[k]
        g = lambda m: d.get(f"sm__sass_thread_inst_executed_op_{m}_pred_on.sum", 0.0) or 0.0
        if any(f"sm__sass_thread_inst_executed_op_{m}_pred_on.sum" in d for m in ("dadd", "dmul", "dfma")):
            d["fp64_flops"] = g("dadd") + g("dmul") + 2 * g("dfma")
            d["fp64_instr"] = g("dadd") + g("dmul") + g("dfma")
        out.append(d)
    return out


if __name__ == "__main__":
    res = load(sys.argv[1])
    for d in res:
        t = d.get("gpu__time_duration.sum", 0)
        print(f'{d["id"]:4d} {d["kernel"][:48]:48s} t={t/1e3 if t else 0:9.1f}us '
              f'dadd={d.get("sm__sass_thread_inst_executed_op_dadd_pred_on.sum", 0):.3e} '
              f'dmul={d.get("sm__sass_thread_inst_executed_op_dmul_pred_on.sum", 0):.3e} '
              f'dfma={d.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0):.3e} '
              f'pipe={d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "")} '
              f'regs={d.get("launch__registers_per_thread", "")} lmem={d.get("l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum", "")}')
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)
