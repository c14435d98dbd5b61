"""Registers / spills / stack per kernel from the nvcc -Xptxas -v logs in
paper_2301_12659_b200/build/*.log.  usage: python scripts/ptxas_table.py [regex]"""
import glob
import re
import subprocess
import sys

pat = re.compile(sys.argv[1]) if len(sys.argv) > 1 else None
for log in sorted(glob.glob("paper_2301_12659_b200/build/*.cu.log")):
    cur = None
    info = {}
    for line in open(log):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
            info[cur] = {}
            continue
        if cur is None:
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            info[cur].update(stack=int(m.group(1)), spill_st=int(m.group(2)), spill_ld=int(m.group(3)))
        m = re.search(r"Used (\d+) registers", line)
        if m:
            info[cur]["regs"] = int(m.group(1))
    names = list(info)
    dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    for mangled, d in zip(names, dem):
        short = d.split("(")[0]
        if pat and not pat.search(short):
            continue
        v = info[mangled]
        print(f"{log.split('/')[-1]:18s} {short[:70]:70s} regs {v.get('regs', '?'):>3} spill {v.get('spill_st', 0):>4}/{v.get('spill_ld', 0):<4} stack {v.get('stack', 0)}")
