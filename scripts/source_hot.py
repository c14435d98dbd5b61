"""Top source lines of an `ncu --page source --csv` dump (stdin) by warp-stall
samples: the per-line cost map of a kernel compiled with -lineinfo.
usage: ncu -i rep --page source --csv | python scripts/source_hot.py [N]"""
import csv
import io
import sys

N = int(sys.argv[1]) if len(sys.argv) > 1 else 40
text = sys.stdin.read()
lines = text.splitlines()
start = next((i for i, l in enumerate(lines) if "Source" in l and "," in l), None)
if start is None:
    print("no source table")
    sys.exit(0)
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]
key = next((h for h in hdr if "Warp Stall Sampling (All" in h), None) or \
    next((h for h in hdr if "Sampling" in h), None)
src = hdr.index("Source") if "Source" in hdr else 1
ki = hdr.index(key) if key else None
data = []
for r in rows[1:]:
    if ki is None or len(r) <= max(ki, src):
        continue
    try:
        v = float(r[ki].replace(",", "") or 0)
    except ValueError:
        continue
    data.append((v, r[0], r[src][:140]))
tot = sum(v for v, _, _ in data) or 1.0
print(f"columns: {hdr[:12]}\nkey: {key}; total samples {tot:.0f}")
for v, a, t in sorted(data, reverse=True)[:N]:
    print(f"{100 * v / tot:6.2f}%  {a:>8}  {t}")
