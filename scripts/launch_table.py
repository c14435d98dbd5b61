"""Per-kernel mean device time from an ncu launch-list CSV (gpu__time_duration.sum)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, defaultdict(lambda: [0, 0.0])
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            k = d["Kernel Name"].split("(")[0][:60]
            agg[k][0] += 1
            agg[k][1] += float(d["Metric Value"])
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{c:4d} {t / c / 1e3:10.1f} us/launch  {k}")
