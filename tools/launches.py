"""Per-kernel mean duration from an ncu --metrics gpu__time_duration.sum --csv log."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = defaultdict(list)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        d[r[ki][:70]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):4d} x {sum(v) / len(v) / 1e3:9.1f} us  {100 * sum(v) / tot:5.1f}%  {k}")
