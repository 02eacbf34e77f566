#!/usr/bin/env python
"""Print (kernel, metric, unit, value) rows of an `ncu --metrics ... --csv` log (program
output lines before the CSV header are skipped)."""
import csv
import sys


def rows(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    r = list(csv.reader(lines))
    h = r[0]
    for x in r[1:]:
        d = dict(zip(h, x))
        yield d["ID"], d["Kernel Name"], d["Metric Name"], d["Metric Unit"], d["Metric Value"]


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        for i, k, m, u, v in rows(p):
            print(f"  {i:>3s} {k[:34]:34s} {m:60s} {u:8s} {v}")
