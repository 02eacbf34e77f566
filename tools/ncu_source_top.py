"""Summarise an ncu --page source --csv --print-source cuda,sass dump: the CUDA
source lines with the most warp-stall samples and their dominant stall reasons."""
import csv
import sys
from collections import defaultdict


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    per_line = defaultdict(lambda: defaultdict(float))
    text = {}
    cur_file = None
    hdr = None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
            continue
        d = dict(zip(hdr, r))
        key = (cur_file, int(r[0]))
        text[key] = r[1][:90]
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k or k in (
                    "Warp Stall Sampling (All Samples)", "Instructions Executed"):
                try:
                    per_line[key][k] += float(v.replace(",", "")) if v else 0.0
                except ValueError:
                    pass
    tot = sum(v["Warp Stall Sampling (All Samples)"] for v in per_line.values()) or 1.0
    items = sorted(per_line.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])
    for key, v in items[:top]:
        s = v["Warp Stall Sampling (All Samples)"]
        stalls = sorted(((x, k[6:]) for k, x in v.items() if k.startswith("stall_")), reverse=True)[:3]
        st = " ".join(f"{k}:{100 * x / max(s, 1):.0f}%" for x, k in stalls if x > 0)
        print(f"{100 * s / tot:5.1f}% {key[0]}:{key[1]:<4d} {text[key]:<90s} {st}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)


def instr(path, top=40):
    """Top source lines by executed warp instructions."""
    rows = list(csv.reader(open(path)))
    per, text, cur, hdr = defaultdict(float), {}, None, None
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
            continue
        d = dict(zip(hdr, r))
        k = (cur, int(r[0]))
        text[k] = r[1][:80]
        try:
            per[k] += float(d["Instructions Executed"].replace(",", "") or 0)
        except ValueError:
            pass
    tot = sum(per.values())
    print("total warp instructions", tot)
    for k, v in sorted(per.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]:<4d} {text[k]}")
