#!/usr/bin/env python
"""Write profiles/ncu_traffic.json from one `ncu --set full` capture of the bench's render
kernel: DRAM bytes per launch and the L2 hit rate, stamped with the sha of the kernel
sources (bench.py reports them only while the running kernel has the same sha).

    python tools/ncu_traffic.py tcgen05 gpurun_out/prof_tc.ncu-rep
"""
import csv
import datetime
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(engine, rep):
    import bench
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    d = dict(zip(rows[0], rows[-1]))
    units = dict(zip(rows[0], rows[1]))

    def val(k):
        v = float(d[k].replace(",", ""))
        u = units.get(k, "")
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    out = json.load(open(p)) if os.path.exists(p) else {}
    out["_about"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant "
                     "render kernel from one `ncu --set full` capture of bench.py; *_l2_hit_pct = "
                     "lts__t_sector_hit_rate.pct; *_source_sha = bench.kernel_source_sha of the "
                     "captured build (tools/ncu_traffic.py)")
    out[engine] = int(round(val("dram__bytes_read.sum") + val("dram__bytes_write.sum")))
    out[engine + "_l2_hit_pct"] = float(d["lts__t_sector_hit_rate.pct"])
    out[engine + "_source_sha"] = bench.kernel_source_sha(engine)
    out[engine + "_captured"] = datetime.date.today().isoformat() + " " + os.path.basename(rep)
    json.dump(out, open(p, "w"), indent=2)
    print(json.dumps(out, indent=2))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
