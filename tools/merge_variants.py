#!/usr/bin/env python
"""Join tools/variants.py lines with the per-variant ncu launch metrics (gpu_variants.sh)
into profiles/rNN_variants.jsonl: DRAM bytes per launch of K0 (pre-projection) and K1
(render) next to the compulsory bytes of the variant.

    python tools/merge_variants.py gpurun_out/variants.jsonl gpurun_out profiles/r02_variants.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_csv import rows  # noqa: E402


def compulsory(d):
    """Bytes the render kernel must move per launch: G once per asset (fp16, 64 wide),
    x_t (+ z) read and x_{t-1} written for the DDIM views, rgb/alpha written if asked."""
    v = d["variant"]
    if v.startswith("cfg3"):
        A, R, dv, V, hw, rgb = 1, 64, 4, 8, 256 * 256, True
    elif v == "cfg2x8":
        A, R, dv, V, hw, rgb = 8, 64, 4, 4, 128 * 128, False
    elif v == "cfg4":
        A, R, dv, V, hw, rgb = 8, 64, 4, 4, 256 * 256, False
    else:  # cachebust
        A, R, dv, V, hw, rgb = 8, 256, 4, 4, 256 * 256, False
    g = A * (3 * R * R + 1) * 64 * 2
    x = A * dv * 3 * hw * 4 * (3 if "eta1" in v else 2)  # x_t (+ z) in, x_{t-1} out
    out = A * V * 4 * hw * 4 if rgb else 0
    return {"G": g, "x": x, "rgb_alpha": out, "total": g + x + out}


def main(var, ncu_dir, out):
    lines = []
    for ln in open(var):
        d = json.loads(ln)
        name = d["variant"].replace("_skip", "")
        p = os.path.join(ncu_dir, f"ncu_var_{name}.csv")
        if os.path.exists(p) and not d["variant"].endswith("_skip"):
            k = {}
            for i, kern, m, u, val in rows(p):
                key = "K0_preproject" if "preproject" in kern else "K1_render"
                k.setdefault(key, {})[m] = float(val.replace(",", ""))
            d["ncu_per_launch"] = {
                kk: {"dram_bytes": vv.get("dram__bytes_read.sum", 0) + vv.get("dram__bytes_write.sum", 0),
                     "dram_read": vv.get("dram__bytes_read.sum"), "dram_write": vv.get("dram__bytes_write.sum"),
                     "ms": vv.get("gpu__time_duration.sum", 0) / 1e6,
                     "l2_hit_pct": vv.get("lts__t_sector_hit_rate.pct"),
                     "tensor_pipe_pct": vv.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active")}
                for kk, vv in k.items()}
            d["render_compulsory_bytes"] = compulsory(d)
            k1 = d["ncu_per_launch"].get("K1_render")
            if k1:
                d["render_dram_read_over_compulsory_read"] = k1["dram_read"] / (
                    d["render_compulsory_bytes"]["G"] + d["render_compulsory_bytes"]["x"] * (2 / 3 if "eta1" in name else 1 / 2))
        lines.append(d)
    with open(out, "w") as f:
        for d in lines:
            f.write(json.dumps(d) + "\n")
    for d in lines:
        print(d["variant"], round(d["rays_per_s"] / 1e6, 1), "M rays/s", round(d["roofline"]["frac"], 3),
              d.get("render_dram_read_over_compulsory_read"))


if __name__ == "__main__":
    main(*sys.argv[1:4])
