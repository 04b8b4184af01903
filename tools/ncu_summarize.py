#!/usr/bin/env python
"""Summarise the ncu evidence of one verify step into profiles/<name>.json:
  --list  CSV of `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv`
          (every launch of one step: cold-cache, serialised -> per-kind time SHARE of the step)
  --full  .ncu-rep of `ncu --set full` on the GEMM / attention launches of one layer
Per kernel kind: launches, mean duration, mean DRAM bytes (read + write) per launch,
DRAM / SM throughput % of peak, registers, grid, cluster size."""
import argparse
import csv
import json
import subprocess
from collections import defaultdict

KIND_BY_NAME = [("embed_kernel", "embed"), ("attn3_kernel", "attention"), ("row_stats", "accept_stats"),
                ("accept_kernel", "accept"), ("gemm_big", "gemm_big"), ("gemm_kernel", "gemm")]
GEMM_EPI = {"0": "qkv", "1": "resid(o/down)", "2": "gate_up", "3": "lm_head"}


def kind_of(name):
    for key, k in KIND_BY_NAME:
        if key in name:
            if k == "gemm" and "<" in name:
                epi = name.split("<")[1].split(">")[0].split(",")[1].strip().replace("(int)", "")
                return f"gemm_{GEMM_EPI.get(epi, epi)}"
            return k
    return name.split("(")[0]


def read_list(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    iK, iM, iU, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    iID = hdr.index("ID")
    per = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        v = float(r[iV].replace(",", ""))
        u = r[iU]
        if u in ("ns",):
            v /= 1e3
        elif u == "usecond":
            pass
        elif u == "msecond":
            v *= 1e3
        elif u == "Kbyte":
            v *= 1e3
        elif u == "Mbyte":
            v *= 1e6
        elif u == "Gbyte":
            v *= 1e9
        per[r[iID]][r[iM]] = v
        names[r[iID]] = r[iK]
    fam = defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        k = kind_of(names[i])
        f = fam[k]
        f[0] += 1
        f[1] += m.get("gpu__time_duration.sum", 0.0)
        f[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(f[1] for f in fam.values())
    return {k: {"launches": f[0], "us_total": round(f[1], 2), "share_of_step": round(f[1] / tot, 4),
                "us_per_launch": round(f[1] / f[0], 3), "dram_bytes_per_launch": round(f[2] / f[0])}
            for k, f in sorted(fam.items(), key=lambda kv: -kv[1][1])}, tot


def read_full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, data = rows[0], rows[2:]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "launch__grid_size", "launch__cluster_dim_z", "launch__cluster_dim_x", "lts__t_sector_hit_rate.pct"]
    units = rows[1]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")][:80], "kind": kind_of(r[hdr.index("Kernel Name")])}
        for w in want:
            if w in hdr:
                d[w] = f"{r[hdr.index(w)]} {units[hdr.index(w)]}".strip()
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--list")
    ap.add_argument("--full")
    ap.add_argument("--out", required=True)
    ap.add_argument("--source", default="")
    a = ap.parse_args()
    js = {"source": a.source}
    if a.list:
        fam, tot = read_list(a.list)
        js["step_us_serialised"] = round(tot, 1)
        js["families"] = fam
        g = [v for k, v in fam.items() if k.startswith("gemm")]
        n = sum(v["launches"] for v in g)
        js["dram_bytes_per_launch"] = {
            "gemm": sum(v["dram_bytes_per_launch"] * v["launches"] for v in g) / max(1, n),
            "attn": fam.get("attention", {}).get("dram_bytes_per_launch")}
    if a.full:
        js["full_capture"] = read_full(a.full)
    json.dump(js, open(a.out, "w"), indent=1)
    print(json.dumps({k: v for k, v in js.items() if k != "full_capture"}, indent=1)[:3000])


if __name__ == "__main__":
    main()
