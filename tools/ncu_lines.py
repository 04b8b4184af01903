#!/usr/bin/env python
"""Per-source-line warp-stall samples and executed instructions of one kernel in
an ncu report (reads `ncu --page source --print-source cuda,sass --csv`)."""
import csv
import subprocess
import sys


def main(rep, skip=0, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(skip),
                          "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    agg, fname = {}, ""
    for r in csv.reader(out.splitlines()):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] in ("Function Name", "Line No") or r[0] == "":
            continue
        try:
            samp, inst = float(r[4] or 0), float(r[7] or 0)
        except (ValueError, IndexError):
            continue
        agg[(fname, r[0], r[1][:90])] = (samp, inst)
    tot = sum(v[0] for v in agg.values())
    print(f"total samples {tot:.0f}")
    for (f, ln, src), (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{s:7.0f} {100 * s / tot:5.1f}% {i:10.0f}  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
