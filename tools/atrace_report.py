#!/usr/bin/env python
"""Attention phase timeline (SV_ATRACE=<csv>) joined with the launch timeline
(SV_KTRACE=<csv>): per phase, median over layers of the time since the QKV launch
of the same layer ended (negative = before)."""
import sys
import numpy as np

PH = ["start", "pagetable", "pdl_wait", "q_ready", "mainloop", "warp_merge", "cluster_sync", "end"]


def main(apath, kpath):
    a = np.genfromtxt(apath, delimiter=",", names=True, dtype=np.int64)
    k = np.genfromtxt(kpath, delimiter=",", names=True, dtype=None, encoding=None)
    qkv_end = {int(r["layer"]): int(r["end_ns"]) for r in k if int(r["kind"]) == 1}
    for cta in (0, 1):
        print(f"CTA {'first' if cta == 0 else 'last'} (us relative to the end of the layer's QKV launch)")
        for p, nm in enumerate(PH):
            v = [(int(r["t_ns"]) - qkv_end[int(r["layer"])]) / 1e3 for r in a
                 if int(r["cta"]) == cta and int(r["phase"]) == p and int(r["t_ns"]) > 0 and int(r["layer"]) in qkv_end]
            if v:
                print(f"  {nm:>12}: median {np.median(v):8.2f}  min {np.min(v):8.2f}  max {np.max(v):8.2f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
