#!/usr/bin/env python
"""Persistent-GEMM wait accounting of one traced step (libsv_tr.so, -DSV_GB_TRACE,
SV_GTRACE=<csv>): per GEMM kind, the mean over CTAs (and layers) of the time the
producer waited for a free ring slot, the MMA issuer for operands / a free TMEM
accumulator, and the epilogue for a finished accumulator (us per CTA)."""
import sys
from collections import defaultdict

KIND = {1: "qkv", 3: "o", 4: "gate_up", 5: "down", 6: "lm_exit", 8: "lm_final"}
rows = [l.strip().split(",") for l in open(sys.argv[1]).readlines()[1:]]
acc = defaultdict(lambda: defaultdict(float))
for r in rows:
    i, k, layer, ph, first = int(r[0]), int(r[1]), int(r[2]), int(r[3]), int(r[4])
    if k in KIND and ph in (6, 7, 8, 9, 10):
        acc[(KIND[k], i)][ph] = first + 1   # stored as sum - 1
per = defaultdict(lambda: defaultdict(list))
for (kind, i), d in acc.items():
    n = d.get(10, 0)
    if n:
        for ph in (6, 7, 8, 9):
            per[kind][ph].append(d.get(ph, 0) / n / 1e3)
for kind, d in per.items():
    print(f"{kind:>8}: producer waits slot {sum(d[6])/len(d[6]):7.2f} us | MMA waits operands {sum(d[7])/len(d[7]):7.2f}"
          f" | MMA waits TMEM {sum(d[8])/len(d[8]):7.2f} | epilogue waits accumulator {sum(d[9])/len(d[9]):7.2f}  ({len(d[6])} launches)")
