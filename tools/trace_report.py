#!/usr/bin/env python
"""Summarise a fused-kernel timeline (SV_TRACE=<csv> dump of the last step):
per stage, when its first weight load was issued, when its activations became
available (first B load), when its first/last work item ran, across all CTAs."""
import sys
from collections import defaultdict

import numpy as np

TYPES = {1: "embed", 2: "gemm", 3: "attn", 4: "stats", 5: "accept"}


def main(path, nstages_show=40, first_stage=0):
    rows = np.genfromtxt(path, delimiter=",", names=True, dtype=None, encoding=None)
    t0 = min(r["t_a"] for r in rows if r["t_a"] > 0) if any(r["t_a"] > 0 for r in rows) else rows["t_work"][rows["t_work"] > 0].min()
    t0 = min(t0, rows["t_work"][rows["t_work"] > 0].min())
    by = defaultdict(list)
    for r in rows:
        by[int(r["stage"])].append(r)
    end_all = rows["t_end"].max()
    print(f"step span {(end_all - t0) / 1e3:.1f} us, items {len(rows)}")
    print(f"{'stage':>5} {'type':>6} {'n':>5} {'A_first':>9} {'B_first':>9} {'B_last':>9} {'work_first':>10} {'end_first':>9} {'end_last':>9}  (us from step start)")
    for st in sorted(by)[first_stage:first_stage + nstages_show]:
        rs = by[st]
        f = lambda k, fn: (fn([r[k] for r in rs if r[k] > 0]) - t0) / 1e3 if any(r[k] > 0 for r in rs) else float("nan")
        print(f"{st:5d} {TYPES[int(rs[0]['type'])]:>6} {len(rs):5d} {f('t_a', min):9.1f} {f('t_b', min):9.1f} "
              f"{f('t_b', max):9.1f} {f('t_work', min):10.1f} {f('t_end', min):9.1f} {f('t_end', max):9.1f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40, int(sys.argv[3]) if len(sys.argv) > 3 else 0)
