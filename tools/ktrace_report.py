#!/usr/bin/env python
"""Summarise a per-launch timeline (SV_KTRACE=<csv>): real kernel spans in graph
replay with programmatic dependent launch, per kind, and the idle gaps between
consecutive launches (first CTA start of launch i+1 minus last CTA end of i)."""
import sys
from collections import defaultdict

import numpy as np

KINDS = ["embed", "qkv", "attn", "o", "gate_up", "down", "lm_exit", "acc_exit", "lm_final", "acc_final"]


def main(path):
    r = np.genfromtxt(path, delimiter=",", names=True, dtype=None, encoding=None)
    t0 = r["start_ns"].min()
    st = (r["start_ns"] - t0) / 1e3
    en = (r["end_ns"] - t0) / 1e3
    print(f"step span {en.max():.1f} us over {len(r)} launches")
    dur = defaultdict(list)
    gap = defaultdict(list)
    main = [i for i in range(len(r)) if KINDS[r["kind"][i]] not in ("lm_exit", "acc_exit")]
    for i in range(len(r)):
        dur[KINDS[r["kind"][i]]].append(en[i] - st[i])
    for a, b in zip(main, main[1:]):
        gap[KINDS[r["kind"][b]]].append(st[b] - en[a])
    print(f"{'kind':>10} {'n':>4} {'span_us':>8} {'gap_before_us':>14}")
    for k in KINDS:
        if dur[k]:
            g = np.mean(gap[k]) if gap[k] else float("nan")
            print(f"{k:>10} {len(dur[k]):4d} {np.mean(dur[k]):8.2f} {g:14.2f}")
    lay = [i for i in main if r["layer"][i] == 5]
    print("layer 5 launches (start, end us):", [(KINDS[r['kind'][i]], round(st[i], 1), round(en[i], 1)) for i in lay])


if __name__ == "__main__":
    main(sys.argv[1])
