#!/usr/bin/env python
"""Per-launch timeline of one graph-replayed verify step (sv_debug_trace_*), PDL on:
for a few layers, every launch's first-CTA start and last-CTA end relative to the
end of the previous main-stream launch, and the per-kind critical-path charge
(end of launch - end of the previous launch) against its HBM floor.

  python tools/trace_step.py [--batch B] [--ctx C] [--gamma G] [--exit L] [--reps R]
"""
import argparse
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--ctx", type=int, default=512)
    ap.add_argument("--gamma", type=int, default=4)
    ap.add_argument("--exit", type=int, default=16)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--layers", default="10,11")
    args = ap.parse_args()
    import torch
    from paper_2505_21594_b200 import sv
    from workload import drafts as wd
    from workload import llama2_7b
    mc = llama2_7b()
    B, G = args.batch, args.gamma + 1
    W = sv.Weights(mc, seed=1)
    blocks = (args.ctx + G + 63) // 64
    eng = sv.Engine(mc, W, max_batch=B, max_gamma=args.gamma, kv_blocks=B * blocks)
    ss = []
    for b in range(B):
        s = eng.open_session(b + 1, 7 + b)
        s.fill_kv(args.ctx, kv_seed=100 + b)
        ss.append(s)
    x, q = wd.timing_drafts(3, B, args.gamma, mc.vocab)
    qd = torch.from_numpy(q).cuda()
    rnd = [0]

    def step(trace):
        rnd[0] += 1
        for s in ss:
            s.rewind(args.ctx)
        if trace:
            eng.trace_next()
        t = eng.submit([sv.Request(s, rnd[0], 5, x[b], qd[b]) for b, s in enumerate(ss)], exit_layer=args.exit)
        if args.exit:
            t.wait_early()
        t.wait_final()
        t.release()
        return eng.trace_read() if trace else None

    for _ in range(5):
        step(False)
    M = B * G
    d, F, V = mc.d_model, mc.d_ff, mc.vocab
    floor_bytes = {"gemm_qkv": 3 * d * d * 2, "gemm_o": d * d * 2, "gemm_gate_up": 2 * F * d * 2,
                   "gemm_down": d * F * 2, "attention": B * (args.ctx + G) * d * 4, "gemm_lm_final": V * d * 2}
    hbm = 6557.1e9
    charged = {}
    spans = {}
    last_trace = [None]
    for rep in range(args.reps):
        tr = step(True)
        last_trace[0] = tr
        prev = None
        for r in tr:
            if r["stream"] != 0:
                continue
            c = r["end_us"] - (r["start_us"] if prev is None else prev)
            charged.setdefault((r["kind"], r["layer"]), []).append(c)
            spans.setdefault((r["kind"], r["layer"]), []).append(
                (r["start_us"] - (prev if prev is not None else r["start_us"]), r["end_us"] - r["start_us"]))
            prev = r["end_us"] if prev is None else max(prev, r["end_us"])
        step(False)
    print(f"B={B} ctx={args.ctx} gamma={args.gamma}: traced step {tr[-1]['end_us']:.1f} us")
    kinds = ["embed", "gemm_qkv", "attention", "gemm_o", "gemm_gate_up", "gemm_down", "gemm_lm_final", "accept_final"]
    print(f"{'kind':>14} {'charged us/launch':>18} {'floor us':>9} {'start-prev_end':>15} {'span':>7}")
    for k in kinds:
        keys = [kk for kk in charged if kk[0] == k]
        if not keys:
            continue
        ch = statistics.mean(statistics.median(charged[kk]) for kk in keys)
        st = statistics.mean(statistics.median(v[0] for v in spans[kk]) for kk in keys)
        sp = statistics.mean(statistics.median(v[1] for v in spans[kk]) for kk in keys)
        fl = floor_bytes.get(k, 0) / hbm * 1e6
        print(f"{k:>14} {ch:18.2f} {fl:9.2f} {st:15.2f} {sp:7.2f}")
    for L in (int(v) for v in args.layers.split(",")):
        print(f"layer {L}:", [(r["kind"], round(r["start_us"], 1), round(r["end_us"], 1)) for r in tr
                              if r["layer"] == L and r["stream"] == 0])
    gpath = os.environ.get("SV_GTRACE")
    if gpath and os.path.exists(gpath):   # GEMM phase stamps of the last traced step
        tr = last_trace[0]
        base = {}
        prev = None
        for r in tr:
            if r["stream"] != 0:
                continue
            base[(r["kind"], r["layer"])] = (prev, r)
            prev = r["end_us"]
        t0ns = None
        rows = [ln.strip().split(",") for ln in open(gpath).readlines()[1:]]
        t0ns = min(int(x[4]) for x in rows)
        kinds = ["embed", "gemm_qkv", "attention", "gemm_o", "gemm_gate_up", "gemm_down"]
        names = ["start", "pdl_wait", "mma_done|first_full", "ticket|mma_end", "reduce_beg|flags_ok", "end",
                 "reduce_end", "partials|flags_wait", "epi_beg|c0_acc", "epi_end|c0_sout", "c0_epi", "lp_beg",
                 "lp_rstd", "lp_tfull", "lp_end"]
        # the final acceptance pair: accept phases at its id, row_stats at id + 1 (relative to the LM head end)
        ids = sorted({int(x[0]) for x in rows if int(x[1]) == 9})
        if ids:
            i0 = ids[0]
            pe, rec = base[("accept_final", -1)]
            st0 = min(int(x[4]) for x in rows if int(x[0]) in (i0, i0 + 1))
            off = rec["start_us"] * 1e3 - (st0 - t0ns)
            for i, nm in ((i0 + 1, "row_stats"), (i0, "accept")):
                ph = {int(x[3]): (int(x[4]), int(x[5])) for x in rows if int(x[0]) == i}
                print(f"accept_final {nm:>9} (us after the LM head ended):",
                      ", ".join(f"p{p} {((ph[p][0] - t0ns + off) / 1e3 - pe):.1f}..{((ph[p][1] - t0ns + off) / 1e3 - pe):.1f}"
                                for p in sorted(ph)))
        for L in (int(v) for v in args.layers.split(",")):
            for k in (1, 3, 4, 5):
                ph = {int(x[3]): (int(x[4]), int(x[5])) for x in rows if int(x[1]) == k and int(x[2]) == L}
                pe, rec = base[(kinds[k], L)]
                # the trace's times are relative to the step's first kernel start; re-base the stamps on it
                off = (rec["start_us"] * 1e3) - (ph[0][0] - t0ns) if 0 in ph else 0
                rel = lambda ns: (ns - t0ns + off) / 1e3 - pe
                print(f"layer {L} {kinds[k]:>13} (us after the previous launch ended):",
                      ", ".join(f"{names[p]} {rel(ph[p][0]):.1f}..{rel(ph[p][1]):.1f}" for p in sorted(ph)))
    for s in ss:
        s.close()
    eng.close()


if __name__ == "__main__":
    main()
