#!/usr/bin/env python
"""Run verify steps of a config with the CUDA profiler API bracketing only the
measured steps, for `ncu --profile-from-start off` (launch lists and full
captures of the kernels of one step; numbers printed under ncu are never bench
values).

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
      --csv --log-file gpurun_out/launches.csv python tools/ncu_step.py --config C2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--ctx", type=int, default=512)
    ap.add_argument("--gamma", type=int, default=4)
    ap.add_argument("--exit-layer", type=int, default=16)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--graphs", type=int, default=1)
    args = ap.parse_args()
    import torch

    from paper_2505_21594_b200 import sv
    from workload import llama2_7b
    from workload.drafts import prefix_tokens, timing_drafts
    mc = llama2_7b()
    W = sv.Weights(mc, seed=1)
    B = args.batch
    eng = sv.Engine(mc, W, max_batch=B, max_gamma=args.gamma,
                    kv_blocks=B * ((args.ctx + 16) // 64 + 2), use_graphs=bool(args.graphs))
    ss = []
    for b in range(B):
        s = eng.open_session(b + 1, 77 + b)
        s.fill_kv(args.ctx, kv_seed=5 + b)
        ss.append(s)
    pend = prefix_tokens(1, B, mc.vocab)
    x, q = timing_drafts(2, B, args.gamma, mc.vocab)
    qd = torch.from_numpy(q).cuda()
    rnd = [0]

    def step():
        rnd[0] += 1
        for s in ss:
            s.rewind(args.ctx)
        eng.verify([sv.Request(s, rnd[0], pend[b], x[b], qd[b]) for b, s in enumerate(ss)],
                   exit_layer=args.exit_layer)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("kernels/step", eng.last_launches())


if __name__ == "__main__":
    main()
