"""Debug: compare graph replay vs direct launches at the 7B width (2 layers)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_21594_b200 import sv  # noqa: E402
from workload import drafts as wd  # noqa: E402
from workload.configs import ModelCfg  # noqa: E402

mc = ModelCfg(n_layers=2, d_model=4096, n_heads=32, d_ff=11008, vocab=32000, max_ctx=512)
W = sv.Weights(mc, seed=1)
for B, ctx, ex in [(2, 300, 1), (2, 300, 0), (2, 200, 1), (1, 300, 1), (3, 300, 1)]:
    out = {}
    for ug in (True, False):
        eng = sv.Engine(mc, W, max_batch=B, max_gamma=8, use_graphs=ug)
        ss = [eng.open_session(1 + b, 7 + b) for b in range(B)]
        for b, s in enumerate(ss):
            s.fill_kv(ctx, kv_seed=5 + b)
        x, q = wd.timing_drafts(9, B, 4, mc.vocab, s=1.1)
        qd = torch.from_numpy(q).cuda()
        t = eng.submit([sv.Request(ss[b], 1, 3, x[b], qd[b]) for b in range(B)], exit_layer=ex)
        if ex:
            t.wait_early()
        t.wait_final()
        z = t.logits(1, 4).cpu().numpy()
        t.release()
        eng.close()
        out[ug] = z
    za, zb = out[True], out[False]
    print(f"B={B} ctx={ctx} exit={ex}: nan graph {np.isnan(za).sum(axis=(1,2))} direct {np.isnan(zb).sum(axis=(1,2))} "
          f"maxdiff {np.nanmax(np.abs(za - zb)):.3e} equal {np.array_equal(za, zb)}", flush=True)
