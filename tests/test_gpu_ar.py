"""gamma = 0: the plain autoregressive step on the same kernels ("Cloud AR",
PAPER.md:318, T-latency row 1): one query row per
request, next token = argmax p_0 (greedy) or the exponential-race sample of p_0
(Leviathan's bonus draw with no drafts, R2).  Multi-round decoding
through the C ABI against the oracle, margin-binned."""
import numpy as np
import pytest
import torch

from oracle import model as om
from oracle.verify import verify_step
from workload import tiny
from workload.configs import ModelCfg

from .gpu_helpers import Tally, oracle_session, row_rel_err, save_report

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape", ["tiny", "7b_width"])
@pytest.mark.parametrize("greedy", [True, False], ids=["greedy", "sampled"])
def test_ar_decode_against_oracle(svlib, shape, greedy):
    from paper_2505_21594_b200 import sv
    mc = tiny() if shape == "tiny" else ModelCfg(n_layers=2, d_model=4096, n_heads=32, d_ff=11008,
                                                  vocab=32000, max_ctx=256)
    B, ctx, rounds = 3, 40, 6
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=B, max_gamma=4)
    model = om.Model(mc, seed=1)
    dummy = torch.empty(1, device="cuda")              # gamma = 0 sampled: non-NULL, never read
    gs, os_ = [], []
    for b in range(B):
        s = eng.open_session(40 + b, 900 + b)
        s.fill_kv(ctx, kv_seed=11 + b)
        gs.append(s)
        os_.append(oracle_session(mc, model, 40 + b, 900 + b, 11 + b, ctx))
    pending = [17 + b for b in range(B)]
    tally, tally_e = Tally("ar_final"), Tally("ar_exit")
    for rnd in range(1, rounds + 1):
        reqs = [sv.Request(gs[b], rnd, pending[b], [], None if greedy else dummy) for b in range(B)]
        t = eng.submit(reqs, exit_layer=1)
        early = t.wait_early()
        final = t.wait_final()
        zf = t.logits(1, 0).cpu().numpy()
        ze = t.logits(0, 0).cpu().numpy()
        t.release()
        for b in range(B):
            out = verify_step(model, os_[b], rnd, pending[b], [], None if greedy else np.zeros((0, mc.vocab)),
                              exit_layer=1)
            rel, eps = row_rel_err(zf[b], out.final_logits)
            assert rel.max() < 2e-2
            assert final[b].accepted == 0 and len(final[b].emitted()) == 1
            rel_e, eps_e = row_rel_err(ze[b], out.exit_logits)
            assert rel_e.max() < 2e-2
            ctr = (900 + b, 40 + b, rnd)
            tally.add(out.final, final[b], out.final_logits, eps, None, ctr, tag=(rnd, b))
            tally_e.add(out.early, early[b], out.exit_logits, eps_e, None, ctr, tag=("exit", rnd, b))
            assert gs[b].length == ctx + rnd
            if out.final.tokens == final[b].emitted():
                pending[b] = final[b].emitted()[0]
            else:
                pending[b] = None
        if any(p is None for p in pending):
            break
    print(tally.report(), "|", tally_e.report())
    assert not tally.hard_mismatch and not tally_e.hard_mismatch
    assert tally.checked >= 0.5 * tally.n
    for s in gs:
        s.close()
    eng.close()
