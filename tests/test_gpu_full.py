"""Full-size parity: configs[1] (Llama2-7B shape, 32 layers, d 4096, V 32000, bf16,
batch 1, ctx 512, gamma 4, early exit at layer 16) in the launch configuration
bench.py times (graph replay, stochastic acceptance), against the fp64 oracle
computing the same single request (weights regenerated layer by layer)."""
import numpy as np
import pytest
import torch

from oracle import model as om
from oracle.verify import Session as OSession
from oracle.verify import verify_step
from workload import drafts as wd
from workload import llama2_7b

from .gpu_helpers import Tally, decision_bound, row_rel_err

pytestmark = pytest.mark.gpu


def test_c2_full_size_against_oracle(svlib):
    from paper_2505_21594_b200 import sv
    mc = llama2_7b()
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=1, max_gamma=4, kv_blocks=12)
    s = eng.open_session(1, 0x5EED0001)
    s.fill_kv(512, kv_seed=1000)
    pend = int(wd.prefix_tokens(3, 1, mc.vocab)[0])
    x, q = wd.timing_drafts(9, 1, 4, mc.vocab)
    t = eng.submit([sv.Request(s, 1, pend, x[0], torch.from_numpy(q[0]).cuda())], exit_layer=16)
    early = t.wait_early()[0]
    final = t.wait_final()[0]
    zf = t.logits(1, 4).cpu().numpy()[0]
    ze = t.logits(0, 4).cpu().numpy()[0]
    t.release()
    k_gpu, v_gpu = s.kv_rows(31, 512, final.accepted + 1)
    s.close()
    eng.close()
    del W
    torch.cuda.empty_cache()

    model = om.Model(mc, seed=1, lazy=True)
    osess = OSession(1, 0x5EED0001, om.KVCache.synthetic(mc, 1000, 512))
    out = verify_step(model, osess, 1, pend, x[0], q[0].astype(np.float64), exit_layer=16)
    rel_f, eps_f = row_rel_err(zf, out.final_logits)
    rel_e, eps_e = row_rel_err(ze, out.exit_logits)
    print("final rel err per row", rel_f, "exit", rel_e)
    assert rel_f.max() < 2e-2 and rel_e.max() < 2e-2
    tally = Tally()
    tally.add(out.final, final, decision_bound(eps_f.max()), "final")
    tally.add(out.early, early, decision_bound(eps_e.max()), "exit")
    print(tally.report(), "oracle", out.final.tokens, out.early.tokens, "gpu", final.emitted(), early.emitted())
    assert not tally.hard_mismatch
    # KV rows the step appended at layer 32 (accepted prefix) vs the oracle's, to bf16
    if out.final.tokens == final.emitted():
        kref = osess.cache.k[31][:, 512:512 + final.accepted + 1, :].transpose(1, 0, 2).reshape(-1, mc.d_model)
        kg = (k_gpu.astype(np.uint32) << 16).view(np.float32)
        assert np.abs(kg - kref).max() <= 2e-2 * np.abs(kref).max()
