"""Exit adapters (structure only): GPU
adapter weights bit-identical to the oracle generator; early exits through
A_l(h) = h + silu(RMSNorm(h) g W_dn^T) W_up^T (R7b) against the fp64
oracle (exit logits within 2e-2, decisions margin-binned), single exit and the
all-exits stream; the final result is unchanged by the adapters."""
import dataclasses

import numpy as np
import pytest
import torch

from oracle import gen
from oracle import model as om
from oracle.verify import verify_step
from workload import drafts as wd
from workload import tiny
from workload.configs import ModelCfg

from .gpu_helpers import Tally, oracle_session, row_rel_err, save_report

pytestmark = pytest.mark.gpu


def _cfg(shape):
    if shape == "tiny4":
        return dataclasses.replace(tiny(), n_layers=4), 128
    return ModelCfg(n_layers=3, d_model=4096, n_heads=32, d_ff=11008, vocab=32000, max_ctx=256), 384


@pytest.mark.parametrize("shape", ["tiny4", "7b_width3"])
def test_exit_adapters_against_oracle(svlib, shape):
    from paper_2505_21594_b200 import sv
    mc, rank = _cfg(shape)
    L, B, gamma, ctx = mc.n_layers, 2, 4, 40
    W = sv.Weights(mc, seed=1)
    A = sv.Adapters(mc, rank, seed=9)
    # generator bits: one adapter, every tensor, against oracle/gen.py
    for l in (1, L - 1):
        w = gen.adapter_weights(mc, 9, l, rank)
        for k, ref in (("dn", w["dn"]), ("up", w["up"]), ("g", w["g"])):
            n = ref.size
            off = A._arr[k][l - 1] - A.buf.data_ptr()
            got = A.buf[off:off + 2 * n].view(torch.bfloat16).float().cpu().numpy().astype(np.float64)
            assert np.array_equal(got.reshape(ref.shape), ref), (l, k)
    eng = sv.Engine(mc, W, max_batch=B, max_gamma=gamma)
    model = om.Model(mc, seed=1)
    oad = om.Adapters(mc, 9, rank, range(1, L))
    x, q = wd.timing_drafts(41, B, gamma, mc.vocab, s=1.1)
    qd = torch.from_numpy(q).cuda()

    def run(exit_layer=None, exits=None):
        ss = []
        for b in range(B):
            s = eng.open_session(50 + b, 600 + b)
            s.fill_kv(ctx, kv_seed=21 + b)
            ss.append(s)
        reqs = [sv.Request(ss[b], 1, 13 + b, x[b], qd[b]) for b in range(B)]
        if exits:
            t = eng.submit_exits(reqs, exits)
            got = [t.wait_exit(k) for k in range(len(exits))]
        else:
            t = eng.submit(reqs, exit_layer=exit_layer)
            got = [t.wait_early()]
        f = t.wait_final()
        ze = t.logits(0, gamma).cpu().numpy()
        zf = t.logits(1, gamma).cpu().numpy()
        t.release()
        for s in ss:
            s.close()
        return got, f, ze, zf

    _, f_plain, _, zf_plain = run(exit_layer=1)
    eng.set_adapters(A)
    tally = Tally("adapters")
    for le in range(1, L):
        got, f, ze, zf = run(exit_layer=le)
        assert np.array_equal(zf, zf_plain)                       # exits are read-only
        assert [r.asdict() for r in f] == [r.asdict() for r in f_plain]
        for b in range(B):
            out = verify_step(model, oracle_session(mc, model, 50 + b, 600 + b, 21 + b, ctx), 1, 13 + b, x[b],
                              q[b].astype(np.float64), exit_layer=le, adapters=oad)
            rel, eps = row_rel_err(ze[b], out.exit_logits)
            assert rel.max() < 2e-2, (le, b, rel.max())
            plain = verify_step(model, oracle_session(mc, model, 50 + b, 600 + b, 21 + b, ctx), 1, 13 + b, x[b],
                                q[b].astype(np.float64), exit_layer=le)
            assert not np.allclose(out.exit_logits, plain.exit_logits)   # the adapter acts
            tally.add(out.early, got[0][b], out.exit_logits, eps, q[b], (600 + b, 50 + b, 1), tag=(le, b))
    # the all-exits stream with adapters: exit k equals the single-exit run of that layer
    exits = list(range(1, L + 1))
    got_all, _, _, _ = run(exits=exits)
    for k, le in enumerate(exits[:-1]):
        single, _, _, _ = run(exit_layer=le)
        assert [r.asdict() for r in got_all[k]] == [r.asdict() for r in single[0]]
    print(tally.report())
    save_report(tally.name, tally.asdict())
    assert not tally.hard_mismatch and tally.checked >= 1
    eng.set_adapters(None)
    eng.close()
