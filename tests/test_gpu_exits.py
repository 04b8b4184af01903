"""All-exits streaming verify (Alg-S, PAPER.md:1103-1106:
the server verifies the draft at every exit and pushes each exit's result as soon
as it is computed) through the C ABI (sv_verify_submit_exits / sv_wait_exit /
sv_exits_ready), against the oracle and against the single-exit path."""
import dataclasses

import numpy as np
import pytest
import torch

from oracle import model as om
from oracle.verify import verify_step
from workload import drafts as wd
from workload import tiny
from workload.configs import ModelCfg

from .gpu_helpers import Tally, oracle_session, row_rel_err, save_report

pytestmark = pytest.mark.gpu


def _cfg(shape):
    if shape == "tiny4":
        return dataclasses.replace(tiny(), n_layers=4)
    return ModelCfg(n_layers=4, d_model=4096, n_heads=32, d_ff=11008, vocab=32000, max_ctx=256)


@pytest.mark.parametrize("shape", ["tiny4", "7b_width4"])
@pytest.mark.parametrize("greedy", [True, False], ids=["greedy", "stochastic"])
def test_all_exits_against_oracle_and_single_exit(svlib, shape, greedy):
    from paper_2505_21594_b200 import sv
    mc = _cfg(shape)
    L, B, gamma, ctx = mc.n_layers, 2, 4, 40
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=B, max_gamma=gamma)
    model = om.Model(mc, seed=1)
    exits = list(range(1, L + 1))                    # every layer; l = L is the final layer
    x, q = wd.timing_drafts(21, B, gamma, mc.vocab, s=1.1)
    qd = torch.from_numpy(q).cuda()

    def fresh():
        ss = []
        for b in range(B):
            s = eng.open_session(30 + b, 500 + b)
            s.fill_kv(ctx, kv_seed=7 + b)
            ss.append(s)
        return ss

    def reqs(ss):
        return [sv.Request(ss[b], 1, 11 + b, x[b], None if greedy else qd[b]) for b in range(B)]

    # 1. all exits in one step, streamed
    ss = fresh()
    t = eng.submit_exits(reqs(ss), exits)
    got = [t.wait_exit(k) for k in range(len(exits))]
    assert t.exits_ready() == len(exits)
    final = t.wait_final()
    zf = t.logits(1, gamma).cpu().numpy()
    t.release()
    lens = [s.length for s in ss]
    for s in ss:
        s.close()
    # 2. no exit: the final result and logits are bitwise the same (exits are read-only)
    ss = fresh()
    t = eng.submit(reqs(ss), exit_layer=0)
    f0 = t.wait_final()
    z0 = t.logits(1, gamma).cpu().numpy()
    t.release()
    assert [s.length for s in ss] == lens
    for s in ss:
        s.close()
    assert np.array_equal(z0, zf)
    assert [r.asdict() for r in f0] == [r.asdict() for r in final]
    # 3. every exit equals the single-exit run of that layer, bitwise (whose exit
    # logits are downloaded for the oracle comparison below)
    ze = {}
    for k, le in enumerate(exits):
        ss = fresh()
        t = eng.submit(reqs(ss), exit_layer=le)
        e1 = t.wait_early()
        t.wait_final()
        ze[le] = t.logits(0, gamma).cpu().numpy()
        t.release()
        for s in ss:
            s.close()
        for b in range(B):
            a, c = got[k][b].asdict(), e1[b].asdict()
            assert a == c, (le, b, a, c)
            assert a["exit_layer"] == le and a["is_final"] == 0
    # exit at l = L equals the final result
    for b in range(B):
        e, f = got[-1][b].asdict(), final[b].asdict()
        for key in ("accepted", "tokens", "score", "next_prob", "status"):
            assert e[key] == f[key], key
    # 4. against the oracle: every exit's decisions (margin-binned)
    tally = Tally(f"all_exits_{shape}_{'greedy' if greedy else 'stochastic'}")
    for b in range(B):
        osess = oracle_session(mc, model, 30 + b, 500 + b, 7 + b, ctx)
        out = verify_step(model, osess, 1, 11 + b, x[b], None if greedy else q[b].astype(np.float64),
                          exit_layers=exits)
        rel, eps = row_rel_err(zf[b], out.final_logits)
        assert rel.max() < 2e-2
        for k, (le, r, zl) in enumerate(out.exits):
            rel_l, eps_l = row_rel_err(ze[le][b], zl)
            assert rel_l.max() < 2e-2
            tally.add(r, got[k][b], zl, eps_l, None if greedy else q[b], (500 + b, 30 + b, 1), tag=(le, b))
    print(tally.report())
    save_report(tally.name, tally.asdict())
    assert not tally.hard_mismatch, tally.hard_mismatch
    assert tally.checked >= (0.75 if shape == "tiny4" else 0.3) * tally.n
    eng.close()


def test_exit_list_validation(svlib):
    from paper_2505_21594_b200 import sv
    mc = _cfg("tiny4")
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=1, max_gamma=4)
    s = eng.open_session(1, 2)
    s.fill_kv(20, kv_seed=3)
    for bad in ([2, 1], [0], [5], [1, 1]):
        with pytest.raises(sv.SvError):
            eng.submit_exits([sv.Request(s, 1, 3, [1, 2, 3, 4])], bad)
    assert s.length == 20
    s.close()
    eng.close()
