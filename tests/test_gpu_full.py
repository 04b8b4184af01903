"""Full-size parity: configs[1] (Llama2-7B shape, 32 layers, d 4096, V 32000, bf16,
batch 1, ctx 512, gamma 4, early exit at layer 16) in the launch configuration
bench.py times (one request per submit, graph replay, stochastic acceptance).

- Level E: eight sessions, two rounds each, against the fp64 oracle computing the
  same requests (weights regenerated layer by layer, one pass for all sessions);
  every decision binned by its propagated bound (tests/gpu_helpers.py), at least
  20 decisions must be checked, and none of them may differ.
- Level U: the oracle's acceptance on the GPU's own downloaded fp32 logits with the
  session's counters, over calibrated drafts (bench.py's workload) that exercise
  every acceptance length: bit-exact wherever every margin > 1e-3.
Tallies are written with save_report (copied to profiles/)."""
import numpy as np
import pytest
import torch

from oracle import model as om
from oracle.verify import Session as OSession
from oracle.verify import verify_steps
from workload import drafts as wd
from workload import llama2_7b

from .gpu_helpers import Tally, UTally, row_rel_err, save_report

pytestmark = pytest.mark.gpu
N_SESS, ROUNDS, CTX, GAMMA, EXIT = 8, 2, 512, 4, 16


def test_c2_full_size_against_oracle(svlib):
    from paper_2505_21594_b200 import sv
    mc = llama2_7b()
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=1, max_gamma=GAMMA, kv_blocks=N_SESS * 10)
    ss = []
    for b in range(N_SESS):
        s = eng.open_session(1 + b, 0x5EED0001 + b)
        s.fill_kv(CTX, kv_seed=1000 + b)
        ss.append(s)
    pend = [int(t) for t in wd.prefix_tokens(3, N_SESS, mc.vocab)]
    gpu = []              # per round: [(x, q, early, final, zf, ze, k_rows)]
    live = list(range(N_SESS))
    for rnd in range(1, ROUNDS + 1):
        x, q = wd.timing_drafts(9 + rnd, N_SESS, GAMMA, mc.vocab)
        out = {}
        for b in live:
            t = eng.submit([sv.Request(ss[b], rnd, pend[b], x[b], torch.from_numpy(q[b]).cuda())],
                           exit_layer=EXIT)
            early = t.wait_early()[0]
            final = t.wait_final()[0]
            zf = t.logits(1, GAMMA).cpu().numpy()[0]
            ze = t.logits(0, GAMMA).cpu().numpy()[0]
            t.release()
            ctx = final.new_len - final.accepted - 1
            k_rows = ss[b].kv_rows(31, ctx, final.accepted + 1)[0]
            out[b] = (x[b], q[b], early, final, zf, ze, k_rows, ctx)
            pend[b] = final.emitted()[-1]
        gpu.append(out)
    for s in ss:
        s.close()
    eng.close()
    del W
    torch.cuda.empty_cache()

    model = om.Model(mc, seed=1, lazy=True)
    osess = [OSession(1 + b, 0x5EED0001 + b, om.KVCache.synthetic(mc, 1000 + b, CTX)) for b in range(N_SESS)]
    opend = [int(t) for t in wd.prefix_tokens(3, N_SESS, mc.vocab)]
    tf, te, ut = Tally("c2_full_final"), Tally("c2_full_exit"), UTally("c2_full level U")
    errs = []
    live = list(range(N_SESS))
    for rnd, out in enumerate(gpu, start=1):
        live = [b for b in live if b in out]
        res = verify_steps(model, [osess[b] for b in live], [rnd] * len(live), [opend[b] for b in live],
                           [out[b][0] for b in live], [out[b][1].astype(np.float64) for b in live], exit_layer=EXIT)
        nxt = []
        for b, o in zip(live, res):
            xb, qb, early, final, zf, ze, k_rows, ctx = out[b]
            rel_f, eps_f = row_rel_err(zf, o.final_logits)
            rel_e, eps_e = row_rel_err(ze, o.exit_logits)
            errs += [rel_f.max(), rel_e.max()]
            ctr = (0x5EED0001 + b, 1 + b, rnd)
            tf.add(o.final, final, o.final_logits, eps_f, qb, ctr, tag=(rnd, b))
            te.add(o.early, early, o.exit_logits, eps_e, qb, ctr, tag=(rnd, b))
            ut.add(zf, final, xb, qb, ctr, tag=("final", rnd, b))
            ut.add(ze, early, xb, qb, ctr, tag=("exit", rnd, b))
            if o.final.tokens == final.emitted():
                # K rows the step kept at layer 32 (pending + accepted drafts) vs the oracle's
                kref = osess[b].cache.k[31][:, ctx:ctx + final.accepted + 1, :].transpose(1, 0, 2)
                kref = kref.reshape(-1, mc.d_model)
                kg = (k_rows.astype(np.uint32) << 16).view(np.float32)
                assert np.abs(kg - kref).max() <= 2e-2 * np.abs(kref).max()
                assert o.new_len == final.new_len
                opend[b] = o.final.tokens[-1]
                nxt.append(b)
        live = nxt
    report = dict(final=tf.asdict(), exit=te.asdict(), level_u=ut.asdict(), max_rel_logit_err=float(max(errs)),
                  config="C2: Llama2-7B shape, B=1 per submit, ctx 512, gamma 4, exit 16, stochastic, "
                         f"{N_SESS} sessions x {ROUNDS} rounds")
    print(tf.report(), "|", te.report(), "|", ut.report(), "| max rel logit err", max(errs))
    save_report("c2_full_level_e", report)
    assert max(errs) < 2e-2
    assert not tf.hard_mismatch and not te.hard_mismatch and not ut.hard_mismatch
    assert tf.decisions_safe + te.decisions_safe >= 20
    assert ut.checked >= 0.8 * ut.n


@pytest.mark.parametrize("greedy", [False, True], ids=["stochastic", "greedy"])
def test_c2_level_u_calibrated_drafts(svlib, greedy):
    """Level U at the full C2 shape over bench.py's calibrated drafts (alpha 0.825,
    every acceptance length occurs): 16 rounds on one session, each rewound to ctx
    512 (the stationary bench workload), final and exit results vs the oracle's
    acceptance on the downloaded logits."""
    from bench import Rounds, build_calibrated_drafts
    from paper_2505_21594_b200 import sv
    mc = llama2_7b()
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=1, max_gamma=GAMMA, kv_blocks=10)
    s = eng.open_session(7, 0x5EED0007)
    s.fill_kv(CTX, kv_seed=1007)
    rounds = Rounds()
    pend = [int(wd.prefix_tokens(4, 1, mc.vocab)[0])]
    ut = UTally(f"c2_level_u_{'greedy' if greedy else 'stochastic'}")
    hist = np.zeros(GAMMA + 1, dtype=int)
    for k in range(16):
        x, q = build_calibrated_drafts(sv, eng, [s], pend, CTX, GAMMA, 0.825, mc.vocab, 50 + k, rounds)
        r = rounds.next(s)
        t = eng.submit([sv.Request(s, r, pend[0], x[0], None if greedy else torch.from_numpy(q[0]).cuda())],
                       exit_layer=EXIT)
        early = t.wait_early()[0]
        final = t.wait_final()[0]
        zf = t.logits(1, GAMMA).cpu().numpy()[0]
        ze = t.logits(0, GAMMA).cpu().numpy()[0]
        t.release()
        ctr = (0x5EED0007, 7, r)
        ut.add(zf, final, x[0], None if greedy else q[0], ctr, tag=("final", k))
        ut.add(ze, early, x[0], None if greedy else q[0], ctr, tag=("exit", k))
        hist[final.accepted] += 1
        s.rewind(CTX)
    print(ut.report(), "accepted histogram", hist.tolist())
    save_report(ut.name, dict(ut.asdict(), accepted_hist=hist.tolist()))
    assert not ut.hard_mismatch, ut.hard_mismatch[:2]
    assert ut.checked >= 0.8 * ut.n
    if not greedy:
        assert (hist[1:] > 0).sum() >= 2          # the accept path is exercised, not only delta = 0
    s.close()
    eng.close()
