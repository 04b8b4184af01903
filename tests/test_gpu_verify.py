"""GPU end-to-end parity of the verify step against the oracle (level E of
DESIGN.md "Parity contract"): logits within 2e-2 row-max-relative (north star),
decisions identical wherever the oracle's margin exceeds the propagated bound,
KV rollback bit-exact, exit side-effect free, protocol errors."""
import numpy as np
import pytest
import torch

from oracle import accept as oacc
from oracle import gen
from oracle import model as om
from oracle.verify import verify_step
from workload import drafts as wd
from workload import tiny
from workload.configs import ModelCfg

from .gpu_helpers import Tally, UTally, oracle_session, row_rel_err, save_report

pytestmark = pytest.mark.gpu
LOGIT_TOL = 2e-2


def _setup(mc, B, max_gamma=8, use_graphs=True):
    from paper_2505_21594_b200 import sv
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=B, max_gamma=max_gamma, use_graphs=use_graphs)
    return sv, W, eng


def _run_rounds(mc, B, gamma, ctx, exit_layer, greedy, rounds, use_graphs=True, model=None):
    """Run `rounds` verify steps on B sessions through libsv and the oracle in
    lockstep (each side keeps its own cache); returns the tally and errors."""
    sv, W, eng = _setup(mc, B, use_graphs=use_graphs)
    model = model or om.Model(mc, seed=1)
    gs, os_ = [], []
    for b in range(B):
        s = eng.open_session(10 + b, 1000 + b)
        s.fill_kv(ctx, kv_seed=2 + b)
        gs.append(s)
        os_.append(oracle_session(mc, model, 10 + b, 1000 + b, 2 + b, ctx))
    pending = list(wd.prefix_tokens(3, B, mc.vocab))
    tally_f, tally_e = Tally("final"), Tally("exit")
    errs = []
    for rnd in range(1, rounds + 1):
        x, q = wd.timing_drafts(100 + rnd, B, gamma, mc.vocab, s=1.1)
        qd = torch.from_numpy(q).cuda()
        reqs = [sv.Request(gs[b], rnd, pending[b], x[b], None if greedy else qd[b]) for b in range(B)]
        t = eng.submit(reqs, exit_layer=exit_layer)
        early = t.wait_early() if exit_layer else None
        final = t.wait_final()
        zf = t.logits(1, gamma).cpu().numpy()
        ze = t.logits(0, gamma).cpu().numpy() if exit_layer else None
        t.release()
        for b in range(B):
            out = verify_step(model, os_[b], rnd, pending[b], x[b], None if greedy else q[b].astype(np.float64),
                              exit_layer=exit_layer)
            rel, eps = row_rel_err(zf[b], out.final_logits)
            errs.append(rel.max())
            qb = None if greedy else q[b]
            ctr = (1000 + b, 10 + b, rnd)
            tally_f.add(out.final, final[b], out.final_logits, eps, qb, ctr, tag=("final", rnd, b))
            if exit_layer:
                rel_e, eps_e = row_rel_err(ze[b], out.exit_logits)
                errs.append(rel_e.max())
                tally_e.add(out.early, early[b], out.exit_logits, eps_e, qb, ctr, tag=("exit", rnd, b))
            assert gs[b].length == final[b].new_len
            if out.final.status == oacc.OK and out.final.tokens == final[b].emitted():
                assert final[b].new_len == out.new_len
                pending[b] = final[b].emitted()[-1]
            else:
                pending[b] = None       # the two sides diverged (counted above): stop
        if any(p is None for p in pending):
            break
    for s in gs:
        s.close()
    eng.close()
    return tally_f, tally_e, np.array(errs)


@pytest.mark.parametrize("greedy", [True, False], ids=["greedy", "stochastic"])
@pytest.mark.parametrize("ctx", [64, 59])
def test_tiny_end_to_end(svlib, greedy, ctx):
    """configs[0]: 2 layers, d=128, 4 heads, V=512, ctx 64 (or 59 = 64 - G), gamma=4,
    batch 1, early exit at layer 1."""
    tf, te, errs = _run_rounds(tiny(), 1, 4, ctx, 1, greedy, rounds=4)
    print("final:", tf.report(), "| exit:", te.report(), "| max rel logit err", errs.max())
    save_report(f"tiny_e2e_{'greedy' if greedy else 'stochastic'}_ctx{ctx}",
                dict(final=tf.asdict(), exit=te.asdict(), max_rel_logit_err=float(errs.max())))
    assert errs.max() < LOGIT_TOL
    assert not tf.hard_mismatch and not te.hard_mismatch
    assert tf.checked >= 0.75 * tf.n and te.checked >= 0.75 * te.n


@pytest.mark.parametrize("gamma", [1, 3, 8])
def test_tiny_batched_gamma_sweep(svlib, gamma):
    tf, te, errs = _run_rounds(tiny(), 5, gamma, 37, 2, False, rounds=2)
    print("final:", tf.report(), "| exit:", te.report(), "| max rel logit err", errs.max())
    assert errs.max() < LOGIT_TOL
    assert not tf.hard_mismatch and not te.hard_mismatch
    # long drafts put more decisions on a result's path, so fewer results clear every bound
    assert tf.checked >= 0.5 * tf.n and te.checked >= 0.5 * te.n


def test_tiny_large_batch(svlib):
    """B = 60 requests (M = 300 query rows): the 256-token GEMM tile with two token
    tiles, the batched attention grid and 60 acceptance instances (configs[3]-style
    batching at the tiny shape)."""
    tf, te, errs = _run_rounds(tiny(), 60, 4, 40, 1, False, rounds=2)
    print("final:", tf.report(), "| exit:", te.report(), "| max rel logit err", errs.max())
    save_report("tiny_large_batch", dict(final=tf.asdict(), exit=te.asdict(), max_rel_logit_err=float(errs.max())))
    assert errs.max() < LOGIT_TOL
    assert not tf.hard_mismatch and not te.hard_mismatch
    assert tf.checked >= 0.75 * tf.n and te.checked >= 0.75 * te.n


@pytest.mark.parametrize("shape", ["tiny", "7b_width"])
def test_tiny_no_graphs_matches_graphs(svlib, shape):
    """Graph replay and direct launches produce bitwise-identical results
    (the 7B-width case covers the tensor-core attention with cluster merges)."""
    mc = tiny() if shape == "tiny" else ModelCfg(n_layers=2, d_model=4096, n_heads=32, d_ff=11008,
                                                  vocab=32000, max_ctx=512)
    res = []
    for ug in (True, False):
        sv, W, eng = _setup(mc, 2, use_graphs=ug)
        ss = [eng.open_session(1 + b, 7 + b) for b in range(2)]
        for b, s in enumerate(ss):
            s.fill_kv(40 if shape == "tiny" else 300, kv_seed=5 + b)
        x, q = wd.timing_drafts(9, 2, 4, mc.vocab, s=1.1)
        qd = torch.from_numpy(q).cuda()
        t = eng.submit([sv.Request(ss[b], 1, 3, x[b], qd[b]) for b in range(2)], exit_layer=1)
        t.wait_early()
        f = t.wait_final()
        res.append(([r.asdict() for r in f], t.logits(1, 4).cpu().numpy()))
        t.release()
        eng.close()
    assert res[0][0] == res[1][0]
    assert np.array_equal(res[0][1], res[1][1])


def test_exit_is_side_effect_free(svlib):
    """PAPER.md:177 'all tokens are verified at the final exit': final logits and
    results are bitwise identical with the early exit on (any layer) or off."""
    mc = tiny()
    sv, W, eng = _setup(mc, 1)
    outs = []
    for exit_layer in (0, 1, 2):
        s = eng.open_session(1, 9)
        s.fill_kv(50, kv_seed=3)
        x, q = wd.timing_drafts(4, 1, 4, mc.vocab, s=1.1)
        t = eng.submit([sv.Request(s, 1, 5, x[0], torch.from_numpy(q[0]).cuda())], exit_layer=exit_layer)
        e = t.wait_early() if exit_layer else None
        f = t.wait_final()
        outs.append((f[0].asdict(), t.logits(1, 4).cpu().numpy(), e))
        t.release()
        s.close()
    assert outs[0][0] == outs[1][0] == outs[2][0]
    assert np.array_equal(outs[0][1], outs[1][1]) and np.array_equal(outs[0][1], outs[2][1])
    # exit at the last layer == final (north star pin), bitwise
    e2 = outs[2][2][0].asdict()
    f2 = outs[2][0]
    for k in ("accepted", "tokens", "score", "next_prob", "status"):
        assert e2[k] == f2[k], k
    eng.close()


@pytest.mark.parametrize("shape", ["tiny", "7b_width"])
def test_rollback_bit_exact(svlib, shape):
    """DESIGN.md R22: (i) rows [0, ctx) byte-identical across a step; (ii) two steps
    that differ only in the rejected suffix leave byte-identical visible caches and
    byte-identical next steps; (iv) length == ctx + 1 + delta.  The 7B-width case
    (2 layers, ctx 300, one request) runs split-K GEMMs and split-KV attention."""
    if shape == "tiny":
        mc, ctx = tiny(), 30
    else:
        mc, ctx = ModelCfg(n_layers=2, d_model=4096, n_heads=32, d_ff=11008, vocab=32000, max_ctx=512), 300
    sv, W, eng = _setup(mc, 1)
    model = om.Model(mc, seed=1)
    # the target's greedy continuation from the oracle (an input, not a GPU value)
    osess = oracle_session(mc, model, 1, 1, 4, ctx)
    for pend in range(7, 40):        # a pending token whose greedy successor has a clear top-2 gap
        z, _, _ = om.forward(model, osess.cache.copy(), [pend])
        if oacc.top2_gap(z[0]) > 0.2:
            break
    a1 = int(np.argmax(z[0]))
    final_states = []
    for suffix in ([3, 3, 3], [9, 100, 200]):
        s = eng.open_session(1, 1)
        s.fill_kv(ctx, kv_seed=4)
        k0, v0 = s.kv_rows(0, 0, ctx)
        drafts = [a1] + [(a1 + 1 + suffix[0]) % mc.vocab] + suffix[1:]
        _, f = eng.verify([sv.Request(s, 1, pend, drafts)], exit_layer=0)
        assert f[0].accepted == 1 and s.length == ctx + 1 + 1
        k1, v1 = s.kv_rows(0, 0, ctx)
        assert np.array_equal(k0, k1) and np.array_equal(v0, v1)
        vis = [s.kv_rows(l, 0, s.length) for l in range(mc.n_layers)]
        nxt = f[0].emitted()[-1]
        _, f2 = eng.verify([sv.Request(s, 2, nxt, [1, 2, 3, 4])], exit_layer=0)
        final_states.append((vis, f[0].asdict(), f2[0].asdict(),
                             [s.kv_rows(l, 0, s.length) for l in range(mc.n_layers)]))
        s.close()
    A, B = final_states
    for l in range(mc.n_layers):
        assert np.array_equal(A[0][l][0], B[0][l][0]) and np.array_equal(A[0][l][1], B[0][l][1])
        assert np.array_equal(A[3][l][0], B[3][l][0])
    assert A[1]["tokens"] == B[1]["tokens"]
    assert A[2] == B[2]
    eng.close()


@pytest.mark.parametrize("shape", ["tiny", "7b_width"])
def test_poisoned_kv_tail_is_invisible(svlib, shape):
    """DESIGN.md R22 (iii): KV slots at or beyond the cached length hold arbitrary
    bits (here all-NaN bf16 0xFFFF) without changing a step: results and logits are
    bitwise equal to a run on a zeroed pool."""
    mc = tiny() if shape == "tiny" else ModelCfg(n_layers=2, d_model=4096, n_heads=32, d_ff=11008,
                                                  vocab=32000, max_ctx=512)
    from paper_2505_21594_b200 import sv
    W = sv.Weights(mc, seed=1)
    outs = []
    for fill in (0, 255):
        eng = sv.Engine(mc, W, max_batch=2, max_gamma=8)
        eng.kv_pool.fill_(fill)
        ss = [eng.open_session(1 + b, 7 + b) for b in range(2)]
        for b, s in enumerate(ss):
            s.fill_kv(37 + 50 * b, kv_seed=5 + b)
        x, q = wd.timing_drafts(9, 2, 4, mc.vocab, s=1.1)
        qd = torch.from_numpy(q).cuda()
        t = eng.submit([sv.Request(ss[b], 1, 3, x[b], qd[b]) for b in range(2)], exit_layer=1)
        t.wait_early()
        f = t.wait_final()
        z = t.logits(1, 4).cpu().numpy()
        outs.append(([r.asdict() for r in f], z))
        t.release()
        eng.close()
    assert np.isfinite(outs[1][1]).all()
    assert outs[0][0] == outs[1][0]
    assert np.array_equal(outs[0][1], outs[1][1])


def test_protocol_errors(svlib):
    mc = tiny()
    sv, W, eng = _setup(mc, 2)
    s = eng.open_session(1, 1)
    s.fill_kv(20, kv_seed=1)
    _, f = eng.verify([sv.Request(s, 5, 1, [1, 2, 3, 4])])           # round 5 is not 0 + 1
    assert f[0].status == sv.SV_E_PROTOCOL and s.length == 20
    _, f = eng.verify([sv.Request(s, 1, 1, [1, 2, 3, 4], prefix_len=7)])
    assert f[0].status == sv.SV_E_PROTOCOL and s.length == 20
    q = np.full((4, mc.vocab), 1.0 / mc.vocab, dtype=np.float32)
    q[3, 4] = 0.0
    _, f = eng.verify([sv.Request(s, 1, 1, [1, 2, 3, 4], q)])          # host probs, q_4(x_4) = 0
    assert f[0].status == sv.SV_E_PROTOCOL and s.length == 20
    _, f = eng.verify([sv.Request(s, 1, 1, [1, 2, 3, 4])])
    assert f[0].status == sv.SV_OK and s.length == 20 + 1 + f[0].accepted
    with pytest.raises(sv.SvError):
        eng.verify([sv.Request(s, 2, 1, [1, 2, 3, mc.vocab])])        # token out of range
    s.close()
    eng.close()


def test_host_probs_equal_device_probs(svlib):
    mc = tiny()
    sv, W, eng = _setup(mc, 1)
    out = []
    for host in (True, False):
        s = eng.open_session(3, 3)
        s.fill_kv(20, kv_seed=1)
        x, q = wd.timing_drafts(8, 1, 4, mc.vocab, s=1.1)
        p = q[0] if host else torch.from_numpy(q[0]).cuda()
        _, f = eng.verify([sv.Request(s, 1, 2, x[0], p)])
        out.append(f[0].asdict())
        s.close()
    assert out[0] == out[1]
    eng.close()


def test_7b_width_two_layers(svlib):
    """Llama2-7B layer shapes (d=4096, 32 heads, F=11008, V=32000) with 2 layers,
    batch 2, ctx 200: logits and decisions vs the fp64 oracle."""
    mc = ModelCfg(n_layers=2, d_model=4096, n_heads=32, d_ff=11008, vocab=32000, max_ctx=512)
    tf, te, errs = _run_rounds(mc, 2, 4, 200, 1, False, rounds=2)
    print("final:", tf.report(), "| exit:", te.report(), "| max rel logit err", errs.max())
    assert errs.max() < LOGIT_TOL
    assert not tf.hard_mismatch and not te.hard_mismatch


def _batch_7b_against_oracle(name, B, gamma, ctx, sampled, seeds=(60, 70, 80, 33)):
    """B requests at the Llama2-7B layer widths (2 layers), one stochastic round with an
    early exit at layer 1: level U on every request, level E on the sampled ones."""
    from paper_2505_21594_b200 import sv
    mc = ModelCfg(n_layers=2, d_model=4096, n_heads=32, d_ff=11008, vocab=32000, max_ctx=(ctx + 40 + 63) // 64 * 64)
    s0, k0, kv0, dseed = seeds
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=B, max_gamma=gamma)
    model = om.Model(mc, seed=1)
    ss = []
    for b in range(B):
        s = eng.open_session(s0 + b, k0 + b)
        s.fill_kv(ctx, kv_seed=kv0 + b)
        ss.append(s)
    x, q = wd.timing_drafts(dseed, B, gamma, mc.vocab, s=1.1)
    qd = torch.from_numpy(q).cuda()
    t = eng.submit([sv.Request(ss[b], 1, 5 + b, x[b], qd[b]) for b in range(B)], exit_layer=1)
    early = t.wait_early()
    final = t.wait_final()
    zf = t.logits(1, gamma).cpu().numpy()
    ze = t.logits(0, gamma).cpu().numpy()
    t.release()
    tally = Tally(name)
    ut = UTally(name + " level U")
    for b in range(B):
        ut.add(zf[b], final[b], x[b], q[b], (k0 + b, s0 + b, 1), tag=("final", b))
        ut.add(ze[b], early[b], x[b], q[b], (k0 + b, s0 + b, 1), tag=("exit", b))
    for b in sampled:
        osess = oracle_session(mc, model, s0 + b, k0 + b, kv0 + b, ctx)
        out = verify_step(model, osess, 1, 5 + b, x[b], q[b].astype(np.float64), exit_layer=1)
        rel, eps = row_rel_err(zf[b], out.final_logits)
        rel_e, eps_e = row_rel_err(ze[b], out.exit_logits)
        assert rel.max() < LOGIT_TOL and rel_e.max() < LOGIT_TOL
        tally.add(out.final, final[b], out.final_logits, eps, q[b], (k0 + b, s0 + b, 1), tag=("final", b))
        tally.add(out.early, early[b], out.exit_logits, eps_e, q[b], (k0 + b, s0 + b, 1), tag=("exit", b))
        assert ss[b].length == final[b].new_len
    print(tally.report(), "|", ut.report())
    save_report(name, dict(level_e=tally.asdict(), level_u=ut.asdict()))
    assert not tally.hard_mismatch and not ut.hard_mismatch
    assert ut.checked >= 0.8 * ut.n and tally.checked >= 2
    for s in ss:
        s.close()
    eng.close()
    return zf, ze


def test_7b_width_c5_batch(svlib):
    """configs[4]-shaped batch at the Llama2-7B layer shapes (2 layers): B = 16
    requests x (gamma + 1) = 80 query rows -> the persistent GEMM (80-token tiles,
    stream-K for QKV / O / down / gate-up: split tiles reduced by all their
    contributors) and the attention ring, in bench.py's launch configuration; sampled
    requests {0, 7, 15} against the fp64 oracle, one stochastic round."""
    _batch_7b_against_oracle("7b_width_c5_batch", 16, 4, 600, (0, 7, 15))


@pytest.mark.parametrize("sk_fill", [None, "1.01"])
def test_7b_width_c4_shard_batch(svlib, sk_fill, monkeypatch):
    """The per-GPU shard of configs[3] on 8 GPUs: B = 32 requests x 5 = 160 query rows
    (160-token persistent tiles; stream-K for O / down / gate-up by default, and for
    every GEMM with SV_SK_FILL=1.01), sampled requests {0, 17, 31} against the fp64
    oracle; the two stream-K settings give logits within the same bound."""
    if sk_fill:
        monkeypatch.setenv("SV_SK_FILL", sk_fill)
    _batch_7b_against_oracle("7b_width_c4_shard_batch" + ("_sk" if sk_fill else ""), 32, 4, 300, (0, 17, 31),
                             seeds=(500, 600, 700, 35))


def test_7b_width_c4_batch(svlib):
    """configs[3]-shaped batch on one GPU at the Llama2-7B layer widths (2 layers):
    B = 256 requests x 5 = 1280 query rows (persistent 128 x 256 GEMM tiles, five
    token tiles, the batched attention grid), ctx 1024; sampled requests
    {0, 131, 255} against the fp64 oracle, one stochastic round with an early exit."""
    from paper_2505_21594_b200 import sv
    mc = ModelCfg(n_layers=2, d_model=4096, n_heads=32, d_ff=11008, vocab=32000, max_ctx=1088)
    B, gamma, ctx = 256, 4, 1024
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=B, max_gamma=gamma, kv_blocks=B * 17)
    model = om.Model(mc, seed=1)
    ss = []
    for b in range(B):
        s = eng.open_session(100 + b, 300 + b)
        s.fill_kv(ctx, kv_seed=400 + b)
        ss.append(s)
    x, q = wd.timing_drafts(34, B, gamma, mc.vocab, s=1.1)
    qd = torch.from_numpy(q).cuda()
    t = eng.submit([sv.Request(ss[b], 1, (7 * b) % mc.vocab, x[b], qd[b]) for b in range(B)], exit_layer=1)
    early = t.wait_early()
    final = t.wait_final()
    zf = t.logits(1, gamma).cpu().numpy()
    ze = t.logits(0, gamma).cpu().numpy()
    t.release()
    tally = Tally("7b_width_c4_batch")
    ut = UTally("7b_width_c4_batch level U")
    for b in range(0, B, 4):
        ut.add(zf[b], final[b], x[b], q[b], (300 + b, 100 + b, 1), tag=("final", b))
        ut.add(ze[b], early[b], x[b], q[b], (300 + b, 100 + b, 1), tag=("exit", b))
    for b in (0, 131, 255):
        osess = oracle_session(mc, model, 100 + b, 300 + b, 400 + b, ctx)
        out = verify_step(model, osess, 1, (7 * b) % mc.vocab, x[b], q[b].astype(np.float64), exit_layer=1)
        rel, eps = row_rel_err(zf[b], out.final_logits)
        rel_e, eps_e = row_rel_err(ze[b], out.exit_logits)
        assert rel.max() < LOGIT_TOL and rel_e.max() < LOGIT_TOL
        tally.add(out.final, final[b], out.final_logits, eps, q[b], (300 + b, 100 + b, 1), tag=("final", b))
        tally.add(out.early, early[b], out.exit_logits, eps_e, q[b], (300 + b, 100 + b, 1), tag=("exit", b))
        assert ss[b].length == final[b].new_len
    print(tally.report(), "|", ut.report())
    save_report("7b_width_c4_batch", dict(level_e=tally.asdict(), level_u=ut.asdict()))
    assert not tally.hard_mismatch and not ut.hard_mismatch
    assert ut.checked >= 0.8 * ut.n and tally.checked >= 2
    for s in ss:
        s.close()
    eng.close()
