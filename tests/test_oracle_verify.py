"""Pins for oracle/verify.py (one verify step on a session).

- l_e = L: the early-exit result equals the final result exactly (north star).
- Rollback (R22): new length = ctx + 1 + delta; rows [0, ctx) unchanged;
  the rolled-back cache equals a full causal recompute of prefix + [pending,
  x_1..x_delta] (invariant: KV-incremental + rollback == recompute).
- Protocol errors leave the session unchanged.
- Multi-round greedy decoding with an oracle-perfect drafter accepts everything.
"""
import numpy as np

from oracle import accept as acc
from oracle import model as om
from oracle.verify import Session, verify_step
from workload import tiny
from workload.drafts import timing_drafts


def _session(cfg, m, ctx=20, seed=4, sid=1, prefill=True):
    cache = om.KVCache(cfg)
    if prefill:
        toks = np.random.default_rng(sid).integers(0, cfg.vocab, size=ctx)
        om.forward(m, cache, toks)
    else:
        cache = om.KVCache.synthetic(cfg, 2, ctx)
    return Session(sid, seed, cache)


def test_exit_at_last_layer_equals_final():
    cfg = tiny()
    m = om.Model(cfg, 1)
    for mode in ("greedy", "stochastic"):
        s = _session(cfg, m)
        x, q = timing_drafts(3, 1, 4, cfg.vocab)
        out = verify_step(m, s, 1, 7, x[0], q[0] if mode == "stochastic" else None,
                          exit_layer=cfg.n_layers)
        assert out.early.accepted == out.final.accepted
        assert out.early.tokens == out.final.tokens
        assert out.early.score == out.final.score
        assert np.array_equal(out.exit_logits, out.final_logits)


def test_rollback_equals_recompute():
    cfg = tiny()
    m = om.Model(cfg, 1)
    s = _session(cfg, m, ctx=15)
    prefix_k = [k.copy() for k in s.cache.k]
    # drafts: the target's own greedy continuation for 2 tokens then a wrong token
    c = s.cache.copy()
    z, _, _ = om.forward(m, c, [9])
    a1 = int(np.argmax(z[0]))
    c = s.cache.copy()
    z, _, _ = om.forward(m, c, [9, a1])
    a2 = int(np.argmax(z[1]))
    bad = (a2 + 1) % cfg.vocab
    out = verify_step(m, s, 1, 9, [a1, a2, bad, 3], None, exit_layer=1)
    assert out.final.accepted == 2 and out.final.tokens[:2] == [a1, a2]
    assert out.new_len == 15 + 1 + 2 and s.cache.length == 18
    for l in range(cfg.n_layers):
        assert np.array_equal(s.cache.k[l][:, :15], prefix_k[l])
    # full recompute of prefix + [pending, a1, a2]
    toks = np.random.default_rng(1).integers(0, cfg.vocab, size=15)
    full = om.KVCache(cfg)
    om.forward(m, full, np.concatenate([toks, [9, a1, a2]]))
    for l in range(cfg.n_layers):
        assert np.allclose(s.cache.k[l], full.k[l], rtol=0, atol=1e-12)
        assert np.allclose(s.cache.v[l], full.v[l], rtol=0, atol=1e-12)


def test_greedy_perfect_drafter_multi_round():
    cfg = tiny()
    m = om.Model(cfg, 1)
    s = _session(cfg, m, ctx=10)
    pending = 3
    for rnd in range(1, 4):
        # perfect drafter: the target's greedy continuation
        c = s.cache.copy()
        seq = [pending]
        for _ in range(4):
            z, _, _ = om.forward(m, c.copy(), seq)
            seq.append(int(np.argmax(z[-1])))
        out = verify_step(m, s, rnd, pending, seq[1:], None, exit_layer=1)
        assert out.final.accepted == 4
        pending = out.final.tokens[-1]
    assert s.cache.length == 10 + 3 * 5


def test_protocol_errors_leave_session_unchanged():
    cfg = tiny()
    m = om.Model(cfg, 1)
    s = _session(cfg, m, ctx=12, prefill=False)
    q = np.full((2, cfg.vocab), 1.0 / cfg.vocab)
    q[1, 5] = 0.0
    out = verify_step(m, s, 1, 1, [2, 5], q, exit_layer=1)
    # x_2 = 5 has q = 0: the whole request is a protocol error, KV not advanced
    assert out.final.status == acc.E_PROTOCOL
    assert s.cache.length == 12 and s.last_round == 0
    bad = verify_step(m, s, 5, 1, [2, 3], None)               # round 5 is not the successor of 0
    assert bad.final.status == acc.E_PROTOCOL and s.cache.length == 12
    ok = verify_step(m, s, 1, 1, [2, 3], None)
    assert ok.final.status == acc.OK and s.cache.length == 12 + 1 + ok.final.accepted


def test_all_exits_match_single_exit_runs():
    """All-exits verify (Alg-S): the exit list gives, for every
    layer, exactly the single-exit result of that layer (same counters, read-only),
    the final result is unchanged by the exits, and the exit at l = L equals it."""
    cfg = tiny().__class__(**{**tiny().__dict__, "n_layers": 4})
    m = om.Model(cfg, 1)
    x, q = timing_drafts(5, 1, 4, cfg.vocab)
    ref = verify_step(m, _session(cfg, m, prefill=False), 1, 7, x[0], q[0])
    out = verify_step(m, _session(cfg, m, prefill=False), 1, 7, x[0], q[0], exit_layers=[1, 2, 3, 4])
    assert [le for le, _, _ in out.exits] == [1, 2, 3, 4]
    assert out.final.tokens == ref.final.tokens and np.array_equal(out.final_logits, ref.final_logits)
    assert out.new_len == ref.new_len
    for le, r, z in out.exits:
        single = verify_step(m, _session(cfg, m, prefill=False), 1, 7, x[0], q[0], exit_layer=le)
        assert np.array_equal(z, single.exit_logits)
        assert r.tokens == single.early.tokens and r.accepted == single.early.accepted
        assert r.score == single.early.score
    le, r, z = out.exits[-1]
    assert np.array_equal(z, out.final_logits) and r.tokens == out.final.tokens


# --------------------------------------------------------------------------------
# prefill_step pinned against HF LlamaForCausalLM float64
# (library routine): the next token of a prompt is HF's last-row argmax, the
# kept K/V rows are HF's cache, a continued prefill equals one pass over the
# whole prompt, and the sampled next token follows softmax of HF's last row.
# --------------------------------------------------------------------------------
import pytest
from scipy import stats

from oracle.verify import prefill_step
from .test_oracle_model import _hf_model


def _hf_run(cfg, m, seq):
    import torch
    hf = _hf_model(cfg, m)
    with torch.no_grad():
        out = hf(torch.from_numpy(np.asarray(seq))[None], use_cache=True)
    return hf, out


def test_prefill_matches_hf_greedy_and_cache():
    cfg = tiny()
    m = om.Model(cfg, 1)
    seq = np.random.default_rng(31).integers(0, cfg.vocab, size=40)
    _, out = _hf_run(cfg, m, seq)
    z_hf = out.logits[0].numpy()
    s = Session(3, 9, om.KVCache(cfg))
    res, zl = prefill_step(m, s, 1, seq)
    assert np.max(np.abs(zl[0] - z_hf[-1])) < 1e-6 * np.max(np.abs(z_hf[-1]))
    assert res.accepted == 0 and res.tokens == [int(np.argmax(z_hf[-1]))]
    assert s.cache.length == 40 and s.last_round == 1
    for l in range(cfg.n_layers):
        k_hf = out.past_key_values.layers[l].keys[0].numpy()      # [H, T, Dh], after RoPE
        v_hf = out.past_key_values.layers[l].values[0].numpy()
        assert np.max(np.abs(s.cache.k[l] - k_hf)) < 1e-6 * np.max(np.abs(k_hf))
        assert np.max(np.abs(s.cache.v[l] - v_hf)) < 1e-6 * np.max(np.abs(v_hf))
    # a continued prefill (25 then 15 tokens) equals the single pass
    s2 = Session(3, 9, om.KVCache(cfg))
    prefill_step(m, s2, 1, seq[:25])
    res2, zl2 = prefill_step(m, s2, 2, seq[25:])
    assert np.max(np.abs(zl2[0] - z_hf[-1])) < 1e-6 * np.max(np.abs(z_hf[-1]))
    assert res2.tokens == res.tokens and s2.cache.length == 40
    with pytest.raises(ValueError):
        prefill_step(m, s2, 7, seq[:3])                             # round 7 is not 2 + 1


def test_prefill_sampled_token_follows_hf_last_row():
    cfg = tiny()
    m = om.Model(cfg, 2)
    seq = np.array([5, 77, 300])
    _, out = _hf_run(cfg, m, seq)
    p = acc.softmax(out.logits[0, -1].numpy())
    N = 3000
    counts = np.zeros(cfg.vocab)
    for r in range(1, N + 1):
        s = Session(4, 11, om.KVCache(cfg), last_round=r - 1)
        res, _ = prefill_step(m, s, r, seq, sample=True)
        assert res.accepted == 0 and len(res.tokens) == 1
        counts[res.tokens[0]] += 1
    big = N * p >= 5
    obs = np.append(counts[big], counts[~big].sum())
    exp = np.append(N * p[big], N * p[~big].sum())
    assert big.sum() >= 3
    assert stats.chisquare(obs, exp).pvalue > 1e-3


def test_verify_steps_equals_per_session_verify_step():
    """verify_steps (one forward over several sessions, layer loop outermost) gives
    every session exactly verify_step's result: same logits bits, same decisions,
    same rolled-back cache; a session with a bad round id is a protocol error and
    does not disturb the others."""
    from oracle.verify import verify_steps
    cfg = tiny()
    m = om.Model(cfg, 1)
    x, q = timing_drafts(5, 3, 4, cfg.vocab)
    ctxs = (20, 33, 7)
    single = []
    for b in range(3):
        s = _session(cfg, m, ctx=ctxs[b], seed=10 + b, sid=b + 1, prefill=False)
        single.append((verify_step(m, s, 1, 3 + b, x[b], q[b], exit_layer=1), s))
    ss = [_session(cfg, m, ctx=ctxs[b], seed=10 + b, sid=b + 1, prefill=False) for b in range(3)]
    bad = _session(cfg, m, ctx=9, seed=3, sid=9, prefill=False)
    outs = verify_steps(m, ss + [bad], [1, 1, 1, 4], [3, 4, 5, 1], list(x) + [x[0]], list(q) + [q[0]],
                        exit_layer=1)
    for (ref, rs), out, s in zip(single, outs, ss):
        assert np.array_equal(ref.final_logits, out.final_logits)
        assert np.array_equal(ref.exit_logits, out.exit_logits)
        assert ref.final == out.final and ref.early == out.early and ref.new_len == out.new_len
        for l in range(cfg.n_layers):
            assert np.array_equal(rs.cache.k[l], s.cache.k[l]) and np.array_equal(rs.cache.v[l], s.cache.v[l])
    assert outs[3].final.status == acc.E_PROTOCOL and bad.cache.length == 9
