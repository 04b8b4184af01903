"""The C-ABI boundary beyond the async submit path:

- sv_verify, the north star's synchronous verify(draft_tokens, draft_probs, kv),
  called through ctypes, equals the async submit path bit for bit and the oracle;
- sv_debug_forward (non-committing forward): KV-incremental verify == full causal
  recompute of prefix + block (the oracle's invariant, now on the GPU), and the
  call leaves the session untouched;
- exit-ready latency (sv_ticket_timing) at the full C2 shape: the early exit's
  result reaches the host before the final result exists (PAPER.md:145-151,
  Alg-S :1103-1106), and the device stamps order exit < final;
- the per-launch timeline of a graph-replayed step (sv_debug_trace_*) covers
  every launch and does not change any result."""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import accept as oacc
from oracle import model as om
from oracle.verify import verify_step
from workload import drafts as wd
from workload import llama2_7b, tiny
from workload.configs import ModelCfg

from .gpu_helpers import oracle_session, row_rel_err

pytestmark = pytest.mark.gpu


def _shape(name):
    if name == "tiny":
        return tiny()
    return ModelCfg(n_layers=2, d_model=4096, n_heads=32, d_ff=11008, vocab=32000, max_ctx=512)


def test_sync_sv_verify_through_ctypes(svlib):
    from paper_2505_21594_b200 import sv
    mc = tiny()
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=1, max_gamma=4)
    x, q = wd.timing_drafts(12, 1, 4, mc.vocab, s=1.1)
    qd = torch.from_numpy(q[0]).cuda()
    outs = []
    for mode in ("sync", "async"):
        s = eng.open_session(5, 55)
        s.fill_kv(45, kv_seed=6)
        req = sv.Request(s, 1, 9, x[0], qd)
        if mode == "sync":
            cr = req.to_c()
            early, final = sv.sv_exit_result(), sv.sv_exit_result()
            sv.check(svlib.sv_verify(s.h, C.byref(cr), 1, C.byref(early), C.byref(final)))
        else:
            t = eng.submit([req], exit_layer=1)
            early, final = t.wait_early()[0], t.wait_final()[0]
            t.release()
        outs.append((early.asdict(), final.asdict(), s.length))
        s.close()
    assert outs[0] == outs[1]
    model = om.Model(mc, seed=1)
    ref = verify_step(model, oracle_session(mc, model, 5, 55, 6, 45), 1, 9, x[0], q[0].astype(np.float64),
                      exit_layer=1)
    if ref.final.min_margin > 1e-2:
        assert outs[0][1]["tokens"] == ref.final.tokens and outs[0][2] == ref.new_len
    # the sync call's argument checks
    s = eng.open_session(6, 1)
    bad = sv.Request(s, 2, 9, x[0], qd).to_c()          # round 2 is not the successor of 0
    early, final = sv.sv_exit_result(), sv.sv_exit_result()
    st = svlib.sv_verify(s.h, C.byref(bad), 1, C.byref(early), C.byref(final))
    assert st == sv.SV_OK and final.status == sv.SV_E_PROTOCOL and s.length == 0
    s.close()
    eng.close()


@pytest.mark.parametrize("shape", ["tiny", "7b_width"])
def test_debug_forward_incremental_equals_recompute(svlib, shape):
    """Session A: prompt P prefilled, then one verify block [pending, x_1..x_4].
    Session B: empty, sv_debug_forward(P + block) in one pass.  The block's logits
    agree (different GEMM / attention tilings: within the logit tolerance, argmax
    equal where the gap is clear), and both match the oracle's full recompute."""
    from paper_2505_21594_b200 import sv
    mc = _shape(shape)
    n = 40 if shape == "tiny" else 200
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=1, max_gamma=4, max_prefill=n + 5)
    rng = np.random.default_rng(3)
    prompt = rng.integers(0, mc.vocab, size=n)
    x = rng.integers(0, mc.vocab, size=4)
    a = eng.open_session(1, 11)
    res = a.prefill(prompt)
    pend = res.emitted()[-1]
    t = eng.submit([sv.Request(a, res.round_id + 1, pend, x)], exit_layer=0)
    t.wait_final()
    z_inc = t.logits(1, 4).cpu().numpy()[0]
    t.release()
    b = eng.open_session(2, 11)
    full = np.concatenate([prompt, [pend], x])
    z_full = b.debug_forward(full).cpu().numpy()
    assert b.length == 0                                # nothing committed
    z_blk = z_full[n:]
    rel, eps = row_rel_err(z_blk, z_inc)
    print("incremental vs recompute: max rel", rel.max(), "eps", eps.max())
    assert rel.max() < 1e-2
    for r in range(5):
        if oacc.top2_gap(z_inc[r]) > 2 * eps[r]:
            assert np.argmax(z_blk[r]) == np.argmax(z_inc[r])
    # the oracle's full causal recompute of the same sequence
    model = om.Model(mc, seed=1)
    zr, _, _ = om.forward(model, om.KVCache(mc), full)
    rel_o, _ = row_rel_err(z_full, zr)
    assert rel_o.max() < 2e-2
    # the non-committing pass left session B usable and unchanged: its prefill +
    # verify now equals session A's bit for bit
    res_b = b.prefill(prompt)
    assert res_b.emitted() == res.emitted()
    t = eng.submit([sv.Request(b, res_b.round_id + 1, pend, x)], exit_layer=0)
    t.wait_final()
    assert np.array_equal(t.logits(1, 4).cpu().numpy()[0], z_inc)
    t.release()
    a.close()
    b.close()
    eng.close()


def test_exit_ready_before_final_c2(svlib):
    """C2 (32 layers, exit at 16): the early result is on the host while the final
    is still running, and the device stamps put the exit near l_e / L of the step."""
    from paper_2505_21594_b200 import sv
    mc = llama2_7b()
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=1, max_gamma=4, kv_blocks=12)
    s = eng.open_session(1, 3)
    s.fill_kv(512, kv_seed=4)
    x, q = wd.timing_drafts(5, 1, 4, mc.vocab)
    qd = torch.from_numpy(q[0]).cuda()
    before, fr = 0, []
    for r in range(12):
        s.rewind(512)
        t = eng.submit([sv.Request(s, r + 1, 7, x[0], qd)], exit_layer=16)
        t.wait_early()
        before += not t.final_ready()
        t.wait_final()
        tm = t.timing()
        t.release()
        if r >= 2:
            fr.append(tm["exit_dev_ms"][0] / tm["final_dev_ms"])
            assert 0 < tm["exit_dev_ms"][0] < tm["final_dev_ms"]
            assert 0 < tm["exit_host_ms"][0] < tm["final_host_ms"]
    print("early before final in", before, "of 12 steps; exit/final device time", np.median(fr))
    assert before >= 10
    assert 0.35 < np.median(fr) < 0.7
    # all exits streamed: a strict prefix of the 31 exits is observed before the final
    seen = set()
    s.rewind(512)
    t = eng.submit_exits([sv.Request(s, 13, 7, x[0], qd)], list(range(1, 32)))
    while True:
        k = t.exits_ready()
        seen.add(k)
        if k == 31:
            break
    t.wait_final()
    tm = t.timing()
    t.release()
    assert any(0 < k < 31 for k in seen), seen
    dev = tm["exit_dev_ms"]
    assert all(dev[i] <= dev[i + 1] for i in range(30)) and dev[-1] <= tm["final_dev_ms"]
    s.close()
    eng.close()


def test_trace_timeline_covers_the_step(svlib):
    from paper_2505_21594_b200 import sv
    mc = _shape("7b_width")
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=1, max_gamma=4)
    s = eng.open_session(1, 3)
    s.fill_kv(300, kv_seed=4)
    x, q = wd.timing_drafts(5, 1, 4, mc.vocab)
    qd = torch.from_numpy(q[0]).cuda()
    outs = []
    for r, traced in enumerate((False, True, False)):
        s.rewind(300)
        if traced:
            eng.trace_next()
        t = eng.submit([sv.Request(s, r + 1, 7, x[0], qd)], exit_layer=1)
        t.wait_early()
        f = t.wait_final()[0]
        outs.append((f.asdict()["tokens"], t.logits(1, 4).cpu().numpy()))
        t.release()
        if traced:
            tr = eng.trace_read()
    assert np.array_equal(outs[0][1], outs[1][1]) and outs[0][0] == outs[1][0]
    kinds = [r["kind"] for r in tr]
    # embed, per layer (QKV, attention, O, gate/up, down), exit LM + accept, final LM + accept
    assert kinds[0] == "embed" and kinds.count("attention") == 2 and kinds.count("gemm_qkv") == 2
    assert "gemm_lm_exit" in kinds and "accept_final" in kinds
    assert all(r["end_us"] >= r["start_us"] >= 0 for r in tr)
    assert [r["stream"] for r in tr if r["kind"] in ("gemm_lm_exit", "accept_exit")] == [1, 1]
    s.close()
    eng.close()
