"""Prefill through the C ABI against the oracle: the
prompt's K/V rows (bf16 vs fp64, row-max relative), the next-token decision
(margin-binned), and verify rounds on top of the prefilled cache (logits within
2e-2, decisions) — the prompt is split into query blocks of 16 rows (attn3,
head_dim 128) or 8 rows (attn_kernel) with a ragged last block, and a second
prefill continues an existing cache (rows written before the call are the only
ones loaded before griddepcontrol.wait)."""
import numpy as np
import pytest
import torch

from oracle import model as om
from oracle.verify import Session as OSession
from oracle.verify import prefill_step, verify_step
from workload import drafts as wd
from workload import tiny
from workload.configs import ModelCfg

from .gpu_helpers import Tally, row_rel_err, save_report

pytestmark = pytest.mark.gpu


def _bf16_to_f64(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("shape", ["tiny", "7b_width"])
@pytest.mark.parametrize("sample", [False, True], ids=["greedy", "sampled"])
def test_prefill_then_verify(svlib, shape, sample):
    from paper_2505_21594_b200 import sv
    if shape == "tiny":
        mc, chunks = tiny(), [37, 13]
    else:
        mc, chunks = ModelCfg(n_layers=2, d_model=4096, n_heads=32, d_ff=11008, vocab=32000, max_ctx=512), [300, 45]
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=1, max_gamma=4, max_prefill=max(chunks))
    model = om.Model(mc, seed=1)
    rng = np.random.default_rng(5)
    prompt = rng.integers(0, mc.vocab, size=sum(chunks))
    s = eng.open_session(3, 77)
    osess = OSession(3, 77, om.KVCache(mc))
    tally = Tally(f"prefill_{shape}_{'sampled' if sample else 'greedy'}")
    off = 0
    for c in chunks:
        res = s.prefill(prompt[off:off + c], sample=sample)
        ores, _ = prefill_step(model, osess, osess.last_round + 1, prompt[off:off + c], sample=sample)
        off += c
        assert res.status == 0 and res.accepted == 0 and s.length == off == osess.cache.length
        tally.add_fixed(ores, res, 1e-2 if shape == "tiny" else 0.25, tag=("prefill", off))
    # the prompt's K/V rows, every layer
    for l in range(mc.n_layers):
        k, v = s.kv_rows(l, 0, off)
        for got, ref in ((k, osess.cache.k[l]), (v, osess.cache.v[l])):
            ref2 = ref.transpose(1, 0, 2).reshape(off, -1)
            err = np.abs(_bf16_to_f64(got) - ref2).max() / np.abs(ref2).max()
            assert err < 2e-2, (l, err)
    # verify rounds on top of the prefilled cache
    pending = int(res.emitted()[-1]) if ores.tokens == res.emitted() else int(ores.tokens[-1])
    for rnd in range(2):
        x, q = wd.timing_drafts(50 + rnd, 1, 4, mc.vocab, s=1.1)
        r_id = osess.last_round + 1
        t = eng.submit([sv.Request(s, r_id, pending, x[0], torch.from_numpy(q[0]).cuda())], exit_layer=0)
        f = t.wait_final()[0]
        zf = t.logits(1, 4).cpu().numpy()[0]
        t.release()
        out = verify_step(model, osess, r_id, pending, x[0], q[0].astype(np.float64))
        rel, eps = row_rel_err(zf, out.final_logits)
        assert rel.max() < 2e-2
        tally.add(out.final, f, out.final_logits, eps, q[0], (77, 3, r_id), tag=("verify", rnd))
        if out.final.tokens != f.emitted():
            break
        pending = f.emitted()[-1]
    print(tally.report())
    save_report(tally.name, tally.asdict())
    assert not tally.hard_mismatch
    s.close()
    eng.close()


def test_prefill_capacity(svlib):
    from paper_2505_21594_b200 import sv
    mc = tiny()
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=1, max_gamma=4, max_prefill=16)
    s = eng.open_session(1, 1)
    with pytest.raises(sv.SvError):
        s.prefill(np.arange(17) % mc.vocab)
    assert s.length == 0
    s.close()
    eng.close()
