"""GPU unit parity: Philox, weight / KV generators (bit-exact), acceptance kernels
on identical fp32 logits (level U of DESIGN.md "Parity contract")."""
import os

import numpy as np
import pytest
import torch

from oracle import accept as oacc
from oracle import gen
from workload import drafts as wd
from workload import tiny
from workload.configs import ModelCfg

from .gpu_helpers import Tally, save_report

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")


def test_philox_kat_on_device(svlib):
    from paper_2505_21594_b200 import sv
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(t, 16) for t in line.split()]
        assert sv.debug_philox(v[:4], v[4:6]) == v[6:]


def _bits(t):
    return t.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.fixture(scope="module")
def tiny_weights(svlib):
    from paper_2505_21594_b200 import sv
    return sv.Weights(tiny(), seed=1)


def test_weights_bit_identical_tiny(tiny_weights):
    mc = tiny()
    W = tiny_weights
    d, F, V = mc.d_model, mc.d_ff, mc.vocab
    sg = gen.sigmas(mc)
    assert np.array_equal(_bits(W.tensor("embed")), gen.gen_bits(1, gen.TID_EMBED, V * d, sg["embed"]).reshape(V, d))
    assert np.array_equal(_bits(W.tensor("lm_head")), gen.gen_bits(1, gen.TID_LM_HEAD, V * d, sg["lm_head"]).reshape(V, d))
    assert np.array_equal(_bits(W.tensor("norm_final")), gen.gen_bits(1, gen.TID_NORM_FINAL, d, 0.1, 1.0))
    for l in range(mc.n_layers):
        t = lambda k: gen.layer_tid(l, k)
        qkv = _bits(W.tensor("qkv", l))
        for s, k in enumerate((gen.WQ, gen.WK, gen.WV)):
            assert np.array_equal(qkv[s * d:(s + 1) * d], gen.gen_bits(1, t(k), d * d, sg["w_in"]).reshape(d, d))
        assert np.array_equal(_bits(W.tensor("o", l)), gen.gen_bits(1, t(gen.WO), d * d, sg["w_out"]).reshape(d, d))
        gu = _bits(W.tensor("gu", l)).reshape(F // 64, 2, 64, d)      # 64-row interleave
        wg = gen.gen_bits(1, t(gen.WG), F * d, sg["w_in"]).reshape(F // 64, 64, d)
        wu = gen.gen_bits(1, t(gen.WU), F * d, sg["w_in"]).reshape(F // 64, 64, d)
        assert np.array_equal(gu[:, 0], wg) and np.array_equal(gu[:, 1], wu)
        assert np.array_equal(_bits(W.tensor("down", l)), gen.gen_bits(1, t(gen.WDOWN), d * F, sg["w_out"]).reshape(d, F))
        assert np.array_equal(_bits(W.tensor("norm_attn", l)), gen.gen_bits(1, t(gen.G_ATTN), d, 0.1, 1.0))
        assert np.array_equal(_bits(W.tensor("norm_mlp", l)), gen.gen_bits(1, t(gen.G_MLP), d, 0.1, 1.0))


def test_kv_fill_bit_identical(svlib, tiny_weights):
    from paper_2505_21594_b200 import sv
    mc = tiny()
    eng = sv.Engine(mc, tiny_weights, max_batch=1, max_gamma=8)
    s = eng.open_session(1, 4)
    s.fill_kv(100, kv_seed=2)
    assert s.length == 100
    for l in range(mc.n_layers):
        k, v = s.kv_rows(l, 0, 100)
        for kv, got in ((0, k), (1, v)):
            ref = gen.gen_bits(2, gen.kv_tid(l, kv), 100 * mc.d_model, 1.0).reshape(100, mc.d_model)
            assert np.array_equal(got, ref)
    s.close()
    eng.close()


def _accept_case(eng, mc, B, gamma, seed, greedy, sessions):
    from paper_2505_21594_b200 import sv
    V = mc.vocab
    logits, x, q = wd.synthetic_accept_case(seed, B, gamma, V)
    zl = torch.from_numpy(logits).cuda()
    qd = torch.from_numpy(q).cuda()
    reqs = []
    for b in range(B):
        reqs.append(sv.Request(sessions[b], 1 + seed % 1000, 0, x[b], None if greedy else qd[b]))
    got = eng.debug_accept(zl, reqs)
    refs = []
    for b in range(B):
        s = sessions[b]
        refs.append(oacc.accept(logits[b].astype(np.float64), x[b], None if greedy else q[b].astype(np.float64),
                                seed=s.philox_seed, session_id=s.session_id, round_id=1 + seed % 1000))
    return refs, got


@pytest.mark.parametrize("V", [512, 32000])
@pytest.mark.parametrize("greedy", [True, False])
def test_accept_matches_oracle_on_identical_logits(svlib, V, greedy):
    """Level U: K5 vs oracle on the same fp32 logits / draft probs / counters:
    delta and tokens bit-exact wherever every decision margin > 1e-3."""
    from paper_2505_21594_b200 import sv
    mc = ModelCfg(n_layers=1, d_model=128, n_heads=4, d_ff=128, vocab=V, max_ctx=256)
    W = sv.Weights(mc, seed=1)
    eng = sv.Engine(mc, W, max_batch=8, max_gamma=8)
    sessions = [eng.open_session(100 + b, 0x1234 + 77 * b) for b in range(8)]
    tally = Tally(f"level_u_V{V}_{'greedy' if greedy else 'stochastic'}")
    for gamma in (1, 2, 4, 8):
        for seed in range(6):
            refs, got = _accept_case(eng, mc, 8, gamma, seed * 10 + gamma, greedy, sessions)
            for r, g in zip(refs, got):
                tally.add_fixed(r, g, 1e-3, tag=(gamma, seed))
                if r.status == oacc.OK and r.tokens == g.emitted():
                    assert abs(g.score - r.score) <= 1e-5 * max(1.0, r.score)
                    assert abs(g.next_prob - r.next_prob) <= 1e-4 * max(1e-3, r.next_prob)
    print(tally.report())
    save_report(tally.name, tally.asdict())
    assert not tally.hard_mismatch, tally.hard_mismatch[:3]
    assert tally.checked >= 0.9 * tally.n
    for s in sessions:
        s.close()
    eng.close()


def test_accept_protocol_error_zero_draft_mass(svlib):
    from paper_2505_21594_b200 import sv
    mc = ModelCfg(n_layers=1, d_model=128, n_heads=4, d_ff=128, vocab=512, max_ctx=256)
    eng = sv.Engine(mc, sv.Weights(mc, seed=1), max_batch=2, max_gamma=8)
    s = eng.open_session(1, 2)
    logits, x, q = wd.synthetic_accept_case(5, 1, 3, 512)
    q = q.copy()
    q[0, 2, x[0, 2]] = 0.0
    got = eng.debug_accept(torch.from_numpy(logits).cuda(), [sv.Request(s, 1, 0, x[0], torch.from_numpy(q[0]).cuda())])
    assert got[0].status == sv.SV_E_PROTOCOL
    s.close()
    eng.close()


def test_gpu_sampler_leviathan_law_chi_square(svlib):
    """The GPU acceptance kernels as a sampler: over many rounds
    (fresh Philox counters each) with drafts x_1 ~ q_1, the first emitted token is
    distributed as the target p_0 = softmax(z_0) (Leviathan's exactness, the rule
    of Eq. 2 / DESIGN.md R2), and x_1 is accepted with probability sum_v min(p_0, q_1);
    chi-square / binomial at alpha = 1e-3, bins with expectation < 5 merged."""
    from scipy import stats
    from paper_2505_21594_b200 import sv
    V, B, rounds = 128, 8, 1500
    mc = ModelCfg(n_layers=1, d_model=128, n_heads=4, d_ff=128, vocab=V, max_ctx=256)
    eng = sv.Engine(mc, sv.Weights(mc, seed=1), max_batch=B, max_gamma=8)
    sessions = [eng.open_session(500 + b, 0xABC + 31 * b) for b in range(B)]
    rng = np.random.default_rng(12)
    z0 = rng.standard_normal(V) * 2.0
    z = np.stack([z0, rng.standard_normal(V)]).astype(np.float32)          # rows 0 (scores x_1), 1 (bonus)
    p0 = np.exp(z0 - z0.max()); p0 /= p0.sum()
    q1 = np.exp(rng.standard_normal(V) * 2.0); q1 /= q1.sum()
    q1 = q1.astype(np.float32)
    zl = torch.from_numpy(np.broadcast_to(z, (B, 2, V)).copy()).cuda()
    qd = torch.from_numpy(np.broadcast_to(q1[None], (B, 1, V)).copy()).cuda()
    counts = np.zeros(V)
    acc = 0
    for r in range(1, rounds + 1):
        x = rng.choice(V, size=B, p=q1.astype(np.float64) / q1.sum())
        got = eng.debug_accept(zl, [sv.Request(sessions[b], r, 0, [int(x[b])], qd[b]) for b in range(B)])
        for g in got:
            assert g.status == 0
            counts[g.emitted()[0]] += 1
            acc += g.accepted
    n = B * rounds
    exp = n * p0
    big = exp >= 5
    obs = np.append(counts[big], counts[~big].sum())
    ex = np.append(exp[big], exp[~big].sum())
    assert stats.chisquare(obs, ex).pvalue > 1e-3
    alpha = np.minimum(p0, q1.astype(np.float64)).sum()
    assert stats.binomtest(acc, n, alpha).pvalue > 1e-3
    for s in sessions:
        s.close()
    eng.close()


def test_argument_edge_cases(svlib):
    """Synchronous argument errors leave every session untouched: empty batch,
    gamma above the engine's max, batch above max_batch, token ids out of range,
    the same session twice, a second submit while one is in flight, empty prefill."""
    from paper_2505_21594_b200 import sv
    mc = tiny()
    eng = sv.Engine(mc, sv.Weights(mc, seed=1), max_batch=2, max_gamma=4, max_prefill=8)
    s1, s2, s3 = (eng.open_session(i, i) for i in (1, 2, 3))
    for s in (s1, s2, s3):
        s.fill_kv(10, kv_seed=1)
    bad = [
        [],                                                                  # n = 0
        [sv.Request(s1, 1, 3, [1, 2, 3, 4, 5])],                             # gamma 5 > max_gamma 4
        [sv.Request(s, 1, 3, [1, 2]) for s in (s1, s2, s3)],                 # n 3 > max_batch 2
        [sv.Request(s1, 1, mc.vocab, [1, 2])],                               # pending out of range
        [sv.Request(s1, 1, 3, [1, -1])],                                     # draft out of range
        [sv.Request(s1, 1, 3, [1, 2]), sv.Request(s1, 1, 3, [1, 2])],        # same session twice
    ]
    for reqs in bad:
        with pytest.raises((sv.SvError, ValueError)):
            eng.submit(reqs)
    t = eng.submit([sv.Request(s1, 1, 3, [1, 2])])
    with pytest.raises(sv.SvError):                                          # one ticket in flight
        eng.submit([sv.Request(s2, 1, 3, [1, 2])])
    t.wait_final()
    t.release()
    with pytest.raises(sv.SvError):
        s2.prefill([])
    assert s2.length == 10 and s3.length == 10 and s1.length in range(11, 14)
    for s in (s1, s2, s3):
        s.close()
    eng.close()


def test_gpu_sampler_million_trials_v512(svlib):
    """SURVEY.md §8(c) stochastic pin at scale: 10^6 GPU acceptance trials at V = 512
    (256 requests x 4000 rounds, fresh Philox counters per round, x_1 ~ q_1): the
    first emitted token follows p_0 (chi-square, bins with expectation < 5 merged)
    and x_1 is accepted at rate sum_v min(p_0, q_1) (binomial), alpha = 1e-3."""
    import ctypes as C
    from scipy import stats
    from paper_2505_21594_b200 import sv
    V, B, rounds = 512, 256, 4000
    mc = ModelCfg(n_layers=1, d_model=128, n_heads=4, d_ff=128, vocab=V, max_ctx=256)
    eng = sv.Engine(mc, sv.Weights(mc, seed=1), max_batch=B, max_gamma=8)
    sessions = [eng.open_session(1000 + b, 0xDEF + 17 * b) for b in range(B)]
    rng = np.random.default_rng(21)
    z0 = rng.standard_normal(V) * 2.0
    z = np.stack([z0, rng.standard_normal(V)]).astype(np.float32)
    p0 = np.exp(z0 - z0.max()); p0 /= p0.sum()
    q1 = np.exp(rng.standard_normal(V) * 1.5); q1 /= q1.sum()
    q1 = q1.astype(np.float32)
    zl = torch.from_numpy(np.broadcast_to(z, (B, 2, V)).copy()).cuda()
    qd = torch.from_numpy(np.broadcast_to(q1[None], (B, 1, V)).copy()).cuda()
    drafts = np.zeros((B, 1), dtype=np.int32)
    arr = (sv.sv_verify_req * B)()
    for b in range(B):                        # the request structs are built once, re-used every round
        r = arr[b]
        r.session = sessions[b].h
        r.prefix_len = 1
        r.pending_token = 0
        r.gamma = 1
        r.draft_tokens = drafts[b].ctypes.data_as(C.POINTER(C.c_int32))
        r.draft_probs = qd[b].data_ptr()
        r.probs_on_host = 0
    out = (sv.sv_exit_result * B)()
    counts = np.zeros(V)
    acc = 0
    qcdf = np.cumsum(q1.astype(np.float64) / q1.sum())
    for rnd in range(1, rounds + 1):
        drafts[:, 0] = np.minimum(np.searchsorted(qcdf, rng.random(B)), V - 1)
        for b in range(B):
            arr[b].round_id = rnd
        sv.check(svlib.sv_debug_accept(eng.h, C.c_void_p(zl.data_ptr()), arr, B, out))
        for b in range(B):
            assert out[b].status == 0
            counts[out[b].tokens[0]] += 1          # the first emitted token: x_1 if accepted, else the residual draw
            acc += out[b].accepted
    n = B * rounds
    exp = n * p0
    big = exp >= 5
    obs = np.append(counts[big], counts[~big].sum())
    ex = np.append(exp[big], exp[~big].sum())
    p_chi = stats.chisquare(obs, ex).pvalue
    alpha = np.minimum(p0, q1.astype(np.float64)).sum()
    p_bin = stats.binomtest(acc, n, alpha).pvalue
    print(f"{n} trials: chi-square p = {p_chi:.3f}, acceptance {acc / n:.5f} vs {alpha:.5f} (p = {p_bin:.3f})")
    assert p_chi > 1e-3 and p_bin > 1e-3
    for s in sessions:
        s.close()
    eng.close()
