"""Pins for oracle/model.py.

(a) Library routine: HF transformers LlamaForCausalLM (v5.5) in float64 with the
    same generated weights, over the whole sequence prefix+block in one causal
    pass, must equal the oracle's KV-incremental forward (prefill, then the
    gamma+1 query block), for the final head and the exit head at every layer.
(b) Special cases: RoPE at position 0 is the identity; attention over identical
    keys returns the mean of V; an RMSNorm output has unit RMS.
"""
import numpy as np
import pytest
import torch

from oracle import gen, model as om
from workload import tiny
from workload.configs import ModelCfg


def _hf_model(cfg, m):
    from transformers import LlamaConfig, LlamaForCausalLM
    hc = LlamaConfig(vocab_size=cfg.vocab, hidden_size=cfg.d_model, intermediate_size=cfg.d_ff,
                     num_hidden_layers=cfg.n_layers, num_attention_heads=cfg.n_heads,
                     num_key_value_heads=cfg.n_heads, rms_norm_eps=cfg.rms_eps,
                     max_position_embeddings=cfg.max_ctx, tie_word_embeddings=False,
                     attention_bias=False, mlp_bias=False, hidden_act="silu")
    hc.rope_parameters = {"rope_theta": cfg.rope_theta, "rope_type": "default"}
    hf = LlamaForCausalLM(hc).to(torch.float64).eval()
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))
    with torch.no_grad():
        hf.model.embed_tokens.weight.copy_(t(m.glob["embed"]))
        hf.lm_head.weight.copy_(t(m.glob["lm_head"]))
        hf.model.norm.weight.copy_(t(m.glob["g_final"]))
        for l, layer in enumerate(hf.model.layers):
            w = m.layer(l)
            layer.self_attn.q_proj.weight.copy_(t(w["wq"]))
            layer.self_attn.k_proj.weight.copy_(t(w["wk"]))
            layer.self_attn.v_proj.weight.copy_(t(w["wv"]))
            layer.self_attn.o_proj.weight.copy_(t(w["wo"]))
            layer.mlp.gate_proj.weight.copy_(t(w["wg"]))
            layer.mlp.up_proj.weight.copy_(t(w["wu"]))
            layer.mlp.down_proj.weight.copy_(t(w["wdown"]))
            layer.input_layernorm.weight.copy_(t(w["g_attn"]))
            layer.post_attention_layernorm.weight.copy_(t(w["g_mlp"]))
    # HF evaluates the RoPE angles in float32 (LlamaRotaryEmbedding casts with
    # .float()); evaluate them in float64.  Two float32 islands remain inside HF
    # even for a float64 model (LlamaRMSNorm's variance, the eager softmax), so the
    # pin tolerance is TOL = 1e-6 relative: any structural error (sign, index,
    # transposed operand, wrong norm or RoPE pairing) is O(1).
    Dh = cfg.head_dim
    inv = cfg.rope_theta ** (-torch.arange(0, Dh, 2, dtype=torch.float64) / Dh)

    def rope64(x, position_ids):
        f = position_ids[..., None].to(torch.float64) * inv
        e = torch.cat([f, f], dim=-1)
        return e.cos().to(x.dtype), e.sin().to(x.dtype)

    hf.model.rotary_emb.forward = rope64
    return hf


TOL = 1e-6


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


@pytest.mark.parametrize("cfg", [tiny(),
                                 ModelCfg(n_layers=3, d_model=256, n_heads=2, d_ff=512, vocab=384, max_ctx=128),
                                 # the Llama2-7B layer widths (d 4096, 32 heads, F 11008, V 32000) of
                                 # configs[1..4], 2 layers: pins the oracle's values at the bench shape
                                 ModelCfg(n_layers=2, d_model=4096, n_heads=32, d_ff=11008, vocab=32000, max_ctx=128)],
                         ids=["C1", "Dh128", "7B_width"])
def test_forward_matches_hf_float64(cfg):
    m = om.Model(cfg, seed=1)
    rng = np.random.default_rng(5)
    ctx, G = 37, 5
    seq = rng.integers(0, cfg.vocab, size=ctx + G)
    hf = _hf_model(cfg, m)
    with torch.no_grad():
        out = hf(torch.from_numpy(seq)[None], output_hidden_states=True, use_cache=False)
    ref_final = out.logits[0, ctx:].numpy()
    cache = om.KVCache(cfg)
    om.forward(m, cache, seq[:ctx])                      # prefill
    for le in range(1, cfg.n_layers + 1):
        c = cache.copy()
        z, ze, hs = om.forward(m, c, seq[ctx:], exit_layer=le)
        assert _rel(z, ref_final) < TOL
        # HF hidden_states[l] is the output of decoder layer l (l < L, pre final norm)
        if le < cfg.n_layers:
            hl = out.hidden_states[le][0, ctx:].numpy()
            assert _rel(hs[le], hl) < TOL
            with torch.no_grad():
                ref_exit = hf.lm_head(hf.model.norm(torch.from_numpy(hl))).numpy()
            assert _rel(ze, ref_exit) < TOL
        else:
            assert np.array_equal(ze, z)                 # l_e = L: exit head == final head


def test_incremental_equals_full_recompute():
    cfg = tiny()
    m = om.Model(cfg, seed=3)
    seq = np.random.default_rng(1).integers(0, cfg.vocab, size=30)
    full = om.KVCache(cfg)
    z_full, _, _ = om.forward(m, full, seq)
    inc = om.KVCache(cfg)
    om.forward(m, inc, seq[:25])
    z_inc, _, _ = om.forward(m, inc, seq[25:])
    assert _rel(z_inc, z_full[25:]) < 1e-12
    for l in range(cfg.n_layers):
        assert np.allclose(inc.k[l], full.k[l], rtol=0, atol=1e-12)


def test_rope_position_zero_is_identity():
    x = np.random.default_rng(0).standard_normal((1, 4, 32))
    assert np.array_equal(om.rope(x, np.array([0]), 1e4), x)


def test_rope_is_rotation_of_pairs():
    """rotate-half pairs (i, i+Dh/2) rotate by angle pos*theta^(-2i/Dh)."""
    Dh = 8
    x = np.zeros((1, 1, Dh)); x[0, 0, 1] = 1.0            # unit vector on dim 1 (pair 1 / 5)
    y = om.rope(x, np.array([3]), 100.0)[0, 0]
    ang = 3 * 100.0 ** (-2.0 / Dh)
    assert np.isclose(y[1], np.cos(ang)) and np.isclose(y[5], np.sin(ang))
    assert np.isclose(np.linalg.norm(y), 1.0)


def test_attention_identical_keys_is_mean_of_values():
    H, Dh, ctx, G = 2, 16, 6, 3
    rng = np.random.default_rng(2)
    K = np.tile(rng.standard_normal((H, 1, Dh)), (1, ctx + G, 1))
    V = rng.standard_normal((H, ctx + G, Dh))
    q = rng.standard_normal((G, H, Dh))
    out = om.attention(q, K, V, ctx)
    for j in range(G):
        assert np.allclose(out[j], V[:, :ctx + j + 1, :].mean(axis=1))


def test_attention_causal_mask():
    """Changing keys/values beyond ctx+j must not change query j."""
    H, Dh, ctx, G = 2, 8, 4, 3
    rng = np.random.default_rng(3)
    K = rng.standard_normal((H, ctx + G, Dh)); V = rng.standard_normal((H, ctx + G, Dh))
    q = rng.standard_normal((G, H, Dh))
    a = om.attention(q, K, V, ctx)
    K2, V2 = K.copy(), V.copy(); K2[:, ctx + 1:] += 5; V2[:, ctx + 1:] -= 3
    b = om.attention(q, K2, V2, ctx)
    assert np.array_equal(a[0], b[0]) and not np.allclose(a[1], b[1])


def test_rms_norm_unit_rms():
    h = np.random.default_rng(4).standard_normal((3, 64)) * 7
    x = om.rms_norm(h, np.ones(64), 0.0)
    assert np.allclose(np.sqrt(np.mean(x * x, axis=-1)), 1.0)


def test_synthetic_cache_roundtrip():
    cfg = tiny()
    c = om.KVCache.synthetic(cfg, 2, 20)
    K, V = gen.synthetic_kv(cfg, 2, 1, 20)
    assert np.array_equal(c.k[1], K) and c.length == 20
    c.truncate(7)
    assert c.k[0].shape[1] == 7 and c.length == 7


def test_exit_adapter_against_torch_modules_and_identity():
    """NEXT-3 exit adapter (oracle.model.Adapters, R7b) against the same
    composition built from library modules in float64 (HF LlamaRMSNorm, torch Linear,
    SiLU), and the W_up = 0 special case (identity: the exit equals the plain exit)."""
    import torch
    from transformers.models.llama.modeling_llama import LlamaRMSNorm
    cfg = tiny()
    ad = om.Adapters(cfg, seed=3, rank=128, layers=[1])
    w = ad.w[1]
    h = np.random.default_rng(0).standard_normal((5, cfg.d_model)) * 2.0
    norm = LlamaRMSNorm(cfg.d_model, eps=cfg.rms_eps).double()
    dn = torch.nn.Linear(cfg.d_model, 128, bias=False).double()
    up = torch.nn.Linear(128, cfg.d_model, bias=False).double()
    with torch.no_grad():
        norm.weight.copy_(torch.from_numpy(w["g"]))
        dn.weight.copy_(torch.from_numpy(w["dn"]))
        up.weight.copy_(torch.from_numpy(w["up"]))
        ht = torch.from_numpy(h)
        ref = (ht + up(torch.nn.functional.silu(dn(norm(ht))))).numpy()
    assert np.allclose(ad.apply(1, h), ref, rtol=1e-6, atol=1e-6)   # HF RMSNorm computes its variance in fp32
    assert not np.allclose(ad.apply(1, h), h)            # a random adapter does act
    w["up"] = np.zeros_like(w["up"])
    assert np.array_equal(ad.apply(1, h), h)
