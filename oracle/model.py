"""fp64 Llama forward with a KV cache, early-exit head and final head.

The paper names the target only as "Llama2-7B" and gives the
layer recurrence h^(l) = f^(l)(h^(l-1), x), h^(0) = embedding (PAPER.md:96-100,
Eq. 3) and z^(l) = LMHead(h^(l)).  f^(l) is the Llama-2
decoder block with HF defaults (R6):

  x  = RMSNorm(h) * g_attn              RMSNorm(v) = v / sqrt(mean(v^2) + eps)
  q, k, v = x Wq^T, x Wk^T, x Wv^T      (32 heads, no biases)
  q, k  <- RoPE(q, k, pos)              rotate-half, inv_freq_i = theta^(-2i/Dh)
  append k, v to the cache at positions ctx .. ctx+G-1
  a_j = softmax(q_j K^T / sqrt(Dh)) V   keys 0 .. ctx+j (causal inside the block)
  h += a Wo^T
  x  = RMSNorm(h) * g_mlp
  h += (silu(x Wg^T) * (x Wu^T)) Wdown^T

The exit head at layer l_e reads h^(l_e) (output of decoder layer l_e, 1-based)
and applies the shared final norm + shared LM head (R7/R8: adapters are
identity for random-init weights; "each adapter connects to the LM head",
PAPER.md:212).  Pinned against HF LlamaForCausalLM in float64
(tests/test_oracle_model.py).
"""
import numpy as np

from . import gen


def rms_norm(h: np.ndarray, g: np.ndarray, eps: float) -> np.ndarray:
    return h / np.sqrt(np.mean(h * h, axis=-1, keepdims=True) + eps) * g


def silu(x: np.ndarray) -> np.ndarray:
    return x / (1.0 + np.exp(-x))


def rope(x: np.ndarray, pos: np.ndarray, theta: float) -> np.ndarray:
    """x [T, H, Dh]; rotate-half RoPE at integer positions pos [T]."""
    Dh = x.shape[-1]
    half = Dh // 2
    inv_freq = theta ** (-np.arange(0, half, dtype=np.float64) * 2.0 / Dh)
    ang = pos.astype(np.float64)[:, None] * inv_freq[None, :]          # [T, half]
    cos = np.concatenate([np.cos(ang), np.cos(ang)], axis=-1)[:, None, :]
    sin = np.concatenate([np.sin(ang), np.sin(ang)], axis=-1)[:, None, :]
    rot = np.concatenate([-x[..., half:], x[..., :half]], axis=-1)
    return x * cos + rot * sin


class Model:
    """Holds the generated weights (float64) of one random-init model."""

    def __init__(self, cfg, seed: int, lazy: bool = False):
        self.cfg = cfg
        self.seed = seed
        self.glob = gen.global_weights(cfg, seed)
        self.lazy = lazy
        self._layers = None if lazy else [gen.layer_weights(cfg, seed, l) for l in range(cfg.n_layers)]

    def layer(self, l: int) -> dict:
        if self._layers is not None:
            return self._layers[l]
        return gen.layer_weights(self.cfg, self.seed, l)


class KVCache:
    """Per-layer K, V arrays [H, T, Dh] in float64, plus the committed length."""

    def __init__(self, cfg):
        self.cfg = cfg
        H, Dh = cfg.n_heads, cfg.head_dim
        self.k = [np.zeros((H, 0, Dh)) for _ in range(cfg.n_layers)]
        self.v = [np.zeros((H, 0, Dh)) for _ in range(cfg.n_layers)]
        self.length = 0

    @classmethod
    def synthetic(cls, cfg, kv_seed: int, length: int):
        c = cls(cfg)
        for l in range(cfg.n_layers):
            c.k[l], c.v[l] = gen.synthetic_kv(cfg, kv_seed, l, length)
        c.length = length
        return c

    def truncate(self, length: int):
        """KV rollback: keep rows 0..length-1 (accepted rows are a prefix of the
        rows a verify step wrote)."""
        for l in range(self.cfg.n_layers):
            self.k[l] = self.k[l][:, :length, :]
            self.v[l] = self.v[l][:, :length, :]
        self.length = length

    def copy(self):
        c = KVCache(self.cfg)
        c.k = [a.copy() for a in self.k]
        c.v = [a.copy() for a in self.v]
        c.length = self.length
        return c


def attention(q, K, V, ctx: int) -> np.ndarray:
    """q [G, H, Dh]; K, V [H, ctx+G, Dh]; query j attends keys 0..ctx+j."""
    G, H, Dh = q.shape
    out = np.empty_like(q)
    for j in range(G):
        n = ctx + j + 1
        for h in range(H):
            s = K[h, :n, :] @ q[j, h, :] / np.sqrt(Dh)
            s = np.exp(s - s.max())
            out[j, h, :] = (s / s.sum()) @ V[h, :n, :]
    return out


def decoder_layer(cfg, w: dict, cache: KVCache, l: int, h: np.ndarray, pos: np.ndarray) -> np.ndarray:
    """One decoder layer f^(l) (Eq. 3) on the block h [G, d] at
    positions pos (cache rows 0..pos[0]-1 are the cached context); appends the
    block's K/V rows to layer l of `cache` and returns h^(l+1)."""
    H, Dh = cfg.n_heads, cfg.head_dim
    G = h.shape[0]
    ctx = int(pos[0])
    x = rms_norm(h, w["g_attn"], cfg.rms_eps)
    q = (x @ w["wq"].T).reshape(G, H, Dh)
    k = (x @ w["wk"].T).reshape(G, H, Dh)
    v = (x @ w["wv"].T).reshape(G, H, Dh)
    q = rope(q, pos, cfg.rope_theta)
    k = rope(k, pos, cfg.rope_theta)
    cache.k[l] = np.concatenate([cache.k[l][:, :ctx, :], k.transpose(1, 0, 2)], axis=1)
    cache.v[l] = np.concatenate([cache.v[l][:, :ctx, :], v.transpose(1, 0, 2)], axis=1)
    a = attention(q, cache.k[l], cache.v[l], ctx).reshape(G, H * Dh)
    h = h + a @ w["wo"].T
    x = rms_norm(h, w["g_mlp"], cfg.rms_eps)
    return h + (silu(x @ w["wg"].T) * (x @ w["wu"].T)) @ w["wdown"].T


def forward(model: Model, cache: KVCache, tokens: np.ndarray, exit_layer: int = 0):
    """Run the query block `tokens` (positions cache.length ..) through all layers.

    Appends the block's K/V rows to `cache` (cache.length is advanced by len(tokens);
    the caller rolls back).  Returns (final_logits [G, V], exit_logits [G, V] or None,
    hidden states list h^(0..L) [G, d]).
    """
    return forward_many(model, [cache], [tokens], exit_layer)[0]


def forward_many(model: Model, caches, blocks, exit_layer: int = 0):
    """`forward` for several independent sessions (cache_i, block_i): the layer loop
    is outermost so a lazily generated layer is built once for all of them; each
    session's arithmetic is exactly `forward`'s.  Returns a list of
    (final_logits, exit_logits, hidden states) per session."""
    cfg = model.cfg
    blocks = [np.asarray(t, dtype=np.int64) for t in blocks]
    ctxs = [c.length for c in caches]
    poss = [np.arange(ctx, ctx + len(t)) for ctx, t in zip(ctxs, blocks)]
    hs = [model.glob["embed"][t].copy() for t in blocks]   # h^(0), Eq. 3
    hist = [[h.copy()] for h in hs]
    exit_logits = [None] * len(blocks)
    for l in range(cfg.n_layers):
        w = model.layer(l)
        for i, cache in enumerate(caches):
            hs[i] = decoder_layer(cfg, w, cache, l, hs[i], poss[i])
            hist[i].append(hs[i].copy())
            if exit_layer and l + 1 == exit_layer:
                exit_logits[i] = lm_head(model, hs[i])
    for cache, ctx, t in zip(caches, ctxs, blocks):
        cache.length = ctx + len(t)
    return [(lm_head(model, hs[i]), exit_logits[i], hist[i]) for i in range(len(blocks))]


class Adapters:
    """Exit adapters, SURVEY.md §8(f) NEXT-3 (structure only, random init): "adapter
    layers after each layer ... Each adapter connects to the LM head",
    ~3.26M parameters per exit for Llama2-7B (101M / 31 exits).  Reading
    (R7b): a residual bottleneck of rank r on h^(l),
        A_l(h) = h + silu(RMSNorm(h) * g_l  W_dn^T) W_up^T ,
    whose output goes through the shared final norm + LM head (r = 384 at d = 4096:
    2 d r + d = 3.15M parameters)."""

    def __init__(self, cfg, seed: int, rank: int, layers):
        self.cfg, self.rank = cfg, rank
        self.w = {l: gen.adapter_weights(cfg, seed, l, rank) for l in layers}

    def apply(self, layer: int, h: np.ndarray) -> np.ndarray:
        w = self.w[layer]
        x = rms_norm(h, w["g"], self.cfg.rms_eps)
        return h + silu(x @ w["dn"].T) @ w["up"].T


def lm_head(model: Model, h: np.ndarray) -> np.ndarray:
    """z = LMHead(RMSNorm(h) * g_final)."""
    x = rms_norm(h, model.glob["g_final"], model.cfg.rms_eps)
    return x @ model.glob["lm_head"].T
