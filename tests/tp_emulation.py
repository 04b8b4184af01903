"""Tensor-parallel decomposition of the verify step (DESIGN.md
§12), emulated on the host with the oracle's fp64 arithmetic: which slice of every
weight a rank holds, the partial results it computes, and the reductions that must
reproduce the unsharded step.  Test infrastructure only (no product code uses it):
it pins the decomposition the 8-way TP kernels are to implement.

Plan for `world` ranks (Megatron-style, per layer):
  attention : heads split in contiguous groups; rank r holds the W_q / W_k / W_v rows
              of its heads (column split), their K/V cache, and the W_o columns of its
              heads (row split) -> partial O output, all-reduce (sum over ranks)
  MLP       : d_ff split in 128-row GEMM tiles (uneven when d_ff/128 is not a multiple
              of world: 11008 = 86 tiles -> 11/11/11/11/11/11/10/10); W_gate / W_up rows
              (column split), W_down columns (row split) -> partial, all-reduce
  norms     : replicated (every rank holds h after each all-reduce)
  LM head   : vocabulary split in 128-row tiles; logits stay sharded; acceptance
              combines per-rank softmax statistics and race winners (all-gather of a
              few scalars per row), so the [G, V] logits never move
"""
import numpy as np

from oracle import accept as oacc
from oracle import model as om
from oracle import philox


def split_tiles(n: int, world: int, tile: int = 128):
    """Contiguous [start, end) of `n` rows per rank, boundaries on `tile` multiples."""
    tiles = n // tile
    base, extra = divmod(tiles, world)
    out, t = [], 0
    for r in range(world):
        k = base + (1 if r < extra else 0)
        out.append((t * tile, (t + k) * tile))
        t += k
    return out


def plan(cfg, world: int):
    if cfg.n_heads % world:
        raise ValueError("heads must split evenly")
    hp = cfg.n_heads // world
    return [dict(heads=(r * hp, (r + 1) * hp), ff=split_tiles(cfg.d_ff, world)[r],
                 vocab=split_tiles(cfg.vocab, world)[r]) for r in range(world)]


def layer_partials(cfg, w, cache, l, h, pos, shard):
    """Rank-local work of decoder layer l: returns (attention partial of W_o, a function
    that maps the all-reduced h_mid to the MLP partial of W_down)."""
    H, Dh = cfg.n_heads, cfg.head_dim
    G = h.shape[0]
    ctx = int(pos[0])
    h0, h1 = shard["heads"]
    cols = slice(h0 * Dh, h1 * Dh)
    x = om.rms_norm(h, w["g_attn"], cfg.rms_eps)                 # replicated
    q = (x @ w["wq"][cols].T).reshape(G, h1 - h0, Dh)           # column split
    k = (x @ w["wk"][cols].T).reshape(G, h1 - h0, Dh)
    v = (x @ w["wv"][cols].T).reshape(G, h1 - h0, Dh)
    q, k = om.rope(q, pos, cfg.rope_theta), om.rope(k, pos, cfg.rope_theta)
    cache.k[l] = np.concatenate([cache.k[l][:, :ctx, :], k.transpose(1, 0, 2)], axis=1)   # own heads only
    cache.v[l] = np.concatenate([cache.v[l][:, :ctx, :], v.transpose(1, 0, 2)], axis=1)
    a = om.attention(q, cache.k[l], cache.v[l], ctx).reshape(G, (h1 - h0) * Dh)
    part_o = a @ w["wo"][:, cols].T                              # row split -> partial of h += a W_o^T

    def mlp(h_mid):
        f0, f1 = shard["ff"]
        x2 = om.rms_norm(h_mid, w["g_mlp"], cfg.rms_eps)         # replicated
        act = om.silu(x2 @ w["wg"][f0:f1].T) * (x2 @ w["wu"][f0:f1].T)
        return act @ w["wdown"][:, f0:f1].T                      # row split -> partial
    return part_o, mlp


class ShardCache:
    """A rank's KV cache: the layer caches of its heads only."""

    def __init__(self, full: om.KVCache, heads):
        h0, h1 = heads
        self.k = [a[h0:h1].copy() for a in full.k]
        self.v = [a[h0:h1].copy() for a in full.v]
        self.length = full.length


def tp_forward(model, full_cache: om.KVCache, tokens, world: int, allreduce=None, rank=None):
    """The step's final logits [G, V] computed shard by shard.  allreduce(x) sums x
    over ranks; None = emulate every rank in this process (rank must be None) and sum
    their partials here.  Returns the logits of this rank's vocabulary slice (or, when
    emulating, the concatenation of all slices)."""
    cfg = model.cfg
    shards = plan(cfg, world)
    ranks = range(world) if rank is None else [rank]
    caches = {r: ShardCache(full_cache, shards[r]["heads"]) for r in ranks}
    tokens = np.asarray(tokens, dtype=np.int64)
    pos = np.arange(full_cache.length, full_cache.length + len(tokens))
    h = model.glob["embed"][tokens].copy()
    reduce = allreduce or (lambda parts: sum(parts))
    for l in range(cfg.n_layers):
        w = model.layer(l)
        outs = {r: layer_partials(cfg, w, caches[r], l, h, pos, shards[r]) for r in ranks}
        h_mid = h + reduce([outs[r][0] for r in ranks]) if allreduce is None else h + allreduce(outs[rank][0])
        h = h_mid + (reduce([outs[r][1](h_mid) for r in ranks]) if allreduce is None
                     else allreduce(outs[rank][1](h_mid)))
    xf = om.rms_norm(h, model.glob["g_final"], cfg.rms_eps)
    return np.concatenate([xf @ model.glob["lm_head"][shards[r]["vocab"][0]:shards[r]["vocab"][1]].T
                           for r in ranks], axis=-1)


def sharded_accept(z_slices, vocab_slices, drafts, q, seed, session_id, round_id):
    """Leviathan acceptance (oracle/accept.py) with the target logits split by
    vocabulary: per rank only its slice's softmax statistics (max, sum of exp,
    lowest argmax), its drafted tokens' logits and its race winner are combined —
    the way the TP engine would gather a few scalars per row instead of [G, V]."""
    G = z_slices[0].shape[0]
    gamma = len(drafts)
    M = np.array([[z[r].max() for z in z_slices] for r in range(G)])          # [G, ranks]
    Mg = M.max(axis=1)
    S = np.array([sum(np.exp(z[r] - Mg[r]).sum() for z in z_slices) for r in range(G)])
    owner = lambda v: next(i for i, (a, b) in enumerate(vocab_slices) if a <= v < b)
    logit = lambda r, v: z_slices[owner(v)][r, v - vocab_slices[owner(v)][0]]
    p_at = lambda r, v: np.exp(logit(r, v) - Mg[r]) / S[r]
    if q is None:                                                             # greedy
        def amax(r):   # lowest index among the per-rank argmaxes of the global max
            return min(a + int(np.argmax(z[r])) for z, (a, b) in zip(z_slices, vocab_slices)
                       if z[r].max() == Mg[r])
        delta = 0
        for j in range(1, gamma + 1):
            if int(drafts[j - 1]) != amax(j - 1):
                break
            delta = j
        return delta, [int(x) for x in drafts[:delta]] + [amax(delta)]
    q = np.asarray(q, np.float64)
    delta = 0
    for j in range(1, gamma + 1):
        x = int(drafts[j - 1])
        u = philox.uniforms(seed, session_id, round_id, j - 1, philox.PURPOSE_ACCEPT, 1)[0]
        if not (u < p_at(j - 1, x) / q[j - 1, x]):
            break
        delta = j
    V = sum(b - a for a, b in vocab_slices)
    uu = philox.uniforms(seed, session_id, round_id, delta, philox.PURPOSE_RACE, V)
    best = (-1.0, -1)
    for z, (a, b) in zip(z_slices, vocab_slices):                             # per-rank race winner
        p = np.exp(z[delta] - Mg[delta]) / S[delta]
        w = np.maximum(0.0, p - q[delta, a:b]) if delta < gamma else p
        keys = w / -np.log(uu[a:b])
        i = int(np.argmax(keys))
        if keys[i] > best[0]:
            best = (keys[i], a + i)
    return delta, [int(x) for x in drafts[:delta]] + [best[1]]
