"""One verify step for one session (in order).

Alg-S Listener: verify the draft at every exit, push the
early-exit results with their score, send the final result flagged final.
This oracle runs one early exit l_e plus the final exit (the north star's
configuration), or any list of exits (`exit_layers`: the all-exits streaming
verify of Alg-S; each exit is the LM head on h^(l),
PAPER.md:101-102, accepted with the same counters as the final exit).

The query block is [pending, x_1..x_gamma] at positions ctx..ctx+gamma
(R15).  After the final acceptance the cache is rolled back to
ctx + 1 + delta rows: the pending token plus the accepted drafts (R22);
the emitted correction / bonus token becomes the next step's pending token.
The early exit shares the final exit's Philox counters (R10) and never
changes the session (its output is read-only: "all tokens are verified at the
final exit").
"""
from dataclasses import dataclass

import numpy as np

from . import accept as acc
from .model import KVCache, Model, forward_many, lm_head


@dataclass
class Session:
    session_id: int
    philox_seed: int
    cache: KVCache
    last_round: int = 0


@dataclass
class StepOut:
    final: acc.Result
    early: acc.Result
    final_logits: np.ndarray
    exit_logits: np.ndarray
    new_len: int
    exits: list = None            # [(layer, Result, logits)] for exit_layers


def verify_step(model: Model, sess: Session, round_id: int, pending: int, drafts,
                probs=None, exit_layer: int = 0, exit_layers=(), adapters=None) -> StepOut:
    """adapters (oracle.model.Adapters or None): exit adapters applied to h^(l_e)
    before the shared LM head for every early exit l_e < L (NEXT-3)."""
    return verify_steps(model, [sess], [round_id], [pending], [drafts], [probs], exit_layer, exit_layers,
                        adapters)[0]


def verify_steps(model: Model, sessions, round_ids, pendings, drafts_list, probs_list,
                 exit_layer: int = 0, exit_layers=(), adapters=None):
    """verify_step for several independent sessions at once (one forward pass with
    the layer loop outermost, `forward_many`); per session the arithmetic and the
    acceptance are exactly verify_step's.  Returns a list of StepOut."""
    cfg = model.cfg
    outs = [None] * len(sessions)
    live = []
    for i, (sess, round_id, drafts) in enumerate(zip(sessions, round_ids, drafts_list)):
        if not (0 <= len(drafts) <= 8):  # gamma = 0: the plain autoregressive step ("Cloud AR",
            raise ValueError("gamma must be in 0..8")   # PAPER.md:318): one query, next token from p_0
        if round_id != sess.last_round + 1:
            bad = acc.Result(0, [], 0.0, 0.0, acc.E_PROTOCOL, [])
            outs[i] = StepOut(bad, bad, None, None, sess.cache.length)
        else:
            live.append(i)
    ctxs = {i: sessions[i].cache.length for i in live}
    blocks = [np.array([pendings[i]] + [int(x) for x in drafts_list[i]], dtype=np.int64) for i in live]
    fw = forward_many(model, [sessions[i].cache for i in live], blocks, exit_layer)
    for i, (z, ze, hs) in zip(live, fw):
        sess, round_id = sessions[i], round_ids[i]
        drafts = [int(x) for x in drafts_list[i]]
        ctx = ctxs[i]
        if adapters is not None and exit_layer and exit_layer < cfg.n_layers:
            ze = lm_head(model, adapters.apply(exit_layer, hs[exit_layer]))
        kw = dict(seed=sess.philox_seed, session_id=sess.session_id, round_id=round_id)
        q = None if probs_list[i] is None else np.asarray(probs_list[i], dtype=np.float64)
        final = acc.accept(z, drafts, q, **kw)
        early = acc.accept(ze, drafts, q, **kw) if ze is not None else None
        exits = []
        for le in exit_layers:                        # h^(le) = hs[le] (output of layer le)
            hl = adapters.apply(le, hs[le]) if adapters is not None and le < cfg.n_layers else hs[le]
            zl = lm_head(model, hl)
            exits.append((le, acc.accept(zl, drafts, q, **kw), zl))
        if final.status != acc.OK:
            sess.cache.truncate(ctx)                  # protocol error: KV not advanced
            outs[i] = StepOut(final, early, z, ze, ctx, exits)
            continue
        new_len = ctx + 1 + final.accepted
        sess.cache.truncate(new_len)                  # S14 rollback
        sess.last_round = round_id
        outs[i] = StepOut(final, early, z, ze, new_len, exits)
    return outs


def prefill_step(model: Model, sess: Session, round_id: int, tokens, sample: bool = False):
    """Prefill: run the prompt block through all layers
    (Eq. 3, causal inside the block), keep all its K/V rows, and
    emit the next token from the last row: argmax, or a race sample of p with the
    session's counters at round_id (the gamma = 0 acceptance, R2).
    Returns (Result, last-row logits [1, V])."""
    if round_id != sess.last_round + 1:
        raise ValueError("round_id must be last_round + 1")
    tokens = np.asarray(tokens, dtype=np.int64)
    z, _, _ = forward_many(model, [sess.cache], [tokens])[0]   # cache.length += len(tokens)
    zl = z[-1:]
    q = np.zeros((0, zl.shape[1])) if sample else None
    res = acc.accept(zl, [], q, seed=sess.philox_seed, session_id=sess.session_id, round_id=round_id)
    sess.last_round = round_id
    return res, zl
