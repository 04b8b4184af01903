"""Acceptance rule of the verify step, in float64, in the paper's order.

Letters follow the north star / Leviathan convention (R1):
p = TARGET distribution, q = DRAFT distribution.  (PAPER.md uses the opposite
letters: draft M_p emits p; target M_q.)

Verify (Eq. 2) decides delta <= gamma accepted drafts and emits
one more token, x_{t:t+delta+1}.  The rule is adopted by citation from Leviathan
et al.; R2 writes it out:

  rows r = 0..gamma of the target logits; row r is the distribution after query r,
  so draft x_j (j = 1..gamma, distribution q_j) is scored by target row j-1.

  greedy  : accept x_j iff x_j == argmax z_{j-1} (lowest index on ties); stop at
            the first mismatch; next token = argmax z_delta.
  sampling: p_r = softmax(z_r); accept x_j iff u_j < p_{j-1}(x_j) / q_j(x_j)
            (u_j = Philox purpose 0, row j-1, element 0); any q_j(x_j) <= 0
            is a protocol error for the whole request.  If delta < gamma the next token is
            drawn from normalize(max(0, p_delta - q_{delta+1})), else (bonus)
            from p_gamma, by an exponential race: argmax_v w_v / E_v with
            E_v = -ln u_v (Philox purpose 1, row delta).  If the residual is
            numerically all zero, w = p_delta (R13).

Confidence S_r = max softmax(z_r) (Eq. 4); exit score
s = max_{r <= delta} S_r (Alg-S "s^(i) <- max(q^(i)_{1:delta+1})", PAPER.md:1104,
DESIGN.md R9).

Decision margins: top-2 logit gap for an argmax,
|u - ratio| for an accept test, top-2 gap of the race keys in the log domain.
"""
from dataclasses import dataclass, field

import numpy as np

from . import philox

OK = 0
E_PROTOCOL = 2


@dataclass
class Result:
    accepted: int
    tokens: list
    score: float
    next_prob: float
    status: int = OK
    margins: list = field(default_factory=list)   # (kind, row, margin)

    @property
    def min_margin(self) -> float:
        return min((m for _, _, m in self.margins), default=float("inf"))


def softmax(z: np.ndarray) -> np.ndarray:
    z = np.asarray(z, dtype=np.float64)
    e = np.exp(z - z.max())
    return e / e.sum()


def confidence(p: np.ndarray) -> float:
    """Eq. 4: S = max softmax(z), given the softmax output p."""
    return float(np.max(p))


def argmax_lowest(z: np.ndarray) -> int:
    """argmax with the lowest index winning ties (numpy returns the first)."""
    return int(np.argmax(z))


def top2_gap(z: np.ndarray) -> float:
    """Difference between the largest and second-largest entries (0 on a tie)."""
    z = np.asarray(z, dtype=np.float64)
    if z.size < 2:
        return float("inf")
    part = np.partition(z, -2)
    return float(part[-1] - part[-2])


def residual_distribution(p: np.ndarray, q: np.ndarray) -> np.ndarray:
    """normalize(max(0, p - q)) (SPEC.md:134-142 in survey letters)."""
    w = np.maximum(0.0, np.asarray(p, np.float64) - np.asarray(q, np.float64))
    s = w.sum()
    if s <= 0.0:
        raise ValueError("residual distribution undefined: p <= q everywhere")
    return w / s


def race(w: np.ndarray, u: np.ndarray):
    """Exponential race: argmax_v w_v / E_v, E_v = -ln u_v.  An exact draw from
    normalize(w) when u_v are iid uniform(0,1) (min of independent exponentials
    E_v / w_v is attained at v with probability w_v / sum(w)).
    Returns (token, margin) with margin = log-domain top-2 gap of the keys."""
    w = np.asarray(w, dtype=np.float64)
    E = -np.log(np.asarray(u, dtype=np.float64))
    keys = w / E
    v = int(np.argmax(keys))
    pos = keys[keys > 0]
    if pos.size >= 2:
        top = np.partition(pos, -2)
        margin = float(np.log(top[-1]) - np.log(top[-2]))
    else:
        margin = float("inf")
    return v, margin


def accept_greedy(z: np.ndarray, drafts) -> Result:
    """z [G, V] target logits (rows 0..gamma); drafts [gamma]."""
    z = np.asarray(z, dtype=np.float64)
    gamma = len(drafts)
    margins = []
    delta = 0
    for j in range(1, gamma + 1):
        a = argmax_lowest(z[j - 1])
        margins.append(("argmax", j - 1, top2_gap(z[j - 1])))
        if int(drafts[j - 1]) != a:
            break
        delta = j
    nxt = argmax_lowest(z[delta])
    if delta == gamma:
        margins.append(("argmax", delta, top2_gap(z[delta])))
    probs = [softmax(z[r]) for r in range(delta + 1)]
    score = max(confidence(p) for p in probs)
    return Result(delta, [int(t) for t in drafts[:delta]] + [nxt], score,
                  float(probs[delta][nxt]), OK, margins)


def philox_uniforms(seed: int, session_id: int, round_id: int):
    """The session's counter-based uniforms: a function
    (row, purpose, n) -> n uniforms of (purpose, logits row, round, session)."""
    return lambda row, purpose, n: philox.uniforms(seed, session_id, round_id, row, purpose, n)


def accept_stochastic(z: np.ndarray, drafts, q: np.ndarray, seed: int, session_id: int,
                      round_id: int, uniforms=None, sample=None) -> Result:
    """z [G, V] target logits; drafts [gamma]; q [gamma, V] draft distributions
    (q[j-1] is q_j, the distribution x_j was drafted from).

    uniforms(row, purpose, n) supplies the random numbers (default: the session's
    Philox stream); sample(w, u) -> (token, margin) draws from normalize(w)
    (default: the exponential race).  Both are parameters so the tests can
    enumerate the rule's branches exactly (tests/test_oracle_accept.py)."""
    z = np.asarray(z, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    uniforms = uniforms or philox_uniforms(seed, session_id, round_id)
    sample = sample or race
    gamma = len(drafts)
    V = z.shape[1]
    # a drafted token the drafter gave no mass is a corrupt batch,
    # checked for every position before any decision (R12)
    if not all(q[j - 1, int(drafts[j - 1])] > 0.0 for j in range(1, gamma + 1)):
        return Result(0, [], 0.0, 0.0, E_PROTOCOL, [])
    p = [softmax(z[r]) for r in range(gamma + 1)]
    margins = []
    delta = 0
    for j in range(1, gamma + 1):
        x = int(drafts[j - 1])
        ratio = p[j - 1][x] / q[j - 1, x]
        u = uniforms(j - 1, philox.PURPOSE_ACCEPT, 1)[0]
        margins.append(("ratio", j - 1, abs(u - ratio)))
        if not (u < ratio):
            break
        delta = j
    if delta < gamma:                                   # rejection at x_{delta+1}, q_{delta+1} = q[delta]
        try:
            w = residual_distribution(p[delta], q[delta])
        except ValueError:                              # numerically all-zero residual (R13)
            w = p[delta]
    else:                                               # all accepted: bonus token from p_gamma
        w = p[gamma]
    nxt, m = sample(w, uniforms(delta, philox.PURPOSE_RACE, V))
    margins.append(("race", delta, m))
    score = max(confidence(p[r]) for r in range(delta + 1))
    return Result(delta, [int(t) for t in drafts[:delta]] + [nxt], score,
                  float(p[delta][nxt]), OK, margins)


def accept(z, drafts, q=None, seed=0, session_id=0, round_id=0) -> Result:
    """Greedy when q is None (R3), stochastic otherwise."""
    if q is None:
        return accept_greedy(z, drafts)
    return accept_stochastic(z, drafts, q, seed, session_id, round_id)
