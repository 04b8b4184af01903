"""Pins for oracle/accept.py.

- SPEC.md worked examples (greedy SPEC.md:120-123, residual SPEC.md:139-142,
  confidence SPEC.md:62-66), translated to survey letters (p = target).
- Brute force: greedy delta == longest prefix with x_j == argmax row j-1.
- Leviathan's theorem (adopted): with x_j ~ q_j the emitted
  token at position 1 is distributed as p_0, and conditional on acceptance of
  x_1 the token at position 2 is distributed as p_1 (chi-square, alpha=1e-3);
  per-position acceptance frequency equals E_x~q[min(1, p(x)/q(x))] = sum_v min(p, q).
- Special cases: q == p accepts everything; p(x_j) = 0 always
  rejects; q(x_j) = 0 is a protocol error.
- Exponential race: draws follow normalize(w) (chi-square).
"""
import numpy as np
import pytest
from scipy import stats

from oracle import accept as acc
from oracle import philox


def _logits_with_argmax(ids, V=12, gap=2.0, seed=0):
    rng = np.random.default_rng(seed)
    z = rng.standard_normal((len(ids), V))
    for r, a in enumerate(ids):
        z[r, a] = z[r].max() + gap
    return z


def test_spec_greedy_examples():
    z = _logits_with_argmax([5, 7, 9, 2])
    r = acc.accept_greedy(z, [5, 7, 9])
    assert r.accepted == 3 and r.tokens == [5, 7, 9, 2]
    z = _logits_with_argmax([5, 8, 1, 3])
    r = acc.accept_greedy(z, [5, 7, 9])
    assert r.accepted == 1 and r.tokens == [5, 8]


def test_spec_residual_examples():
    assert np.allclose(acc.residual_distribution([0.2, 0.5, 0.3], [0.6, 0.3, 0.1]), [0, 0.5, 0.5])
    assert np.allclose(acc.residual_distribution([0.5, 0.5], [1.0, 0.0]), [0, 1])
    assert np.allclose(acc.residual_distribution([1.0, 0.0], [0.0, 1.0]), [1, 0])
    with pytest.raises(ValueError):
        acc.residual_distribution([0.5, 0.5], [0.5, 0.5])


def test_spec_confidence_examples():
    assert acc.confidence(acc.softmax(np.zeros(4))) == pytest.approx(0.25)
    assert acc.confidence(acc.softmax(np.array([0.0, -1e4, -1e4]))) == pytest.approx(1.0)
    assert acc.confidence(acc.softmax(np.array([np.log(2.0), 0.0, 0.0]))) == pytest.approx(0.5)


def test_greedy_tie_lowest_index():
    z = np.zeros((2, 5)); z[0, [1, 3]] = 1.0; z[1, 0] = 1.0
    assert acc.accept_greedy(z, [3]).tokens == [1]
    assert acc.accept_greedy(z, [1]).tokens == [1, 0]


def test_greedy_brute_force_random():
    rng = np.random.default_rng(7)
    for _ in range(300):
        V, gamma = int(rng.integers(2, 6)), int(rng.integers(1, 9))
        z = rng.integers(0, 3, size=(gamma + 1, V)).astype(float)      # many ties
        drafts = rng.integers(0, V, size=gamma)
        # brute force: enumerate delta as the largest k with all x_j == argmax(row j-1)
        best = 0
        for k in range(1, gamma + 1):
            if all(drafts[j - 1] == min(np.flatnonzero(z[j - 1] == z[j - 1].max())) for j in range(1, k + 1)):
                best = k
        r = acc.accept_greedy(z, drafts)
        assert r.accepted == best
        assert r.tokens[:best] == list(drafts[:best])
        assert r.tokens[best] == min(np.flatnonzero(z[best] == z[best].max()))
        assert len(r.tokens) == best + 1


def test_score_is_max_confidence_over_emitted_rows():
    z = np.array([[3.0, 0, 0], [0, 0.1, 0], [0, 0, 9.0]])
    r = acc.accept_greedy(z, [0, 1])      # row0 argmax 0 -> accept; row1 argmax 1 -> accept; bonus row2
    assert r.accepted == 2
    assert r.score == pytest.approx(max(acc.softmax(z[k]).max() for k in range(3)))
    r = acc.accept_greedy(z, [1, 1])      # reject at row 0: only row 0 counts
    assert r.accepted == 0 and r.score == pytest.approx(acc.softmax(z[0]).max())
    assert r.next_prob == pytest.approx(acc.softmax(z[0])[0])


def _rows(rng, n, V, conc=1.0):
    return rng.dirichlet(np.full(V, conc), size=n)


def test_q_equals_p_accepts_all():
    rng = np.random.default_rng(1)
    gamma, V = 4, 7
    p = _rows(rng, gamma + 1, V)
    z = np.log(p)
    for rnd in range(1, 200):
        x = [rng.choice(V, p=p[j]) for j in range(gamma)]
        r = acc.accept_stochastic(z, x, p[:gamma], seed=4, session_id=1, round_id=rnd)
        assert r.accepted == gamma and r.tokens[:gamma] == x


def test_zero_target_mass_always_rejected():
    rng = np.random.default_rng(2)
    V = 5
    p0 = np.array([0.0, 0.4, 0.3, 0.2, 0.1])
    with np.errstate(divide="ignore"):
        z = np.log(np.stack([p0, _rows(rng, 1, V)[0]]))
    q = np.array([[0.5, 0.2, 0.1, 0.1, 0.1]])
    seen = set()
    for rnd in range(1, 300):
        r = acc.accept_stochastic(z, [0], q, seed=4, session_id=1, round_id=rnd)
        assert r.accepted == 0 and r.tokens[0] != 0
        seen.add(r.tokens[0])
    # replacement follows normalize(max(0, p0 - q)) = [0, .2, .2, .1, 0]/.5: tokens 1..3 only
    assert seen <= {1, 2, 3} and len(seen) == 3


def test_zero_draft_mass_is_protocol_error():
    z = np.zeros((2, 3))
    r = acc.accept_stochastic(z, [1], np.array([[0.5, 0.0, 0.5]]), seed=1, session_id=1, round_id=1)
    assert r.status == acc.E_PROTOCOL


def test_leviathan_law_chi_square():
    """Emitted token law equals the target law (position 1, and position 2 given
    x_1 accepted), with context-independent target rows."""
    rng = np.random.default_rng(3)
    V, gamma, N = 6, 2, 20000
    p = _rows(rng, gamma + 1, V, conc=2.0)
    q = _rows(rng, gamma, V, conc=2.0)
    z = np.log(p)
    first = np.zeros(V)
    second = np.zeros(V)
    acc_first = 0
    for t in range(N):
        x = [rng.choice(V, p=q[j]) for j in range(gamma)]
        r = acc.accept_stochastic(z, x, q, seed=11, session_id=5, round_id=t + 1)
        first[r.tokens[0]] += 1
        if r.accepted >= 1:
            acc_first += 1
            second[r.tokens[1]] += 1
    assert stats.chisquare(first, N * p[0]).pvalue > 1e-3
    n2 = second.sum()
    assert stats.chisquare(second, n2 * p[1]).pvalue > 1e-3
    # acceptance rate of x_1: alpha = sum_v min(p0, q1)
    alpha = np.minimum(p[0], q[0]).sum()
    assert stats.binomtest(acc_first, N, alpha).pvalue > 1e-3


def test_race_law_chi_square():
    w = np.array([0.0, 3.0, 1.0, 0.5, 0.0, 5.5])
    N = 40000
    counts = np.zeros(len(w))
    for t in range(N):
        u = philox.uniforms(9, 2, t, 0, philox.PURPOSE_RACE, len(w))
        v, _ = acc.race(w, u)
        counts[v] += 1
    assert counts[0] == 0 and counts[4] == 0
    nz = w > 0
    assert stats.chisquare(counts[nz], N * w[nz] / w.sum()).pvalue > 1e-3


def test_acceptance_chain_probability():
    """P(delta >= k | drafts) = prod_{j<=k} min(1, p_{j-1}(x_j)/q_j(x_j)) for fixed drafts."""
    rng = np.random.default_rng(4)
    V, gamma, N = 5, 3, 6000
    p = _rows(rng, gamma + 1, V, conc=3.0)
    q = _rows(rng, gamma, V, conc=3.0)
    z = np.log(p)
    x = [int(np.argmax(q[j])) for j in range(gamma)]
    ge = np.zeros(gamma + 1)
    for t in range(N):
        r = acc.accept_stochastic(z, x, q, seed=12, session_id=3, round_id=t + 1)
        ge[:r.accepted + 1] += 1
    for k in range(1, gamma + 1):
        pk = np.prod([min(1.0, p[j - 1][x[j - 1]] / q[j - 1][x[j - 1]]) for j in range(1, k + 1)])
        assert stats.binomtest(int(ge[k]), N, pk).pvalue > 1e-3


def test_margins_recorded():
    z = _logits_with_argmax([1, 2, 3], V=6, gap=0.5)
    r = acc.accept_greedy(z, [1, 2])
    assert [k for k, _, _ in r.margins] == ["argmax", "argmax", "argmax"]
    assert r.min_margin == pytest.approx(0.5)


def test_gamma_zero_ar_step():
    """gamma = 0 (plain AR step): no drafts, delta = 0; greedy emits
    argmax z_0, sampling emits a draw from p_0 = softmax(z_0) (chi-square)."""
    rng = np.random.default_rng(8)
    V, N = 7, 20000
    p0 = _rows(rng, 1, V, conc=1.5)
    z = np.log(p0)
    g = acc.accept(z, [])
    assert g.accepted == 0 and g.tokens == [int(np.argmax(z[0]))]
    counts = np.zeros(V)
    for t in range(N):
        r = acc.accept(z, [], np.zeros((0, V)), seed=3, session_id=2, round_id=t + 1)
        assert r.accepted == 0 and len(r.tokens) == 1
        counts[r.tokens[0]] += 1
    assert stats.chisquare(counts, N * p0[0]).pvalue > 1e-3


# --------------------------------------------------------------------------------
# Exact enumeration of the emitted-token law (SURVEY.md §8(c) "Stochastic
# acceptance": V <= 8, gamma <= 2; Leviathan's theorem, adopted by PAPER.md:24, :80;
# SPEC.md:133, :156).  Target rows p_r and draft rows q_j are rationals with
# power-of-two denominators, so every ratio p/q the rule forms is exact in float64.
# accept_stochastic runs once per (drafts x, accept/reject branch of every tested
# position) with uniforms chosen inside each branch (u = r/2 accepts, u = (1+r)/2
# rejects, both exactly on their side of u < r), and its sampler records the
# distribution w it would draw the next token from instead of drawing.  Each call
# carries the exact branch weight prod_j q_j(x_j) * P(branch); the composed law of
# the emitted tokens must equal the target law.  Any plausible mistake (residual
# from the wrong row or with the wrong sign, the bonus from p_{gamma-1}, a
# non-strict or inverted ratio test, a dropped normalisation) changes the law by
# O(1e-2), against the 1e-12 tolerance.
# --------------------------------------------------------------------------------
from fractions import Fraction
import itertools


def _dyadic_rows(rng, n, V, den=64, zero_frac=0.25):
    """n probability rows with entries k/den (some exactly zero)."""
    rows = []
    for _ in range(n):
        while True:
            w = rng.integers(0, 8, size=V) * (rng.random(V) > zero_frac)
            if w.sum() > 0:
                break
        # scale to den: entries k/den summing to 1 (den a power of two >= V*8)
        k = np.floor(w / w.sum() * den).astype(int)
        k[int(np.argmax(w))] += den - k.sum()
        rows.append([Fraction(int(v), den) for v in k])
    return rows


def _enumerate_law(P, Q):
    """Compose the oracle's outcome law over every draft sequence and branch.
    P: gamma+1 rows of Fractions (target), Q: gamma rows (draft).
    Returns {emitted token tuple: probability (float)} and P(delta >= k)."""
    gamma, V = len(Q), len(P[0])
    with np.errstate(divide="ignore"):
        z = np.log(np.array([[float(v) for v in r] for r in P]))
    qf = np.array([[float(v) for v in r] for r in Q])
    law = {}
    reach = np.zeros(gamma + 1)
    supports = [[v for v in range(V) if Q[j][v] > 0] for j in range(gamma)]
    for x in itertools.product(*supports):
        wx = 1.0
        for j in range(gamma):
            wx *= float(Q[j][x[j]])
        # branch = number of accepted positions k (then a rejection if k < gamma)
        for k in range(gamma + 1):
            prob = wx
            us = []
            ok = True
            for j in range(min(k + 1, gamma)):          # positions 1..k accepted, k+1 rejected
                r = P[j][x[j]] / Q[j][x[j]]
                pa = min(Fraction(1), r)
                if j < k:
                    prob *= float(pa)
                    us.append(float(r) / 2 if r < 1 else 0.5)
                else:
                    if r >= 1:
                        ok = False                     # cannot reject
                        break
                    prob *= float(1 - pa)
                    us.append((1.0 + float(r)) / 2)
            if not ok or prob == 0.0:
                continue
            seen = {}

            def uniforms(row, purpose, n):
                return np.array([us[row]]) if purpose == philox.PURPOSE_ACCEPT else np.full(n, 0.5)

            def sample(w, u):
                seen["w"] = np.asarray(w, dtype=np.float64) / np.sum(w)
                return 0, float("inf")

            res = acc.accept_stochastic(z, list(x), qf, 0, 0, 0, uniforms=uniforms, sample=sample)
            assert res.status == acc.OK and res.accepted == k
            reach[:k + 1] += prob
            for v in range(V):
                if seen["w"][v] > 0:
                    key = tuple(x[:k]) + (v,)
                    law[key] = law.get(key, 0.0) + prob * seen["w"][v]
    return law, reach


@pytest.mark.parametrize("V,gamma,seed", [(3, 1, 0), (5, 1, 1), (4, 2, 2), (6, 2, 3), (8, 2, 4)])
def test_leviathan_law_exact_enumeration(V, gamma, seed):
    rng = np.random.default_rng(100 + seed)
    P = _dyadic_rows(rng, gamma + 1, V)
    Q = _dyadic_rows(rng, gamma, V)
    law, reach = _enumerate_law(P, Q)
    pf = np.array([[float(v) for v in r] for r in P])
    qf = np.array([[float(v) for v in r] for r in Q])
    assert sum(law.values()) == pytest.approx(1.0, abs=1e-12)
    # first emitted token ~ p_0
    y1 = np.zeros(V)
    for key, pr in law.items():
        y1[key[0]] += pr
    assert np.abs(y1 - pf[0]).max() < 1e-12
    # P(delta >= 1) = sum_v min(p_0, q_1); for gamma = 2 P(delta >= 2) multiplies by sum min(p_1, q_2)
    a1 = np.minimum(pf[0], qf[0]).sum()
    assert reach[1] == pytest.approx(a1, abs=1e-12)
    if gamma == 2:
        a2 = np.minimum(pf[1], qf[1]).sum()
        assert reach[2] == pytest.approx(a1 * a2, abs=1e-12)
    # conditional on delta >= 1 (x_1 emitted), the next emitted token ~ p_1
    if a1 > 0:
        y2 = np.zeros(V)
        for key, pr in law.items():
            if len(key) >= 2:
                y2[key[1]] += pr
        assert np.abs(y2 / a1 - pf[1]).max() < 1e-12


def test_exact_enumeration_detects_a_wrong_residual():
    """The enumeration is sharp: a rule that draws the replacement from q's
    residual max(0, q - p) instead of max(0, p - q) breaks the law."""
    rng = np.random.default_rng(7)
    P = _dyadic_rows(rng, 2, 5)
    Q = _dyadic_rows(rng, 1, 5)
    orig = acc.residual_distribution
    try:
        acc.residual_distribution = lambda p, q: orig(q, p)
        law, _ = _enumerate_law(P, Q)
    finally:
        acc.residual_distribution = orig
    y1 = np.zeros(5)
    for key, pr in law.items():
        y1[key[0]] += pr
    assert np.abs(y1 - np.array([float(v) for v in P[0]])).max() > 1e-3


# --------------------------------------------------------------------------------
# Decision margins: each margin is the size of the
# smallest perturbation, in its own units, that flips the decision — the property
# the GPU parity gates rely on.  Perturbing by just under the margin keeps the
# decision; just over flips it.
# --------------------------------------------------------------------------------
def test_race_margin_is_the_log_key_gap_that_flips_the_draw():
    rng = np.random.default_rng(21)
    for t in range(200):
        V = int(rng.integers(2, 40))
        w = rng.random(V) * (rng.random(V) > 0.3)
        if (w > 0).sum() < 2:
            continue
        u = philox.uniforms(3, 1, t, 0, philox.PURPOSE_RACE, V)
        v, m = acc.race(w, u)
        keys = np.where(w > 0, w / -np.log(u), 0.0)
        second = int(np.argsort(keys)[-2])
        for f, flips in ((1 - 1e-6, False), (1 + 1e-6, True)):
            w2 = w.copy()
            w2[v] *= np.exp(-m / 2 * f)
            w2[second] *= np.exp(m / 2 * f)
            v2, _ = acc.race(w2, u)
            assert (v2 != v) == flips, (t, f)
    _, m = acc.race(np.array([0.0, 2.0, 0.0]), np.array([0.3, 0.6, 0.9]))
    assert m == float("inf")


def test_argmax_margin_is_the_gap_that_flips_the_argmax():
    rng = np.random.default_rng(22)
    for t in range(200):
        z = rng.standard_normal((1, int(rng.integers(2, 30))))
        r = acc.accept_greedy(z, [])
        a, g = r.tokens[0], r.margins[0][2]
        second = int(np.argsort(z[0])[-2])
        for f, flips in ((1 - 1e-9, False), (1 + 1e-9, True)):
            z2 = z.copy()
            z2[0, a] -= g / 2 * f
            z2[0, second] += g / 2 * f
            assert (int(np.argmax(z2[0])) != a) == flips


def test_ratio_margin_is_distance_to_the_threshold():
    """|u - p/q|: moving the ratio by less than the margin keeps the decision."""
    rng = np.random.default_rng(23)
    V = 6
    for t in range(100):
        p = rng.dirichlet(np.ones(V))
        q = rng.dirichlet(np.ones(V))
        z = np.log(np.stack([p, p]))
        x = [int(rng.integers(0, V))]
        r = acc.accept_stochastic(z, x, q[None], 5, 1, t + 1)
        kind, row, m = r.margins[0]
        assert kind == "ratio" and row == 0
        u = philox.uniforms(5, 1, t + 1, 0, philox.PURPOSE_ACCEPT, 1)[0]
        ratio = p[x[0]] / q[x[0]]
        assert m == pytest.approx(abs(u - ratio), rel=1e-12)
        for f, flips in ((1 - 1e-6, False), (1 + 1e-6, True)):
            q2 = q.copy()
            target = ratio + (m * f if u >= ratio else -m * f)   # push the ratio towards / past u
            q2[x[0]] = p[x[0]] / target
            r2 = acc.accept_stochastic(z, x, q2[None], 5, 1, t + 1)
            assert (r2.accepted != r.accepted) == flips
