"""The level-E decision bounds of tests/gpu_helpers.py are sound and not vacuous
(DESIGN.md §6): perturbing every logit of a row by at most eps never changes a
result whose decisions all clear their propagated bounds, and most results at a
small eps are checked.  Runs on the oracle only (-m "not gpu")."""
import numpy as np
import pytest

from oracle import accept as oacc

from .gpu_helpers import Tally


def _case(rng, V, gamma, spread):
    z = rng.normal(0.0, spread, size=(gamma + 1, V))
    q = rng.dirichlet(np.full(V, 0.3), size=gamma)
    mix = 0.5 * q + 0.5 * np.stack([oacc.softmax(z[j]) for j in range(gamma)])
    x = [int(rng.choice(V, p=mix[j] / mix[j].sum())) for j in range(gamma)]
    return z, mix / mix.sum(axis=1, keepdims=True), x


@pytest.mark.parametrize("greedy", [True, False], ids=["greedy", "stochastic"])
@pytest.mark.parametrize("eps", [0.002, 0.05])
def test_bounds_sound_under_perturbation(greedy, eps):
    rng = np.random.default_rng(11)
    V, gamma = 48, 3
    tally = Tally()
    n_flips = 0
    for trial in range(300):
        z, q, x = _case(rng, V, gamma, 1.5 if greedy else 2.0)
        qq = None if greedy else q
        ctr = (1234 + trial, 5, 1 + trial % 7)
        ref = oacc.accept(z, x, qq, *ctr)
        for _ in range(4):
            zp = z + rng.uniform(-eps, eps, size=z.shape)
            got = oacc.accept(zp, x, qq, *ctr)

            class G:     # the tally compares against the GPU result interface
                status, accepted = got.status, got.accepted

                @staticmethod
                def emitted():
                    return got.tokens

                @staticmethod
                def asdict():
                    return dict(tokens=got.tokens)
            eps_rows = np.abs(zp - z).max(axis=1)
            tally.add(ref, G, z, eps_rows, qq, ctr)
            n_flips += got.tokens != ref.tokens
    assert not tally.hard_mismatch, tally.hard_mismatch[:2]
    assert tally.checked >= (0.8 if eps < 0.01 else 0.25) * tally.n
    if eps > 0.01:
        assert n_flips > 0            # the perturbation does change some results (the test has teeth)
