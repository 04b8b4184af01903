"""Host-side logic of bench.py (no GPU): the per-config workload (requests per GPU,
context, scaling, the calibrated drafts' acceptance rate alpha and the expected
tokens per step it implies), and the calibration bisection."""
import sys

import numpy as np
import pytest

import bench


def _args(monkeypatch, *argv):
    monkeypatch.setattr(sys, "argv", ["bench.py", *argv])
    return bench.parse()


@pytest.mark.parametrize("argv, world, per, ctx, scaling, alpha", [
    ((), 1, 1, 512, "weak", 0.825),                                  # C2: the headline
    (("--config", "C3", "--gamma", "7"), 1, 1, 512, "weak", 0.825),
    (("--config", "C4",), 1, 256, 1024, "strong", 0.825),
    (("--config", "C4",), 8, 32, 1024, "strong", 0.825),              # the per-GPU shard of 8
    (("--config", "C5",), 1, 16, 2048, "weak", 0.73),                 # robot tau = 2.92
    (("--config", "C5", "--alpha", "0.9"), 1, 16, 2048, "weak", 0.9),
    (("--config", "C4", "--batch", "32", "--ctx", "300"), 1, 32, 300, "strong", 0.825),
])
def test_workload_per_config(monkeypatch, argv, world, per, ctx, scaling, alpha):
    a = _args(monkeypatch, *argv)
    p, total, c, s = bench.workload(a, world)
    assert (p, total, c, s) == (per, per * world, ctx, scaling)
    assert a.alpha == alpha


def test_expected_tau_is_the_geometric_sum():
    # E[delta + 1] = sum_{k <= gamma} alpha^k (every drafted position accepted w.p. alpha)
    assert abs(bench.expected_tau(4, 0.825) - 3.5304) < 1e-4
    assert abs(bench.expected_tau(4, 0.73) - 2.9359) < 1e-4       # ~ the paper's robot tau 2.92
    assert bench.expected_tau(0, 0.5) == 1.0
    assert bench.expected_tau(3, 1.0) == 4.0


def test_calibrate_row_hits_alpha():
    rng = np.random.default_rng(3)
    V = 512
    p = rng.dirichlet(np.full(V, 0.2))
    r = rng.dirichlet(np.full(V, 0.2))
    for alpha in (0.3, 0.73, 0.825, 0.95):
        lam = bench.calibrate_row(p, r, alpha)
        q = lam * p + (1 - lam) * r
        q /= q.sum()
        assert abs(np.minimum(p, q).sum() - alpha) < 1e-6
