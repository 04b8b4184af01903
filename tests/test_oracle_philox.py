"""Pins for oracle/philox.py: Random123 known-answer vectors (tests/golden/philox_kat.txt)."""
import os

import numpy as np

from oracle import philox

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")


def _kat():
    rows = []
    for line in open(GOLDEN):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        v = [int(t, 16) for t in line.split()]
        rows.append((v[:4], v[4:6], v[6:]))
    return rows


def test_known_answer_vectors():
    rows = _kat()
    assert len(rows) == 3
    for ctr, key, want in rows:
        got = philox.philox4x32_10(*ctr, *key)
        assert [int(g) for g in got] == want


def test_vectorised_matches_scalar():
    c0 = np.arange(17, dtype=np.uint64)
    vec = philox.philox4x32_10(c0, 5, 6, 7, 0x1234, 0x5678)
    for i in range(17):
        one = philox.philox4x32_10(i, 5, 6, 7, 0x1234, 0x5678)
        assert [int(a[i]) for a in vec] == [int(b) for b in one]


def test_uniform_range_and_extremes():
    x = np.array([0, 0x1FF, 0x200, 0xFFFFFFFF], dtype=np.uint64)
    u = philox.u32_to_uniform(x)
    assert u[0] == 2.0 ** -24 and u[1] == 2.0 ** -24
    assert u[2] == 1.5 * 2.0 ** -23
    assert u[3] == 1.0 - 2.0 ** -24
    # every value is exactly representable in float32
    assert np.all(u.astype(np.float32).astype(np.float64) == u)


def test_stream_layout():
    """element e is word e%4 of counter (e//4, row|purpose<<8, round, session)."""
    seed = 0x0123456789ABCDEF
    w = philox.stream_words(seed, session_id=9, round_id=3, row=2, purpose=1, n=10)
    c = philox.philox4x32_10(2, 2 | (1 << 8), 3, 9, seed & 0xFFFFFFFF, seed >> 32)
    assert int(w[8]) == int(c[0]) and int(w[9]) == int(c[1])


def test_uniform_moments():
    u = philox.uniforms(4, 1, 1, 0, 1, 200_000)
    assert abs(u.mean() - 0.5) < 3e-3
    assert abs(u.var() - 1.0 / 12.0) < 2e-3
    assert np.all((u > 0) & (u < 1))
