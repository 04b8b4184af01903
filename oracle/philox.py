"""Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers: as
easy as 1, 2, 3"), written out round by round in numpy uint64 arithmetic.

Used by the acceptance rule for its uniforms (R10/R11): the stream is
addressed by a 128-bit counter, so the oracle and the CUDA kernel draw the same
numbers without sharing code.

Counter layout:
  c0 = element_index // 4, c1 = row | (purpose << 8), c2 = round_id, c3 = session_id
  key = (seed & 0xffffffff, seed >> 32); word = element_index % 4
Purposes: 0 = acceptance uniform u_j, 1 = race uniforms over the vocabulary.

Pinned by the Random123 known-answer vectors (tests/test_oracle_philox.py).
"""
import numpy as np

M0 = 0xD2511F53
M1 = 0xCD9E8D57
W0 = 0x9E3779B9
W1 = 0xBB67AE85
MASK32 = 0xFFFFFFFF

PURPOSE_ACCEPT = 0
PURPOSE_RACE = 1


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Ten Philox rounds on uint32 counters (numpy arrays or ints, broadcast).

    Each round:  (hi0, lo0) = M0 * c0,  (hi1, lo1) = M1 * c2   (64-bit products)
                 c = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
    and the key is bumped by the Weyl constants (W0, W1) between rounds.
    Returns four uint32 arrays.
    """
    u64 = np.uint64
    c0 = np.asarray(c0, dtype=u64) & u64(MASK32)
    c1 = np.asarray(c1, dtype=u64) & u64(MASK32)
    c2 = np.asarray(c2, dtype=u64) & u64(MASK32)
    c3 = np.asarray(c3, dtype=u64) & u64(MASK32)
    k0 = int(k0) & MASK32
    k1 = int(k1) & MASK32
    for _ in range(10):
        p0 = u64(M0) * c0
        p1 = u64(M1) * c2
        hi0, lo0 = p0 >> u64(32), p0 & u64(MASK32)
        hi1, lo1 = p1 >> u64(32), p1 & u64(MASK32)
        c0, c1, c2, c3 = hi1 ^ c1 ^ u64(k0), lo1, hi0 ^ c3 ^ u64(k1), lo0
        k0 = (k0 + W0) & MASK32
        k1 = (k1 + W1) & MASK32
    return (c0.astype(np.uint32), c1.astype(np.uint32),
            c2.astype(np.uint32), c3.astype(np.uint32))


def u32_to_uniform(x):
    """u = ((x >> 9) + 0.5) * 2^-23, in (0, 1), exact in float32 and float64."""
    x = np.asarray(x, dtype=np.uint64)
    return ((x >> np.uint64(9)).astype(np.float64) + 0.5) * (2.0 ** -23)


def stream_words(seed: int, session_id: int, round_id: int, row: int, purpose: int, n: int):
    """The first n uint32 words of the stream (element e -> word e%4 of counter e//4)."""
    n_ctr = (n + 3) // 4
    c0 = np.arange(n_ctr, dtype=np.uint64)
    c1 = (row | (purpose << 8)) & MASK32
    w = philox4x32_10(c0, c1, round_id & MASK32, session_id & MASK32,
                      seed & MASK32, (seed >> 32) & MASK32)
    return np.stack(w, axis=1).reshape(-1)[:n]


def uniforms(seed: int, session_id: int, round_id: int, row: int, purpose: int, n: int):
    """float64 uniforms for elements 0..n-1 of one (row, purpose) stream."""
    return u32_to_uniform(stream_words(seed, session_id, round_id, row, purpose, n))
