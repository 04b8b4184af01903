"""Seeded draft workloads (SURVEY.md §8(d) "Synthetic workloads").

Every function here is an input generator: it draws token ids and probability
vectors from numpy's seeded PCG64 stream.  None of it is the verify method.

Row convention (R15): a request's query block is
[pending, x_1 .. x_gamma]; target logits row r (0..gamma) is the distribution
of the token after query r, so draft x_j with draft distribution q_j is scored
against target row j-1 and row gamma gives the bonus token.
"""
import numpy as np


def zipf_weights(vocab: int, s: float = 1.5) -> np.ndarray:
    """Zipf(s) mass over ranks 1..V (float64, sums to 1)."""
    w = 1.0 / np.arange(1, vocab + 1, dtype=np.float64) ** s
    return w / w.sum()


def zipf_rows(rng: np.random.Generator, n_rows: int, vocab: int, s: float = 1.5) -> np.ndarray:
    """n_rows distributions: Zipf(s) over an independent random permutation each."""
    base = zipf_weights(vocab, s)
    out = np.empty((n_rows, vocab), dtype=np.float64)
    for r in range(n_rows):
        out[r, rng.permutation(vocab)] = base
    return out


def sample_rows(rng: np.random.Generator, probs: np.ndarray) -> np.ndarray:
    """One categorical draw per row by inverse CDF on a float64 uniform."""
    cdf = np.cumsum(probs, axis=-1)
    u = rng.random(probs.shape[0]) * cdf[:, -1]
    idx = (cdf < u[:, None]).sum(axis=-1)
    return np.minimum(idx, probs.shape[-1] - 1).astype(np.int32)


def timing_drafts(seed: int, batch: int, gamma: int, vocab: int, s: float = 1.5):
    """'Vicuna-68M-style' timing workload: q_j = Zipf(1.5) over a random permutation
    (top-1 mass 1/H_{V,1.5} ~ 0.38 at V=32000), x_j ~ q_j.

    Returns (draft_tokens int32 [B, gamma], draft_probs float32 [B, gamma, V]).
    Drafted tokens always have q_j(x_j) > 0 (every entry of a Zipf row is > 0).
    """
    rng = np.random.default_rng([seed, batch, gamma, vocab])
    q = zipf_rows(rng, batch * gamma, vocab, s)
    x = sample_rows(rng, q)
    return x.reshape(batch, gamma), q.astype(np.float32).reshape(batch, gamma, vocab)


def prefix_tokens(seed: int, n: int, vocab: int) -> np.ndarray:
    """Uniform prompt / pending token ids."""
    rng = np.random.default_rng([seed, 7, n, vocab])
    return rng.integers(0, vocab, size=n, dtype=np.int64).astype(np.int32)


def synthetic_accept_case(seed: int, batch: int, gamma: int, vocab: int,
                          agree: float = 0.7, logit_noise: float = 0.5,
                          zipf_s: float = 1.1):
    """Inputs for the acceptance unit tests (K5 alone, SURVEY.md §8(c) level U).

    Target logits are log(Zipf mass over a random permutation) + Gaussian noise;
    the draft distribution q_j is a mixture  agree * base_{j-1} + (1-agree) * other,
    where base_{j-1} is the generator's own Zipf row behind target row j-1 and
    'other' is an independent Zipf row, so acceptance is frequent but not
    certain.  Returns (logits f32 [B, G, V], drafts i32 [B, gamma], probs f32 [B, gamma, V]).
    """
    rng = np.random.default_rng([seed, 11, batch, gamma, vocab])
    G = gamma + 1
    base = zipf_rows(rng, batch * G, vocab, zipf_s).reshape(batch, G, vocab)
    logits = (np.log(base) + logit_noise * rng.standard_normal(base.shape)).astype(np.float32)
    other = zipf_rows(rng, batch * gamma, vocab, zipf_s).reshape(batch, gamma, vocab)
    q = agree * base[:, :gamma, :] + (1.0 - agree) * other
    q = q / q.sum(axis=-1, keepdims=True)
    x = sample_rows(rng, q.reshape(-1, vocab)).reshape(batch, gamma)
    return logits, x, q.astype(np.float32)
