"""Shared helpers for the -m gpu parity tests: build the CUDA engine and the
oracle side from the same seeds, and compare decisions by margin bins
(DESIGN.md §6 "Parity contract").

Level E (end to end, fp64 oracle forward vs the bf16 GPU forward): a decision
on the oracle's path is *checked* when its margin exceeds both the north star's
1e-3 and the bound that the measured logit error of its row propagates to it
(`decision_bounds`); a mismatch there is a bug.  Mismatches of unchecked
decisions are counted and reported.

Level U (unit, identical inputs): the oracle's acceptance run on the GPU's own
downloaded fp32 logits with the session's counters must reproduce the GPU's
decisions bit-exactly wherever every margin exceeds 1e-3 (`level_u`)."""
import json
import math
import os

import numpy as np

from oracle import accept as oacc
from oracle import model as om
from oracle import philox
from oracle.verify import Session as OSession

MARGIN = 1e-3          # north star: "bit-exact wherever the margin exceeds 1e-3"


def row_rel_err(z_gpu, z_ref):
    """Per-row max_v |z_gpu - z_ref| / max_v |z_ref| and the absolute eps = max_v |dz|."""
    z_gpu = np.asarray(z_gpu, dtype=np.float64)
    z_ref = np.asarray(z_ref, dtype=np.float64)
    d = np.abs(z_gpu - z_ref)
    return d.max(axis=-1) / np.abs(z_ref).max(axis=-1), d.max(axis=-1)


def _race_safe(p, qrow, u, eps, bonus):
    """Whether the exponential race's winner is fixed for every p' with
    |ln p'_v - ln p_v| <= 2 eps (|dz| <= eps moves z_v - lse by at most 2 eps).
    Keys are w_v / E_v, E_v = -ln u_v, w = p (bonus) or max(0, p - q) (residual);
    the race is scale-invariant, so normalisation does not matter.  Returns the
    log-domain slack ln(min key of the winner) - ln(max key of any other) (> 0:
    safe)."""
    E = -np.log(np.asarray(u, dtype=np.float64))
    up, lo = p * math.exp(2 * eps), p * math.exp(-2 * eps)
    if not bonus:
        up, lo = np.maximum(0.0, up - qrow), np.maximum(0.0, lo - qrow)
    w = p if bonus else np.maximum(0.0, p - qrow)
    top = int(np.argmax(w / E))
    k_lo = lo[top] / E[top]
    k_up = up / E
    k_up[top] = 0.0
    other = k_up.max()
    if k_lo <= 0.0:
        return -np.inf
    if other <= 0.0:
        return np.inf
    return float(np.log(k_lo) - np.log(other))


def decision_bounds(ref: oacc.Result, z_ref, eps_rows, q=None, counters=None):
    """For every decision (kind, row, margin) on the oracle's path: (kind, row,
    margin, safe).  Per-kind propagation of a logit error eps = max_v |dz| of the
    row:
      argmax: a top-2 gap > 2 eps cannot flip;
      ratio : p(x)/q(x) moves by a factor within e^(+-2 eps); with u < 1 and
              m = |u - r| the test cannot flip if m > (e^(2eps) - 1) / (2 - e^(2eps));
      race  : every key's bound (see _race_safe) must leave the winner on top.
    `counters` = (seed, session_id, round_id) for the race uniforms."""
    out = []
    z_ref = np.asarray(z_ref, dtype=np.float64)
    gamma = z_ref.shape[0] - 1
    for kind, row, m in ref.margins:
        eps = float(eps_rows[row])
        if kind == "argmax":
            safe = m > max(MARGIN, 2 * eps)
        elif kind == "ratio":
            g = math.exp(2 * eps)
            safe = g < 2 and m > max(MARGIN, (g - 1) / (2 - g))
        else:
            p = oacc.softmax(z_ref[row])
            bonus = row == gamma
            u = philox.uniforms(counters[0], counters[1], counters[2], row, philox.PURPOSE_RACE, p.size)
            safe = m > MARGIN and _race_safe(p, None if bonus else np.asarray(q[row], np.float64), u, eps,
                                             bonus) > 0
        out.append((kind, row, m, bool(safe)))
    return out


def _same(ref: oacc.Result, got) -> bool:
    return (ref.status == got.status and ref.accepted == got.accepted and
            (ref.status != oacc.OK or ref.tokens == got.emitted()))


class Tally:
    """Level-E tally: results whose every decision is safe are 'checked' and must
    match; the rest are counted (mismatches inside the bound are expected at
    ~1-2% of rows at the 7B shape, SURVEY.md §8(c) evidence)."""

    def __init__(self, name=""):
        self.name = name
        self.n = 0
        self.checked = 0
        self.decisions = 0
        self.decisions_safe = 0
        self.excluded_mismatch = 0
        self.hard_mismatch = []

    def add(self, ref: oacc.Result, got, z_ref, eps_rows, q=None, counters=None, tag=""):
        self.n += 1
        dec = decision_bounds(ref, z_ref, eps_rows, q, counters)
        self.decisions += len(dec)
        self.decisions_safe += sum(1 for d in dec if d[3])
        if all(d[3] for d in dec):
            self.checked += 1
            if not _same(ref, got):
                self.hard_mismatch.append((tag, ref, got.asdict()))
        elif not _same(ref, got):
            self.excluded_mismatch += 1

    def add_fixed(self, ref: oacc.Result, got, bound: float, tag=""):
        """A result whose GPU logits are not observable (sv_prefill's last row):
        every decision must clear a fixed bound instead of the propagated one."""
        self.n += 1
        self.decisions += len(ref.margins)
        safe = [m > max(MARGIN, bound) for _, _, m in ref.margins]
        self.decisions_safe += sum(safe)
        if all(safe):
            self.checked += 1
            if not _same(ref, got):
                self.hard_mismatch.append((tag, ref, got.asdict()))
        elif not _same(ref, got):
            self.excluded_mismatch += 1

    def report(self):
        return (f"{self.name}: {self.n} results ({self.decisions} decisions, {self.decisions_safe} beyond their "
                f"propagated bound), {self.checked} results checked, {self.excluded_mismatch} mismatches inside "
                f"the bound (counted), {len(self.hard_mismatch)} hard mismatches")

    def asdict(self):
        return dict(name=self.name, results=self.n, checked=self.checked, decisions=self.decisions,
                    decisions_safe=self.decisions_safe, excluded_mismatch=self.excluded_mismatch,
                    hard_mismatch=len(self.hard_mismatch))


class UTally:
    """Level-U tally: oracle acceptance on the GPU's logits vs the GPU."""

    def __init__(self, name=""):
        self.name = name
        self.n = 0
        self.checked = 0
        self.excluded_mismatch = 0
        self.hard_mismatch = []
        self.score_err = 0.0

    def add(self, z_gpu, got, drafts, q, counters, tag=""):
        """z_gpu [G, V] fp32 logits the GPU accepted on; q [gamma, V] or None (greedy)."""
        ref = oacc.accept(np.asarray(z_gpu, np.float64), [int(x) for x in drafts],
                          None if q is None else np.asarray(q, np.float64), *counters)
        self.n += 1
        if ref.min_margin > MARGIN:
            self.checked += 1
            if not _same(ref, got):
                self.hard_mismatch.append((tag, ref, got.asdict()))
            elif ref.status == oacc.OK:
                self.score_err = max(self.score_err, abs(ref.score - got.score), abs(ref.next_prob - got.next_prob))
        elif not _same(ref, got):
            self.excluded_mismatch += 1
        return ref

    def report(self):
        return (f"{self.name}: {self.n} results, {self.checked} with every margin > {MARGIN} (bit-exact required), "
                f"{self.excluded_mismatch} mismatches inside the margin, {len(self.hard_mismatch)} hard mismatches, "
                f"max |score/next_prob diff| {self.score_err:.2e}")

    def asdict(self):
        return dict(name=self.name, results=self.n, checked=self.checked, excluded_mismatch=self.excluded_mismatch,
                    hard_mismatch=len(self.hard_mismatch), score_err=self.score_err)


def save_report(name: str, payload: dict):
    """Keep a parity tally (json) under $SV_PARITY_OUT (default gpurun_out/parity/,
    copied to profiles/ after a GPU run)."""
    d = os.environ.get("SV_PARITY_OUT", os.path.join(os.path.dirname(os.path.dirname(__file__)),
                                                     "gpurun_out", "parity"))
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, name + ".json"), "w") as f:
        json.dump(payload, f, indent=1, default=str)


def oracle_session(mc, model, session_id, philox_seed, kv_seed, ctx):
    cache = om.KVCache.synthetic(mc, kv_seed, ctx)
    return OSession(session_id, philox_seed, cache)
