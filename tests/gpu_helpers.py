"""Shared helpers for the -m gpu parity tests: build the CUDA engine and the
oracle side from the same seeds, and compare decisions by margin bins
(DESIGN.md "Parity contract")."""
import numpy as np

from oracle import accept as oacc
from oracle import model as om
from oracle.verify import Session as OSession


def row_rel_err(z_gpu, z_ref):
    """Per-row max_v |z_gpu - z_ref| / max_v |z_ref| and the absolute eps = max_v |dz|."""
    z_gpu = np.asarray(z_gpu, dtype=np.float64)
    z_ref = np.asarray(z_ref, dtype=np.float64)
    d = np.abs(z_gpu - z_ref)
    return d.max(axis=-1) / np.abs(z_ref).max(axis=-1), d.max(axis=-1)


def decision_bound(eps: float) -> float:
    """Margin above which a decision cannot flip when every logit moved by <= eps:
    argmax gap 2*eps; ratio p/q moves by a factor e^(+-2 eps) (bound 2*eps*e^(2 eps)
    * ratio, ratio <= a few); race keys move by <= 2 eps in log for the bonus race.
    A conservative common factor 8*eps (and never below the north star's 1e-3)."""
    return max(1e-3, 8.0 * eps)


class Tally:
    def __init__(self):
        self.n = 0
        self.checked = 0
        self.excluded_mismatch = 0
        self.hard_mismatch = []

    def add(self, ref: oacc.Result, got, bound: float, tag=""):
        self.n += 1
        same = (ref.status == got.status and ref.accepted == got.accepted and
                (ref.status != oacc.OK or ref.tokens == got.emitted()))
        if ref.min_margin > bound:
            self.checked += 1
            if not same:
                self.hard_mismatch.append((tag, ref, got.asdict()))
        elif not same:
            self.excluded_mismatch += 1

    def report(self):
        return (f"{self.n} decisions, {self.checked} above the margin bound, "
                f"{self.excluded_mismatch} mismatches inside the bound (counted), "
                f"{len(self.hard_mismatch)} hard mismatches")


def oracle_session(mc, model, session_id, philox_seed, kv_seed, ctx):
    cache = om.KVCache.synthetic(mc, kv_seed, ctx)
    return OSession(session_id, philox_seed, cache)
