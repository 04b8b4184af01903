"""Seeded synthetic inputs shared by the oracle side (tests, bench cpu leg) and the
CUDA side (binding, bench).

This package holds NO arithmetic of the method (no forward pass, no softmax of
target logits, no acceptance rule).  It only produces the *inputs* of a verify
step: model shapes, prefix / draft token ids, draft distributions q_j and
synthetic logits for the acceptance unit tests.  See DESIGN.md "Input recipe".
"""
from .configs import ModelCfg, PRESETS, tiny, llama2_7b  # noqa: F401
