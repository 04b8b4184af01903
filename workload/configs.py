"""Model shapes of BASELINE.json's configs.

Only "Llama2-7B" is named by the paper (§4 Setup); the
architecture constants are HF Llama-2 defaults (reading R6).
"""
from dataclasses import dataclass, asdict


@dataclass(frozen=True)
class ModelCfg:
    n_layers: int
    d_model: int
    n_heads: int
    d_ff: int
    vocab: int
    max_ctx: int = 2304
    page_tokens: int = 64
    rms_eps: float = 1e-5
    rope_theta: float = 10000.0

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    def asdict(self):
        d = asdict(self)
        d["head_dim"] = self.head_dim
        return d


def tiny() -> ModelCfg:
    """configs[0]: 2 layers, d=128, 4 heads, vocab 512 (F=384 is our choice, R6)."""
    return ModelCfg(n_layers=2, d_model=128, n_heads=4, d_ff=384, vocab=512, max_ctx=256)


def llama2_7b(n_layers: int = 32) -> ModelCfg:
    """configs[1..4]: Llama-2-7B shape (32 layers, d=4096, 32 heads, F=11008, V=32000)."""
    return ModelCfg(n_layers=n_layers, d_model=4096, n_heads=32, d_ff=11008, vocab=32000,
                    max_ctx=2304)


PRESETS = {
    "C1": dict(cfg=tiny, batch=1, ctx=64, gamma=4, exit_layer=1),
    "C2": dict(cfg=llama2_7b, batch=1, ctx=512, gamma=4, exit_layer=16),
    "C3": dict(cfg=llama2_7b, batch=1, ctx=512, gamma=(1, 2, 3, 4, 5, 6, 7, 8), exit_layer=(8, 16, 24)),
    "C4": dict(cfg=llama2_7b, batch=256, ctx=1024, gamma=4, exit_layer=16),
    "C5": dict(cfg=llama2_7b, batch=16, ctx=2048, gamma=4, exit_layer=16),
}

# Seeds recorded with every result.
SEED_WEIGHTS = 1
SEED_KV = 2
SEED_WORKLOAD = 3
SEED_PHILOX = 4
