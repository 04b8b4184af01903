"""NEXT-4 (8-way tensor parallelism for batch-1 latency, DESIGN.md §12,
PAPER.md:681) on one GPU: every rank-local GEMM of the decomposition that
tests/tp_emulation.py pins on the host — column splits of W_q / W_k / W_v (heads) and
W_gate / W_up (d_ff tiles) and W_lm (vocabulary tiles), row splits of W_o (heads) and
W_down (d_ff tiles) — run through the step's own tcgen05 GEMM kernels (sv_debug_gemm,
with the tile / split-K / stream-K choice of a step with M rows), the row-split
partials summed in rank order as the all-reduce would; compared with the oracle's
fp64 product of the same bf16 operands (Eq. 3 projections).  The
weights are the oracle's layer-0 / LM-head weights of the Llama2-7B shape."""
import numpy as np
import pytest
import torch

from oracle import gen
from workload.configs import ModelCfg

from .tp_emulation import plan

pytestmark = pytest.mark.gpu

CFG7 = ModelCfg(n_layers=1, d_model=4096, n_heads=32, d_ff=11008, vocab=32000, max_ctx=256)


@pytest.fixture(scope="module")
def eng7():
    from paper_2505_21594_b200 import sv
    W = sv.Weights(CFG7, seed=1)
    e = sv.Engine(CFG7, W, max_batch=32, max_gamma=4)
    yield e
    e.close()


@pytest.fixture(scope="module")
def weights7():
    w = gen.layer_weights(CFG7, 1, 0)
    g = gen.global_weights(CFG7, 1)
    return w, g


def _bf16(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).cuda()


def _check(got, x64, w64, name):
    ref = x64 @ w64.T
    scale = np.abs(ref).max()
    err = np.abs(got.double().cpu().numpy() - ref).max() / scale
    assert err < 2e-5, f"{name}: max err {err:.2e} of max |ref| {scale:.3e}"
    return err


@pytest.mark.parametrize("world", [2, 8])
@pytest.mark.parametrize("M", [5, 80, 160])
def test_tp_rank_gemms_against_oracle(eng7, weights7, world, M):
    w, g = weights7
    d, Dh = CFG7.d_model, CFG7.head_dim
    rng = np.random.default_rng(1000 + 7 * world + M)
    # activations as the GEMMs see them (bf16 rows of RMSNorm(h) * g / SwiGLU outputs)
    x = rng.standard_normal((M, d)).astype(np.float32)
    act = (rng.standard_normal((M, CFG7.d_ff)) * 0.5).astype(np.float32)
    xb, actb = _bf16(x), _bf16(act)
    x64 = xb.double().cpu().numpy()
    act64 = actb.double().cpu().numpy()
    wqkv = np.concatenate([w["wq"], w["wk"], w["wv"]], axis=0)
    errs = {}
    o_sum = None
    down_sum = None
    for shard in plan(CFG7, world):
        h0, h1 = shard["heads"]
        cols = np.r_[h0 * Dh:h1 * Dh]
        # column split: W_q / W_k / W_v rows of this rank's heads -> its q, k, v
        rows = np.concatenate([cols, d + cols, 2 * d + cols])
        errs["qkv"] = _check(eng7.debug_gemm(_bf16(wqkv[rows]), xb), x64, wqkv[rows], "qkv")
        # row split: W_o columns of this rank's heads, partial of h_mid (all-reduce: sum)
        wo = w["wo"][:, cols]
        part = eng7.debug_gemm(_bf16(wo), _bf16(x64[:, cols]))
        o_sum = part.double() if o_sum is None else o_sum + part.double()
        f0, f1 = shard["ff"]
        wgu = np.concatenate([w["wg"][f0:f1], w["wu"][f0:f1]], axis=0)
        errs["gate_up"] = _check(eng7.debug_gemm(_bf16(wgu), xb), x64, wgu, "gate_up")
        wd = w["wdown"][:, f0:f1]
        part = eng7.debug_gemm(_bf16(wd), _bf16(act64[:, f0:f1]))
        down_sum = part.double() if down_sum is None else down_sum + part.double()
        v0, v1 = shard["vocab"]
        errs["lm"] = _check(eng7.debug_gemm(_bf16(g["lm_head"][v0:v1]), xb), x64, g["lm_head"][v0:v1], "lm")
    errs["o_allreduce"] = _check(o_sum, x64, w["wo"], "o all-reduce")
    errs["down_allreduce"] = _check(down_sum, act64, w["wdown"], "down all-reduce")
    print(world, M, {k: f"{v:.1e}" for k, v in errs.items()})


def test_debug_gemm_argument_errors(eng7):
    from paper_2505_21594_b200 import sv
    w = torch.zeros((256, 4096), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(sv.SvError):
        eng7.debug_gemm(w[:100], torch.zeros((5, 4096), dtype=torch.bfloat16, device="cuda"))   # N % 128
    with pytest.raises(sv.SvError):
        eng7.debug_gemm(w, torch.zeros((10000, 4096), dtype=torch.bfloat16, device="cuda"))   # M > max rows
