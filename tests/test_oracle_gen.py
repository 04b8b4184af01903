"""Pins for oracle/gen.py: bf16 rounding vs torch's library conversion, Irwin-Hall
moments, determinism and counter independence."""
import numpy as np
import torch

from oracle import gen
from workload import tiny


def test_bf16_rne_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(100_000).astype(np.float32) * 3,
                        # exact halfway cases in bf16 (low 16 bits = 0x8000)
                        (np.arange(1000, dtype=np.uint32) << 16 | 0x8000).view(np.float32)])
    ours = gen.bf16_rne_bits(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)


def test_irwin_hall_moments():
    s = gen.irwin_hall_sum(1, 42, np.arange(400_000, dtype=np.uint64))
    assert s.min() >= 0 and s.max() <= 1020
    assert abs(s.mean() - 510.0) < 1.0
    assert abs(s.std() - gen.IH_SD) < 1.0


def test_tensor_sd_and_determinism():
    a = gen.gen_tensor(1, gen.layer_tid(0, gen.WQ), (256, 512), 0.02)
    b = gen.gen_tensor(1, gen.layer_tid(0, gen.WQ), (256, 512), 0.02)
    assert np.array_equal(a, b)
    assert abs(a.std() / 0.02 - 1) < 0.02
    assert abs(a.mean()) < 3 * 0.02 / np.sqrt(a.size) * 5
    # every value is a bf16 number
    assert np.array_equal(a.astype(np.float32).view(np.uint32) & 0xFFFF, np.zeros(a.shape, np.uint32))


def test_independent_tensors_uncorrelated():
    a = gen.gen_tensor(1, 100, (100_000,), 1.0)
    b = gen.gen_tensor(1, 101, (100_000,), 1.0)
    c = gen.gen_tensor(2, 100, (100_000,), 1.0)
    assert abs(np.corrcoef(a, b)[0, 1]) < 0.02
    assert abs(np.corrcoef(a, c)[0, 1]) < 0.02


def test_chunk_offset_consistency():
    full = gen.gen_bits(3, 7, 1000, 1.0)
    part = gen.gen_bits(3, 7, 100, 1.0, start=450)
    assert np.array_equal(full[450:550], part)


def test_gain_offset():
    g = gen.gen_tensor(1, gen.TID_NORM_FINAL, (4096,), 0.1, offset=1.0)
    assert abs(g.mean() - 1.0) < 0.01 and abs(g.std() - 0.1) < 0.01


def test_kv_layout():
    cfg = tiny()
    K, V = gen.synthetic_kv(cfg, 2, 1, 10)
    flatK = gen.gen_tensor(2, gen.kv_tid(1, 0), (10, cfg.d_model), 1.0)
    # K[h, pos, dim] == flat[pos, h*Dh + dim]
    assert K[3, 7, 5] == flatK[7, 3 * cfg.head_dim + 5]
    assert V.shape == (cfg.n_heads, 10, cfg.head_dim)
