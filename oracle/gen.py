"""Counter-hash generator for random-init weights and synthetic KV (SURVEY.md §8(c)
"Weights").

The paper's models are trained checkpoints; none can be shipped,
so both sides regenerate the same random-init model from a seed.  The value of
element `idx` of tensor `tid` is a pure function of (seed, tid, idx):

  x  = splitmix64_finalize(seed * 0x9E3779B97F4A7C15 + tid * 0xD1B54A32D192ED03 + idx)  (mod 2^64)
  S  = byte0(x) + byte1(x) + byte2(x) + byte3(x)          Irwin-Hall, mean 510, sd sqrt(21845)
  c  = float32(sigma / sqrt(21845))
  w  = bf16_rne( float32( float32(S - 510) * c ) )                       (weights, KV)
  g  = bf16_rne( float32( float32(float32(S - 510) * c) + 1.0f ) )       (RMSNorm gains)

Only integer ops and correctly rounded fp32 multiply/add/convert occur, so the
CUDA generator (written separately in csrc) produces the same bf16 bits.  Pinned
against torch's fp32->bf16 conversion and by moment checks
(tests/test_oracle_gen.py); the CPU/GPU bit equality is a GPU test.

Tensor ids and sigmas (init recipe measured in SURVEY.md §8(c) "Evidence"):
  1 embed [V,d] sd 1.0            2 lm_head [V,d] sd 3.2/sqrt(d)      3 final norm gain [d] sd 0.1
  16+16l+{0..6}: wq wk wv wo wg wu wdown  [out,in]
     wq wk wv wg wu sd 1.28/sqrt(d);  wo wdown sd 1.28/sqrt(d)/sqrt(2L)
  16+16l+7 / +8: attention / MLP norm gains [d] sd 0.1 around 1.0
  KV: tid 0x100000 + 2*layer + kv (kv 0 = K, 1 = V), idx = pos*d + head*Dh + dim, sd 1.0
"""
import numpy as np

C_SEED = 0x9E3779B97F4A7C15
C_TID = 0xD1B54A32D192ED03
IH_SD = float(np.sqrt(21845.0))

TID_EMBED, TID_LM_HEAD, TID_NORM_FINAL = 1, 2, 3
WQ, WK, WV, WO, WG, WU, WDOWN, G_ATTN, G_MLP = range(9)
TID_KV_BASE = 0x100000


def layer_tid(layer: int, kind: int) -> int:
    return 16 + 16 * layer + kind


def kv_tid(layer: int, kv: int) -> int:
    return TID_KV_BASE + 2 * layer + kv


def _splitmix64_finalize(x):
    u64 = np.uint64
    x = x ^ (x >> u64(30))
    x = x * u64(0xBF58476D1CE4E5B9)
    x = x ^ (x >> u64(27))
    x = x * u64(0x94D049BB133111EB)
    x = x ^ (x >> u64(31))
    return x


def irwin_hall_sum(seed: int, tid: int, idx):
    """S(seed, tid, idx) in [0, 1020] as int64."""
    u64 = np.uint64
    base = (seed * C_SEED + tid * C_TID) & 0xFFFFFFFFFFFFFFFF
    with np.errstate(over="ignore"):
        x = _splitmix64_finalize(u64(base) + np.asarray(idx, dtype=u64))
    m = u64(0xFF)
    s = (x & m) + ((x >> u64(8)) & m) + ((x >> u64(16)) & m) + ((x >> u64(24)) & m)
    return s.astype(np.int64)


def scale_for(sd: float) -> np.float32:
    return np.float32(sd / IH_SD)


def bf16_rne_bits(f32: np.ndarray) -> np.ndarray:
    """Round float32 to bfloat16 (round to nearest even); returns uint16 bits.
    (No NaN/Inf can occur for generator outputs.)"""
    b = np.asarray(f32, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    return b.astype(np.uint16)


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)


def gen_bits(seed: int, tid: int, n: int, sd: float, offset: float = 0.0, start: int = 0) -> np.ndarray:
    """bf16 bits of elements start..start+n-1 of tensor tid."""
    s = irwin_hall_sum(seed, tid, np.arange(start, start + n, dtype=np.uint64))
    v = (s - 510).astype(np.float32) * scale_for(sd)          # fp32 RNE product
    if offset != 0.0:
        v = v + np.float32(offset)                            # fp32 RNE sum
    return bf16_rne_bits(v)


_POOL = None


def _pool():
    """Thread pool over element chunks (numpy releases the GIL inside ufuncs);
    the values do not depend on the chunking (each element is a pure function
    of its index)."""
    global _POOL
    if _POOL is None:
        import concurrent.futures as cf
        import os
        _POOL = cf.ThreadPoolExecutor(max_workers=max(1, min(64, os.cpu_count() or 1)))
    return _POOL


def gen_tensor(seed: int, tid: int, shape, sd: float, offset: float = 0.0) -> np.ndarray:
    """float64 values (exactly the bf16 numbers) of a whole tensor, row-major."""
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np.float64)
    chunk = 1 << 21

    def work(s0):
        m = min(chunk, n - s0)
        out[s0:s0 + m] = bf16_bits_to_f64(gen_bits(seed, tid, m, sd, offset, start=s0))

    if n <= chunk:
        work(0)
    else:
        list(_pool().map(work, range(0, n, chunk)))
    return out.reshape(shape)


def sigmas(cfg):
    d, L = cfg.d_model, cfg.n_layers
    s_in = 1.28 / np.sqrt(d)
    return dict(embed=1.0, lm_head=3.2 / np.sqrt(d), gain=0.1,
                w_in=s_in, w_out=s_in / np.sqrt(2.0 * L), kv=1.0)


def layer_weights(cfg, seed: int, layer: int) -> dict:
    """All float64 weights of decoder layer `layer` (0-based), logical layouts [out, in]."""
    d, F = cfg.d_model, cfg.d_ff
    sg = sigmas(cfg)
    t = lambda k: layer_tid(layer, k)
    return dict(
        wq=gen_tensor(seed, t(WQ), (d, d), sg["w_in"]),
        wk=gen_tensor(seed, t(WK), (d, d), sg["w_in"]),
        wv=gen_tensor(seed, t(WV), (d, d), sg["w_in"]),
        wo=gen_tensor(seed, t(WO), (d, d), sg["w_out"]),
        wg=gen_tensor(seed, t(WG), (F, d), sg["w_in"]),
        wu=gen_tensor(seed, t(WU), (F, d), sg["w_in"]),
        wdown=gen_tensor(seed, t(WDOWN), (d, F), sg["w_out"]),
        g_attn=gen_tensor(seed, t(G_ATTN), (d,), sg["gain"], offset=1.0),
        g_mlp=gen_tensor(seed, t(G_MLP), (d,), sg["gain"], offset=1.0),
    )


def global_weights(cfg, seed: int) -> dict:
    V, d = cfg.vocab, cfg.d_model
    sg = sigmas(cfg)
    return dict(
        embed=gen_tensor(seed, TID_EMBED, (V, d), sg["embed"]),
        lm_head=gen_tensor(seed, TID_LM_HEAD, (V, d), sg["lm_head"]),
        g_final=gen_tensor(seed, TID_NORM_FINAL, (d,), sg["gain"], offset=1.0),
    )


TID_ADAPTER_BASE = 0x200000


def adapter_tid(layer: int, kind: int) -> int:
    """Exit adapter after decoder layer `layer` (1-based): kind 0 = W_dn, 1 = W_up, 2 = gain."""
    return TID_ADAPTER_BASE + 4 * layer + kind


def adapter_sigmas(cfg, rank: int):
    """W_dn as the other input projections (1.28/sqrt(d)); W_up small (0.1/sqrt(r)) so a
    random adapter perturbs the exit without swamping h (R7b)."""
    return dict(dn=1.28 / np.sqrt(cfg.d_model), up=0.1 / np.sqrt(rank), gain=0.1)


def adapter_weights(cfg, seed: int, layer: int, rank: int) -> dict:
    """Exit adapter of layer `layer` (1-based), logical layouts [out, in]:
    dn [rank][d], up [d][rank], g [d]."""
    d = cfg.d_model
    sg = adapter_sigmas(cfg, rank)
    return dict(dn=gen_tensor(seed, adapter_tid(layer, 0), (rank, d), sg["dn"]),
                up=gen_tensor(seed, adapter_tid(layer, 1), (d, rank), sg["up"]),
                g=gen_tensor(seed, adapter_tid(layer, 2), (d,), sg["gain"], offset=1.0))


def synthetic_kv(cfg, kv_seed: int, layer: int, length: int):
    """Synthetic cached K and V for positions 0..length-1 of one layer, as float64
    arrays [H, length, Dh] (the bf16 values the cache holds)."""
    d, H, Dh = cfg.d_model, cfg.n_heads, cfg.head_dim
    out = []
    for kv in (0, 1):
        flat = gen_tensor(kv_seed, kv_tid(layer, kv), (length, d), sigmas(cfg)["kv"])
        out.append(flat.reshape(length, H, Dh).transpose(1, 0, 2).copy())
    return out[0], out[1]
