"""NEXT-4 (8-way tensor parallelism for batch-1 latency):
the decomposition the TP engine would implement, pinned on the host against the
unsharded oracle step — head-split attention with row-split W_o, tile-split MLP with
row-split W_down (two all-reduces per layer), vocabulary-split LM head with the
acceptance combined from per-rank scalars.  Single-process emulation of every rank,
and two real ranks over gloo.  (The fused NVLink all-reduce kernels are not built:
DESIGN.md §12.)"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import accept as oacc
from oracle import model as om
from workload.configs import ModelCfg

from .tp_emulation import plan, sharded_accept, split_tiles, tp_forward

CFG = ModelCfg(n_layers=2, d_model=256, n_heads=8, d_ff=768, vocab=1024, max_ctx=128)


def test_split_tiles_partitions_on_gemm_tiles():
    assert split_tiles(11008, 8) == [(i * 1408 if i < 6 else 6 * 1408 + (i - 6) * 1280,
                                      (i + 1) * 1408 if i < 6 else 6 * 1408 + (i - 5) * 1280) for i in range(8)]
    for n, w in ((11008, 8), (32000, 8), (4096, 4), (768, 2)):
        parts = split_tiles(n, w)
        assert parts[0][0] == 0 and parts[-1][1] == n
        assert all(a % 128 == 0 and b % 128 == 0 and b > a for a, b in parts)
        assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
    pl = plan(ModelCfg(n_layers=32, d_model=4096, n_heads=32, d_ff=11008, vocab=32000), 8)
    assert [p["heads"] for p in pl] == [(4 * r, 4 * r + 4) for r in range(8)]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_tp_forward_equals_unsharded(world):
    m = om.Model(CFG, seed=1)
    cache = om.KVCache.synthetic(CFG, 2, 40)
    toks = [5, 17, 300, 2, 999]
    z_full, _, _ = om.forward(m, cache.copy(), toks)
    z_tp = tp_forward(m, cache, toks, world)
    rel = np.abs(z_tp - z_full).max() / np.abs(z_full).max()
    assert rel < 1e-10, rel


@pytest.mark.parametrize("greedy", [True, False], ids=["greedy", "stochastic"])
def test_sharded_accept_equals_oracle(greedy):
    rng = np.random.default_rng(4)
    V, gamma, world = 1024, 4, 8
    sl = split_tiles(V, world)
    for trial in range(60):
        z = rng.normal(0, 2.0, size=(gamma + 1, V))
        q = rng.dirichlet(np.full(V, 0.2), size=gamma)
        mix = 0.5 * q + 0.5 * np.stack([oacc.softmax(z[j]) for j in range(gamma)])
        mix /= mix.sum(axis=1, keepdims=True)
        x = [int(rng.choice(V, p=mix[j])) for j in range(gamma)]
        qq = None if greedy else mix
        ref = oacc.accept(z, x, qq, 77 + trial, 3, 1 + trial)
        got = sharded_accept([z[:, a:b] for a, b in sl], sl, x, qq, 77 + trial, 3, 1 + trial)
        assert got == (ref.accepted, ref.tokens), (trial, got, ref)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    def allreduce(x):
        t = torch.from_numpy(np.ascontiguousarray(x))
        dist.all_reduce(t)                                   # the per-layer sum over ranks
        return t.numpy()
    m = om.Model(CFG, seed=1)
    cache = om.KVCache.synthetic(CFG, 2, 40)
    z_mine = tp_forward(m, cache, [5, 17, 300, 2, 999], world, allreduce=allreduce, rank=rank)
    parts = [torch.zeros(1) for _ in range(world)]
    t = torch.from_numpy(np.ascontiguousarray(z_mine)).flatten()
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([t.numel()]))
    parts = [torch.zeros(int(s.item()), dtype=t.dtype) for s in sizes]
    dist.all_gather(parts, t)
    if rank == 0:
        q.put(np.concatenate([p.numpy().reshape(5, -1) for p in parts], axis=-1))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_tp_step():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    z_tp = q.get(timeout=180)
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    m = om.Model(CFG, seed=1)
    z_full, _, _ = om.forward(m, om.KVCache.synthetic(CFG, 2, 40), [5, 17, 300, 2, 999])
    assert np.abs(z_tp - z_full).max() / np.abs(z_full).max() < 1e-10
