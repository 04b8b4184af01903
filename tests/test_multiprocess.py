"""Multi-process (gloo, world_size 2, CPU) tests of the request sharding and the
end-of-run counter gather used by bench.py under torchrun."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2505_21594_b200.dist import gather_counters, job_throughput, shard


def test_shard_partitions_requests():
    for total in (1, 7, 16, 256, 257):
        for world in (1, 2, 3, 4, 8):
            ids = [i for r in range(world) for i in shard(total, world, r)]
            assert ids == list(range(total))
            sizes = [len(shard(total, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def test_job_throughput_uses_slowest_rank():
    allv = np.array([[100.0, 2.0], [300.0, 4.0]])
    assert job_throughput(allv) == 100.0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = list(shard(256, world, rank))
    tokens = float(sum(i % 5 + 1 for i in mine))      # stand-in per-request work
    seconds = 1.0 + rank                              # rank 1 is slower
    allv = gather_counters([tokens, seconds, len(mine)])
    if rank == 0:
        q.put(allv.tolist())
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_two_ranks_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    allv = np.array(q.get(timeout=120))
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert allv.shape == (2, 3)
    assert allv[:, 2].sum() == 256
    total = sum(i % 5 + 1 for i in range(256))
    assert allv[:, 0].sum() == total
    assert job_throughput(allv) == total / 2.0
