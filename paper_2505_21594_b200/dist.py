"""Multi-GPU plumbing of the verify service.

Requests are independent units: request r is served by rank r // per_rank
(contiguous shards), weights are replicated and every KV cache is local, so the
hot path has no collective.  The only collective is one all_gather of per-rank
counters at the end of a run (NCCL over NVLink on the GPU box, gloo in the CPU
tests).
"""
import numpy as np


def shard(total: int, world: int, rank: int) -> range:
    """Contiguous shard of request ids [0, total) owned by `rank`
    (sizes differ by at most one when world does not divide total)."""
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def gather_counters(values, device=None):
    """all_gather a vector of per-rank float64 counters; returns [world, n] numpy.
    Without an initialised process group returns [1, n]."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if not (dist.is_available() and dist.is_initialized()):
        return t.cpu().numpy()[None]
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return torch.stack(out).cpu().numpy()


def job_throughput(allv: np.ndarray, work_col: int = 0, time_col: int = 1) -> float:
    """Whole-job throughput: total work of all ranks / the slowest rank's time."""
    return float(allv[:, work_col].sum() / allv[:, time_col].max())
