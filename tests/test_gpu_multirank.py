"""Request sharding on the GPU: two ranks under
torchrun on one GPU (SV_BENCH_DEVICE, gloo for the counter gather) serve a
256-request-style pool split into contiguous shards; each rank's results are
bitwise equal to a single-process run of the same shard (bench.py --shard R/N).
Small per-rank batch and context so the test stays short."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--config", "C4", "--batch", "3", "--ctx", "192", "--steps", "3", "--warmup", "1", "--no-cpu-baseline"]


def _run(cmd, env, tmp):
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return r.stdout


def test_two_ranks_equal_single_rank_shards(svlib, tmp_path):
    env = dict(os.environ, SV_BENCH_DEVICE="0", SV_DIST_BACKEND="gloo")
    dump = str(tmp_path / "multi_{rank}.json")
    out = _run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py", "--gpus", "2",
                "--dump-results", dump] + ARGS, env, tmp_path)
    line = json.loads(out.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["config"]["world_size"] == 2 and line["config"]["global_batch"] == 6
    for r in (0, 1):
        single = str(tmp_path / f"single_{r}.json")
        _run([sys.executable, "bench.py", "--shard", f"{r}/2", "--dump-results", single] + ARGS,
             dict(os.environ, SV_BENCH_DEVICE="0"), tmp_path)
        a = json.load(open(dump.replace("{rank}", str(r))))
        b = json.load(open(single))
        assert sorted(a) == sorted(b) and len(a) == 3
        assert a == b, f"rank {r} differs from its single-process run"
