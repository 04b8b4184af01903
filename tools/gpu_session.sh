export PYTHONUNBUFFERED=1
# the multi-rank bench path (sharding, barriers, max-over-ranks timing, counter gather) with
# two ranks on the one GPU of this box (gloo for the gather; NCCL needs distinct GPUs)
SV_BENCH_DEVICE=0 SV_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/b2.json 2> gpurun_out/b2.err
tail -c 900 gpurun_out/b2.json; tail -3 gpurun_out/b2.err
SV_BENCH_DEVICE=0 SV_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/b2r.json 2> gpurun_out/b2r.err
tail -c 300 gpurun_out/b2r.json; tail -2 gpurun_out/b2r.err
