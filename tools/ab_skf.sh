export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/ab
run() { name=$1; cfg=$2; shift 2; env "$@" timeout 600 python bench.py --no-cpu-baseline $cfg > gpurun_out/ab/$name.json 2>gpurun_out/ab/$name.err;
  python -c "
import json; d=json.load(open('gpurun_out/ab/$name.json')); k=d['roofline']['kernels']; print('%-10s %.3f ms' % ('$name', d['latency_p50_ms']), d['clocks']['sm_mhz'], d['clocks']['reasons'], {kk: round(v['ms']*1e3/max(1,v['launches']),1) for kk,v in k.items() if 'exit' not in kk and 'emb' not in kk and 'acc' not in kk})" || tail -2 gpurun_out/ab/$name.err; }
for rep in 1 2; do
run c5 "--config C5 --steps 20 --warmup 3" X=1
run c5f07 "--config C5 --steps 20 --warmup 3" SV_SK_FILL=0.7
run c5f09 "--config C5 --steps 20 --warmup 3" SV_SK_FILL=0.9
run c4_32 "--config C4 --batch 32 --steps 10 --warmup 3" X=1
run c4_32f09 "--config C4 --batch 32 --steps 10 --warmup 3" SV_SK_FILL=0.9
done
