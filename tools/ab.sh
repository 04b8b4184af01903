# A/B of engine switches on the C2 bench (same box, interleaved twice)
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/ab
run() { name=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 100 --warmup 5 > gpurun_out/ab/$name.json 2>gpurun_out/ab/$name.err;
  python -c "
import json,sys; d=json.load(open('gpurun_out/ab/$name.json')); k=d['roofline']['kernels']; print('%-12s p50 %.4f ms  gemm frac %.4f  attn %.1f O %.1f us' % ('$name', d['latency_p50_ms'], d['roofline']['frac'], k['attention']['ms']*1e3/32, k['gemm_o']['ms']*1e3/32))" || tail -2 gpurun_out/ab/$name.err; }
for rep in 1 2; do
for v in "${VARIANTS[@]}"; do run ${v%%:*}$rep ${v#*:}; done
done
