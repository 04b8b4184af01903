VARIANTS=("base:X=1" "fill:SV_SPLIT_FILL=1")
source tools/ab.sh
for f in base1 fill1 base2 fill2; do python -c "
import json; d=json.load(open('gpurun_out/ab/$f.json')); k=d['roofline']['kernels']; print('$f', d['latency_p50_ms'], {kk: round(v['ms']*1e3/max(1,v['launches']),2) for kk,v in k.items() if 'exit' not in kk})"; done
