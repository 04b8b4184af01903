VARIANTS=("new:X=1" "newcl:SV_ATTN_CLUSTER_LAUNCH=1" "prev:SV_LIB=$PWD/paper_2505_21594_b200/libsv_prev.so")
source tools/ab.sh
for f in new1 newcl1 prev1 new2 newcl2 prev2; do python -c "
import json; d=json.load(open('gpurun_out/ab/$f.json')); k=d['roofline']['kernels']; print('$f', d['latency_p50_ms'], {kk: round(v['ms']*1e3/max(1,v['launches']),2) for kk,v in k.items() if 'exit' not in kk})"; done
