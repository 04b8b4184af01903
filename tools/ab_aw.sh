timeout 1200 python -m pytest tests -m gpu -x -q -k "units or tiny_end or 7b or full or rollback or exits or prefill or graphs" 2>&1 | tail -1
VARIANTS=("new:X=1" "nowarm:SV_NO_ATTN_WARM=1" "prev:SV_LIB=$PWD/paper_2505_21594_b200/libsv_prev.so")
source tools/ab.sh
SV_ATRACE=gpurun_out/ab/atrace.csv timeout 300 python tools/trace_step.py --layers 10 > /dev/null 2>&1
python - <<'PY'
import numpy as np
a=np.genfromtxt('gpurun_out/ab/atrace.csv',delimiter=',',names=True,dtype=np.int64)
PH = ["start", "pagetable", "pdl_wait", "q_ready", "mainloop", "warp_merge", "split_merge", "end"]
for cta in (0,1):
    d={}
    for L in range(32):
        r={int(x['phase']):int(x['t_ns']) for x in a if x['layer']==L and x['cta']==cta}
        for p in range(1,8):
            if p in r and p-1 in r and r[p]>0 and r[p-1]>0: d.setdefault(p,[]).append((r[p]-r[p-1])/1e3)
    print(cta, {PH[p]:round(float(np.median(v)),2) for p,v in d.items()})
PY
