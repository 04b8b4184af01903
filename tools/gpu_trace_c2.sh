# C2 per-layer chain: launch timeline + small-tile GEMM phase stamps + attention phases
export PYTHONUNBUFFERED=1
OUT=gpurun_out/trc2
mkdir -p $OUT
SV_GTRACE=$OUT/g.csv SV_ATRACE=$OUT/a.csv timeout 300 python tools/trace_step.py --layers 10,20 > $OUT/tr.txt 2>&1
python - <<'PY' >> $OUT/tr.txt
import numpy as np
a=np.genfromtxt('gpurun_out/trc2/a.csv',delimiter=',',names=True,dtype=np.int64)
PH = ["start", "pagetable", "pdl_wait", "q_ready", "mainloop", "warp_merge", "split_merge", "end"]
for cta in (0,1):
    d={}
    for L in range(32):
        r={int(x['phase']):int(x['t_ns']) for x in a if x['layer']==L and x['cta']==cta}
        for p in range(1,8):
            if p in r and p-1 in r and r[p]>0 and r[p-1]>0: d.setdefault(p,[]).append((r[p]-r[p-1])/1e3)
    print("attn cta", cta, {PH[p]:round(float(np.median(v)),2) for p,v in d.items()})
PY
cat $OUT/tr.txt
