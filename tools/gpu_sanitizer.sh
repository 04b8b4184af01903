export PYTHONUNBUFFERED=1
# compute-sanitizer: memcheck + racecheck on the tiny config through the C ABI (no graphs: sanitizer sees each launch)
cat > /tmp/san.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2505_21594_b200 import sv
from workload import tiny, drafts as wd
mc = tiny()
W = sv.Weights(mc, seed=1)
eng = sv.Engine(mc, W, max_batch=2, max_gamma=4, use_graphs=False, max_prefill=32)
ss = [eng.open_session(1 + b, 5 + b) for b in range(2)]
for s in ss: s.fill_kv(30, kv_seed=3)
x, q = wd.timing_drafts(3, 2, 4, mc.vocab, s=1.1)
qd = torch.from_numpy(q).cuda()
t = eng.submit_exits([sv.Request(ss[b], 1, 7, x[b], qd[b]) for b in range(2)], [1, 2])
t.wait_early(); f = t.wait_final(); t.release()
s3 = eng.open_session(9, 9)
r = s3.prefill(np.arange(20) % mc.vocab, sample=True)
print("ok", [a.emitted() for a in f], r.emitted())
PY
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python /tmp/san.py > gpurun_out/san_memcheck.txt 2>&1; echo "memcheck rc=$?"
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python /tmp/san.py > gpurun_out/san_racecheck.txt 2>&1; echo "racecheck rc=$?"
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python /tmp/san.py > gpurun_out/san_synccheck.txt 2>&1; echo "synccheck rc=$?"
tail -5 gpurun_out/san_*.txt
