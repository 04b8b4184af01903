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
# 7B-width slice: 640 query rows (persistent GEMM), 80 rows (stream-K persistent GEMM with
# release/acquire partial flags) and one request (tagged split-K pairs, attention split
# partials as tagged pairs, the instruction-cache warm-up passes)
cat > /tmp/san7b.py <<'PY'
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2505_21594_b200 import sv
from workload import drafts as wd
from workload.configs import ModelCfg
mc = ModelCfg(n_layers=2, d_model=4096, n_heads=32, d_ff=11008, vocab=32000, max_ctx=320)
W = sv.Weights(mc, seed=1)
for B, ctx in ((128, 100), (16, 200), (1, 300)):
    eng = sv.Engine(mc, W, max_batch=B, max_gamma=4, use_graphs=False)
    ss = [eng.open_session(1 + b, 5 + b) for b in range(B)]
    for b, s in enumerate(ss): s.fill_kv(ctx, kv_seed=3 + b)
    x, q = wd.timing_drafts(3, B, 4, mc.vocab, s=1.1)
    qd = torch.from_numpy(q).cuda()
    t = eng.submit([sv.Request(ss[b], 1, 7, x[b], qd[b]) for b in range(B)], exit_layer=1)
    t.wait_early(); f = t.wait_final(); t.release()
    print("ok", B, ctx, f[0].emitted())
    for s in ss: s.close()
    eng.close()
PY
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python /tmp/san7b.py > gpurun_out/san7b_$tool.txt 2>&1; echo "7b $tool rc=$?"
done
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python /tmp/san.py > gpurun_out/san_memcheck.txt 2>&1; echo "memcheck rc=$?"
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python /tmp/san.py > gpurun_out/san_racecheck.txt 2>&1; echo "racecheck rc=$?"
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python /tmp/san.py > gpurun_out/san_synccheck.txt 2>&1; echo "synccheck rc=$?"
for f in gpurun_out/san*.txt; do echo "== $f"; tail -n 4 $f; done
