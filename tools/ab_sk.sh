timeout 900 python -m pytest tests -m gpu -x -q -k "units or tiny or 7b or full or rollback or exits or prefill or ar_" 2>&1 | tail -1
VARIANTS=("tag:X=1" "ticket:SV_SK_TICKET=1")
source tools/ab.sh
SV_GTRACE=gpurun_out/tr/gtrace_c2.csv timeout 300 python tools/trace_step.py --layers 10 2>&1 | tail -5
