#!/usr/bin/env bash
# Final round-2 evidence (GPU box helper): smoke, the GPU suite, bench lines +
# ncu (tools/evidence_r02.sh), sanitizers, C2 timelines.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/fin_smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/fin_smoke.log
timeout 1200 python -m pytest tests -m gpu -q > $OUT/fin_gputest.log 2>&1
echo "rc=$?" >> $OUT/fin_gputest.log
bash tools/evidence_r02.sh > $OUT/ev_all.log 2>&1
bash tools/sanitize.sh fin_sanitize > /dev/null 2>&1
timeout 300 python tools/trace_host.py C2 > $OUT/ev_trace_host_c2.txt 2>&1
timeout 300 python tools/trace_step.py C2 > $OUT/ev_trace_c2.txt 2>&1
timeout 300 python tools/trace_e2e.py C2 > $OUT/ev_trace_e2e_c2.txt 2>&1
tail -2 $OUT/fin_smoke.log; tail -2 $OUT/fin_gputest.log; cat $OUT/fin_sanitize_summary.txt
for c in C1 C2 C3 C4 C5; do
  python -c "
import json
d=json.load(open('$OUT/ev_bench_$c.json')); r=d['roofline']
print('$c', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'frac', round(r['frac'],4), r['kernel'][:14], round(r['secondary']['frac'],4), 'hbm', round(r['hbm']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null
done
head -c 300 $OUT/ev_bench_reference_C2.json
