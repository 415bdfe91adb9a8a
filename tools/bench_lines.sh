#!/usr/bin/env bash
# Bench lines C1-C5 + the GPU suite on the current build (GPU box helper).
set -u
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/bl_smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/bl_smoke.log
timeout 1200 python -m pytest tests -m gpu -q > $OUT/bl_gputest.log 2>&1
echo "rc=$?" >> $OUT/bl_gputest.log
for c in C2 C1 C3 C4 C5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 > $OUT/bl_bench_$c.json 2> $OUT/bl_bench_$c.err
done
timeout 300 python bench.py > $OUT/bl_bench_default.json 2> $OUT/bl_bench_default.err
tail -1 $OUT/bl_smoke.log; tail -2 $OUT/bl_gputest.log
for c in C1 C2 C3 C4 C5 default; do
  python -c "
import json
d=json.load(open('$OUT/bl_bench_$c.json')); r=d['roofline']
print('$c', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'frac', round(r['frac'],4), r['kernel'][:14], round(r['secondary']['frac'],4), 'hbm', round(r['hbm']['frac'],4), r['families_ms']['mark'], d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null
done
