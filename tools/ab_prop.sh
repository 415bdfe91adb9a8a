#!/usr/bin/env bash
# Full GPU suite + smoke on the current build, then A/B of the propagation
# gather's thread per (leaf, side) (OW_PROP_SIDES) (GPU box helper).
set -u
T=${1:-abp}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/${T}_smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/${T}_smoke.log
timeout 1200 python -m pytest tests -m gpu -q > $OUT/${T}_gputest.log 2>&1
echo "rc=$?" >> $OUT/${T}_gputest.log
for c in C2 C1 C3 C4 C5; do
  for v in 1 0; do
    OW_PROP_SIDES=$v timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
        > $OUT/${T}_bench_${c}_s$v.json 2> $OUT/${T}_bench_${c}_s$v.err
  done
done
for f in $OUT/${T}_bench_*.json; do
  python -c "
import json
d=json.load(open('$f')); r=d['roofline']
print('$f'.split('/')[-1], round(d['ms_per_step'],4), 'prop', r['families_ms']['propagate'])" 2>/dev/null
done
tail -1 $OUT/${T}_smoke.log; tail -2 $OUT/${T}_gputest.log
