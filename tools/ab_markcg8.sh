#!/usr/bin/env bash
# A/B of the level from which the marking block pass sweeps 8 chunks inline
# (OW_MARK_CG8_FROM; 99 = never) + parity with CG 8 on every level (GPU box helper).
set -u
T=${1:-ab8}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/${T}_build.log 2>&1
OW_MARK_CG8_FROM=0 timeout 900 python -m pytest tests -m gpu -x -q -k "prefilter or pipeline or marking or mark or device or fullsize" \
    > $OUT/${T}_gputest.log 2>&1
echo "rc=$?" >> $OUT/${T}_gputest.log
for c in C3 C4 C2 C5; do
  for v in 99 0 1 2 3; do
    OW_MARK_CG8_FROM=$v timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
        > $OUT/${T}_bench_${c}_f$v.json 2> $OUT/${T}_bench_${c}_f$v.err
  done
done
for f in $OUT/${T}_bench_*.json; do
  python -c "
import json
d=json.load(open('$f')); r=d['roofline']
print('$f'.split('/')[-1], round(d['ms_per_step'],4), 'mark', r['families_ms']['mark'])" 2>/dev/null
done
tail -2 $OUT/${T}_gputest.log
