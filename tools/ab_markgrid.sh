#!/usr/bin/env bash
# A/B of the marking block-pass grid (GPU box helper): OW_MARK_CTAS_PER_SM.
set -u
T=${1:-abg}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/${T}_build.log 2>&1
for c in C2 C3 C4 C5; do
  for g in 24 6 12 48; do
    OW_MARK_CTAS_PER_SM=$g timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
        > $OUT/${T}_bench_${c}_g$g.json 2> $OUT/${T}_bench_${c}_g$g.err
  done
done
for f in $OUT/${T}_bench_*.json; do
  python -c "
import json
d=json.load(open('$f')); r=d['roofline']
print('$f'.split('/')[-1], round(d['ms_per_step'],4), 'sweep', r['families_ms']['lattice_sweep'], 'mark', r['families_ms']['mark'])" 2>/dev/null
done
