#!/usr/bin/env bash
# A/B of k_lat_emit's grid (software-pipelined loop; OW_LAT_EMIT_CTAS_PER_SM,
# 0 = a CTA per candidate block) + lattice parity (GPU box helper).
set -u
T=${1:-abe}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/${T}_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "lattice or device or fullsize or grid_plan or geometry_to_grid or pdl" \
    > $OUT/${T}_gputest.log 2>&1
echo "rc=$?" >> $OUT/${T}_gputest.log
for c in C5 C2 C4; do
  for v in 0 32 16; do
    OW_LAT_EMIT_CTAS_PER_SM=$v timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
        > $OUT/${T}_bench_${c}_e$v.json 2> $OUT/${T}_bench_${c}_e$v.err
  done
done
for f in $OUT/${T}_bench_*.json; do
  python -c "
import json
d=json.load(open('$f')); r=d['roofline']
print('$f'.split('/')[-1], round(d['ms_per_step'],4), 'lattice', r['families_ms']['lattice'], 'sweep', r['families_ms']['lattice_sweep'])" 2>/dev/null
done
tail -2 $OUT/${T}_gputest.log
