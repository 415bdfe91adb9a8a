#!/usr/bin/env bash
# A/B of k_lat_faces launch knobs (GPU box helper): OW_LAT_LANE_ROWS (a row per
# lane for batches of short rows) at C2 / C5 / C3, plus the new parity test.
set -u
T=${1:-abl}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/${T}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "prefilter or lattice or pipeline or marking" \
    > $OUT/${T}_gputest.log 2>&1
echo "rc=$?" >> $OUT/${T}_gputest.log
for c in C5 C2 C3 C4; do
  for lr in 0 1 2 3 4; do
    OW_LAT_LANE_ROWS=$lr timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
        > $OUT/${T}_bench_${c}_lr$lr.json 2> $OUT/${T}_bench_${c}_lr$lr.err
  done
done
for f in $OUT/${T}_bench_*.json; do
  python -c "
import json
d=json.load(open('$f')); r=d['roofline']
print('$f'.split('/')[-1], round(d['ms_per_step'],4), 'sweep', r['families_ms']['lattice_sweep'], 'mark', r['families_ms']['mark'])" 2>/dev/null
done
tail -2 $OUT/${T}_gputest.log
