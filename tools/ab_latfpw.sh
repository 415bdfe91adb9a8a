#!/usr/bin/env bash
# A/B of k_lat_faces faces per warp x lane rows (GPU box helper).
set -u
T=${1:-abf}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/${T}_build.log 2>&1
for c in C5 C4 C2; do
  for v in "0 2" "8 2" "32 2" "16 3" "32 3" "4 2"; do
    set -- $v
    if [ "$1" = "0" ]; then unset OW_FACES_PER_WARP; else export OW_FACES_PER_WARP=$1; fi
    OW_LAT_LANE_ROWS=$2 timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
        > $OUT/${T}_bench_${c}_f$1_l$2.json 2> $OUT/${T}_bench_${c}_f$1_l$2.err
  done
  unset OW_FACES_PER_WARP
done
for f in $OUT/${T}_bench_*.json; do
  python -c "
import json
d=json.load(open('$f')); r=d['roofline']
print('$f'.split('/')[-1], round(d['ms_per_step'],4), 'sweep', r['families_ms']['lattice_sweep'])" 2>/dev/null
done
