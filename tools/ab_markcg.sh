#!/usr/bin/env bash
# A/B of the marking block pass's inline chunk count CG (compile-time,
# OW_NVCC_EXTRA=-DOW_MARK_CG=n) under the dynamic schedule (GPU box helper).
set -u
T=${1:-abc}
OUT=gpurun_out
mkdir -p $OUT
for cg in 4 2 8; do
  OW_NVCC_EXTRA="-DOW_MARK_CG=$cg" python -c "import __graft_entry__ as g; g.build()" > $OUT/${T}_build_$cg.log 2>&1
  for c in C2 C3 C4 C5; do
    OW_NVCC_EXTRA="-DOW_MARK_CG=$cg" timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline \
        --no-e2e > $OUT/${T}_bench_${c}_cg$cg.json 2> $OUT/${T}_bench_${c}_cg$cg.err
  done
done
for f in $OUT/${T}_bench_*.json; do
  python -c "
import json
d=json.load(open('$f')); r=d['roofline']
print('$f'.split('/')[-1], round(d['ms_per_step'],4), 'mark', r['families_ms']['mark'])" 2>/dev/null
done
