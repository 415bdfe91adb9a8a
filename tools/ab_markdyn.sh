#!/usr/bin/env bash
# A/B of the marking block pass's dynamic schedule (GPU box helper): parity
# under OW_MARK_DYN=1, then bench lines for (dyn, CTAs per SM).
set -u
T=${1:-abd}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/${T}_build.log 2>&1
OW_MARK_DYN=1 timeout 900 python -m pytest tests -m gpu -x -q -k "prefilter or pipeline or marking or mark or device or fullsize" \
    > $OUT/${T}_gputest.log 2>&1
echo "rc=$?" >> $OUT/${T}_gputest.log
for c in C2 C4 C3 C5; do
  for v in "0 24" "1 6" "1 12" "1 24"; do
    set -- $v
    OW_MARK_DYN=$1 OW_MARK_CTAS_PER_SM=$2 timeout 300 python bench.py --config $c --steps 20 --warmup 5 \
        --no-cpu-baseline --no-e2e > $OUT/${T}_bench_${c}_d$1_g$2.json 2> $OUT/${T}_bench_${c}_d$1_g$2.err
  done
done
for f in $OUT/${T}_bench_*.json; do
  python -c "
import json
d=json.load(open('$f')); r=d['roofline']
print('$f'.split('/')[-1], round(d['ms_per_step'],4), 'mark', r['families_ms']['mark'], 'frac', round(r['frac'],4))" 2>/dev/null
done
tail -2 $OUT/${T}_gputest.log
