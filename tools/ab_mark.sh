#!/usr/bin/env bash
# A/B of the marking prefilter (GPU box helper): parity suite, bench lines with
# OW_MARK_PREFILTER on / off, launch lists of C4 / C5 and a per-level ncu view of
# k_mark_blocks at C4.   bash tools/ab_mark.sh [tag]
set -u
T=${1:-ab}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/${T}_build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/${T}_gputest.log 2>&1
echo "rc=$?" >> $OUT/${T}_gputest.log
for c in C2 C4 C5 C3; do
  for pf in 1 0; do
    OW_MARK_PREFILTER=$pf timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline \
        > $OUT/${T}_bench_${c}_pf$pf.json 2> $OUT/${T}_bench_${c}_pf$pf.err
  done
done
for c in C4 C5; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file $OUT/${T}_launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-e2e \
      --no-cpu-baseline > /dev/null 2>&1
  python tools/launch_dram.py $OUT/${T}_launches_$c.csv > $OUT/${T}_launches_$c.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_mark_blocks" --launch-skip 0 \
    --launch-count 4 -f -o $OUT/${T}_mark_c4 python bench.py --config C4 --steps 1 --warmup 0 --no-e2e \
    --no-cpu-baseline > $OUT/${T}_mark_c4.log 2>&1
ncu -i $OUT/${T}_mark_c4.ncu-rep --page details --csv > $OUT/${T}_mark_c4_details.csv 2>&1
python tools/ncu_hot.py $OUT/${T}_mark_c4.ncu-rep k_mark_blocks 40 > $OUT/${T}_mark_c4_hot.txt 2>&1
python tools/ncu_lines.py $OUT/${T}_mark_c4.ncu-rep 60 > $OUT/${T}_mark_c4_lines.txt 2>&1
rm -f $OUT/${T}_mark_c4.ncu-rep
for f in $OUT/${T}_bench_*.json; do
  python -c "
import json,sys
d=json.load(open('$f')); r=d['roofline']
print('$f'.split('/')[-1], round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'mark', r['families_ms']['mark'], 'frac', round(r['frac'],4), r['kernel'][:12])" 2>/dev/null
done
tail -2 $OUT/${T}_gputest.log
