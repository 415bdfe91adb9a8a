#!/usr/bin/env bash
# ncu launch lists (C2, C5) + C2 timelines of the current build (GPU box helper).
set -u
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/el_build.log 2>&1
for c in C2 C5; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file $OUT/el_launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
      > /dev/null 2>&1
  python tools/launch_dram.py $OUT/el_launches_$c.csv > $OUT/el_launches_$c.txt 2>&1
done
timeout 300 python tools/trace_host.py C2 > $OUT/el_trace_host_c2.txt 2>&1
timeout 300 python tools/trace_step.py C2 > $OUT/el_trace_c2.txt 2>&1
timeout 300 python tools/trace_e2e.py C2 > $OUT/el_trace_e2e_c2.txt 2>&1
head -12 $OUT/el_launches_C2.txt; head -8 $OUT/el_launches_C5.txt; sed -n 3,5p $OUT/el_trace_c2.txt
