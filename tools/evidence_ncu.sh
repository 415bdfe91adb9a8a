#!/usr/bin/env bash
# ncu --set full of the hot kernels of one C2 / C5 step (raw metrics, details,
# hottest SASS, per-source-line views) on the current build (GPU box helper).
set -u
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/en_build.log 2>&1
for c in C2 C5; do
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k "regex:k_lat_faces|k_mark_blocks|k_mark_items|k_count_fast|k_emit_fast|k_radix_scatter|k_radix_hist|k_scan|k_count_walk|k_prop_gather_dev|k_lat_emit" \
      --launch-skip 0 --launch-count 60 -f -o $OUT/en_full_$c \
      python bench.py --config $c --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/en_ncu_$c.log 2>&1
  ncu -i $OUT/en_full_$c.ncu-rep --page raw --csv \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread,dram__throughput.avg.pct_of_peak_sustained_elapsed \
      > $OUT/en_full_raw_$c.csv 2>&1
  python tools/ncu_hot.py $OUT/en_full_$c.ncu-rep k_lat_faces 40 > $OUT/en_hot_lat_$c.txt 2>&1
  python tools/ncu_hot.py $OUT/en_full_$c.ncu-rep k_mark_blocks 40 > $OUT/en_hot_mark_$c.txt 2>&1
  ncu -i $OUT/en_full_$c.ncu-rep --page details --csv > $OUT/en_details_$c.csv 2>&1
  rm -f $OUT/en_full_$c.ncu-rep
done
for c in C2 C5; do
  for k in k_lat_faces k_mark_blocks; do
    timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" --launch-skip 1 --launch-count 1 -f \
        -o $OUT/en_one python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
    python tools/ncu_lines.py $OUT/en_one.ncu-rep 60 > $OUT/en_lines_${k}_$c.txt 2>&1
    rm -f $OUT/en_one.ncu-rep
  done
done
ls -la $OUT | grep " en_" | wc -l
