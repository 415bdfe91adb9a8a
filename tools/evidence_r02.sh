#!/usr/bin/env bash
# Round-2 evidence on one B200 (GPU box helper): bench lines per config, the
# reference arm, ncu launch lists with DRAM bytes (C2, C5), full captures of
# the hot kernels (C2, C5) and their per-source-line summaries.
set -u
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/ev_build.log 2>&1
for c in C2 C1 C3 C4 C5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 > $OUT/ev_bench_$c.json 2> $OUT/ev_bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/ev_bench_reference_C2.json 2> $OUT/ev_bench_reference_C2.err
for c in C2 C5; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file $OUT/ev_launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
      > /dev/null 2>&1
  python tools/launch_dram.py $OUT/ev_launches_$c.csv > $OUT/ev_launches_$c.txt 2>&1
done
for c in C2 C5; do
  timeout 900 ncu --set full --clock-control none --import-source on \
      -k "regex:k_lat_faces|k_mark_blocks|k_mark_items|k_count_fast|k_emit_fast|k_radix_scatter|k_radix_hist|k_scan|k_count_walk" \
      --launch-skip 0 --launch-count 60 -f -o $OUT/ev_full_$c \
      python bench.py --config $c --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/ev_ncu_$c.log 2>&1
  ncu -i $OUT/ev_full_$c.ncu-rep --page raw --csv \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread,dram__throughput.avg.pct_of_peak_sustained_elapsed \
      > $OUT/ev_full_raw_$c.csv 2>&1
  python tools/ncu_hot.py $OUT/ev_full_$c.ncu-rep k_lat_faces 40 > $OUT/ev_hot_lat_$c.txt 2>&1
  python tools/ncu_hot.py $OUT/ev_full_$c.ncu-rep k_mark_blocks 40 > $OUT/ev_hot_mark_$c.txt 2>&1
  ncu -i $OUT/ev_full_$c.ncu-rep --page details --csv > $OUT/ev_details_$c.csv 2>&1
  rm -f $OUT/ev_full_$c.ncu-rep  # (gpurun copies back at most 64 MiB)
done
for c in C2 C5; do  # per-source-line view of the two hot kernels (small single-kernel reports)
  for k in k_lat_faces k_mark_blocks; do
    timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$k" --launch-skip 1 --launch-count 1 -f \
        -o $OUT/ev_one python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
    python tools/ncu_lines.py $OUT/ev_one.ncu-rep 60 > $OUT/ev_lines_${k}_$c.txt 2>&1
    rm -f $OUT/ev_one.ncu-rep
  done
done
du -sh $OUT; ls -la $OUT | tail -60
