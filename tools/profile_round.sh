#!/usr/bin/env bash
# Round profile capture on the GPU box (run through gpurun from the repo root):
#   tools/profile_round.sh <tag> [config]
# Writes gpurun_out/<tag>_launches.csv (+ .txt summary), gpurun_out/<tag>_full.ncu-rep
# and gpurun_out/<tag>_stages.txt.  Numbers printed under ncu are never bench values.
set -u
TAG=${1:-rXX}
CFG=${2:-C2}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/probe_stages.py $CFG > $OUT/${TAG}_stages.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv \
    python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py $OUT/${TAG}_launches.csv > $OUT/${TAG}_launches.txt 2>&1
# one full capture of each hot kernel of the last warm step (bench --steps 1 --warmup 1)
ncu --set full --clock-control none --import-source on \
    -k "regex:k_lat_mt|k_lat_faces|k_lat_emit|k_lat_hits|k_mark_blocks|k_mark_items|k_chunk_boxes|k_count_fast|k_radix_scatter|k_radix_hist|k_emit_fast|k_stl_to_soa|k_prop_gather_dev|k_split_ring|k_violators_dev" \
    --launch-skip 0 --launch-count 40 -f -o $OUT/${TAG}_full \
    python bench.py --config $CFG --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $OUT/${TAG}_ncu.log 2>&1
ncu -i $OUT/${TAG}_full.ncu-rep --page raw --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread \
    > $OUT/${TAG}_full_raw.csv 2>&1
ls -la $OUT
