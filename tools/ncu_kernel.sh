#!/usr/bin/env bash
# Full ncu capture of one kernel of the C2 bench step (GPU box helper):
#   tools/ncu_kernel.sh <tag> <kernel-regex> [launch-skip] [config]
set -u
TAG=$1; K=$2; SKIP=${3:-0}; CFG=${4:-C2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$K" --launch-skip $SKIP --launch-count 1 -f \
    -o gpurun_out/${TAG} python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline \
    > gpurun_out/${TAG}.log 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>&1
python tools/ncu_hot.py gpurun_out/${TAG}.ncu-rep "$K" 40 > gpurun_out/${TAG}_hot.txt 2>&1
