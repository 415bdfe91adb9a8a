#!/usr/bin/env bash
# compute-sanitizer over smoke() and tools/sanitize_pass.py (GPU box helper):
#   tools/sanitize.sh <tag>      -> gpurun_out/<tag>_<tool>.txt (+ a summary)
set -u
TAG=${1:-r02_sanitize}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
      python tools/sanitize_pass.py > gpurun_out/${TAG}_${tool}.txt 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/${TAG}_${tool}.txt | tail -1)" \
      >> gpurun_out/${TAG}_summary.txt
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python __graft_entry__.py smoke \
    > gpurun_out/${TAG}_smoke_memcheck.txt 2>&1
echo "smoke memcheck rc=$? $(grep 'ERROR SUMMARY' gpurun_out/${TAG}_smoke_memcheck.txt | tail -1)" >> gpurun_out/${TAG}_summary.txt
cat gpurun_out/${TAG}_summary.txt
