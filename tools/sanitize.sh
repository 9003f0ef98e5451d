#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over tools/sanitize_cases.py (every variant,
# factor, solve and factor+solve). Usage: tools/sanitize.sh <tag>
tag=${1:-r02}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/sanitizer_${tag}_${tool}.txt 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_${tag}_${tool}.txt
done
