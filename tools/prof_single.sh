#!/bin/bash
# ncu captures of the single-system kernels (one launch each): c3 WIDE (fp64 N=1024 n=32), c2 WIDE
# (fp64 N=64 n=16), c4 PERSIST2 (fp64 N=256 n=128). Usage: tools/prof_single.sh <tag> [set]
tag=${1:-r02}
set=${2:-full}
mkdir -p gpurun_out
for c in "c3 1024 32" "c2 64 16" "c4 256 128"; do
  set -- $c
  timeout 600 ncu --set $set --clock-control none --import-source on -k regex:btd_ -s 2 -c 1 \
      -o gpurun_out/prof_${tag}_$1 python tools/run_case.py --N $2 --n $3 --batch 1 --dtype f64 --reps 1 > gpurun_out/prof_${tag}_$1.log 2>&1
  tail -1 gpurun_out/prof_${tag}_$1.log
done
ls -la gpurun_out | grep prof_${tag}
