#!/bin/bash
# ncu --set full of one c5 launch, FUSED-R2 and FUSED-R. Usage: tools/prof_ab.sh <tag>
tag=${1:-ab}
mkdir -p gpurun_out
for r2 in 1 0; do
BTD_FUSED_R2=$r2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:btd_fused -s 3 -c 1 \
    -o gpurun_out/prof_${tag}_r2${r2} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-latency > gpurun_out/prof_${tag}_r2${r2}.log 2>&1
tail -2 gpurun_out/prof_${tag}_r2${r2}.log
done
ls -la gpurun_out | tail -4
