#!/bin/bash
# ncu launch list + one --set full capture of the c5 kernel (run on the GPU box). Usage: tools/prof.sh <tag>
tag=${1:-r01}
mkdir -p gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:btd_ --csv \
    --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-latency > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:btd_fused -s 3 -c 1 \
    -o gpurun_out/prof_c5_${tag} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-latency > /dev/null 2>&1
ls -la gpurun_out | tail -5
