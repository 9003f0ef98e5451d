#!/bin/bash
# Full bench + ncu launch list + ncu --set full of the dominant kernel (run on the GPU box).
# Usage: tools/gpu_bench_profile.sh <tag>
tag=${1:-r01}
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
tail -2 gpurun_out/bench_${tag}.err
cat gpurun_out/bench_${tag}.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:btd_ --csv \
    --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-latency > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:btd_fused -s 3 -c 1 \
    -o gpurun_out/prof_c5_${tag} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-latency > /dev/null 2>&1
ls -la gpurun_out | tail -5
