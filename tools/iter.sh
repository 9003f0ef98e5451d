#!/bin/bash
# Quick iteration on the GPU box: fused-variant parity, then c5 timing of the kernel variants
# given as env settings (default: FUSED-R2 at 3 and 2 CTAs/SM, and FUSED-R). Usage: tools/iter.sh <tag>
tag=${1:-it}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fused or c5 or smoke or closed or golden or fail" > gpurun_out/test_${tag}.log 2>&1
tail -3 gpurun_out/test_${tag}.log
for cfg in "BTD_FUSED_R2=1 BTD_R2_MINB=3" "BTD_FUSED_R2=1 BTD_R2_MINB=2" "BTD_FUSED_R2=0"; do
  key=$(echo $cfg | tr ' =' '__')
  env $cfg timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-latency > gpurun_out/bench_${tag}_${key}.json 2> gpurun_out/bench_${tag}_${key}.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${tag}_${key}.json'));print('$cfg', round(d['value']), round(d['ms_per_step'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -5 gpurun_out/bench_${tag}_${key}.err
done
