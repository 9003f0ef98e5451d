#!/bin/bash
# Quick iteration on the GPU box: fused-variant parity, c5 timing, optional phase timing.
# Usage: tools/iter.sh <tag>
tag=${1:-it}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "fused or c5 or smoke" > gpurun_out/test_${tag}.log 2>&1
tail -3 gpurun_out/test_${tag}.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-latency > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
python -c "import json;d=json.load(open('gpurun_out/bench_${tag}.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['clocks'])"
if [ -f paper_2601_03754_b200/libbtd_timing.so ]; then
  BTD_LIB=paper_2601_03754_b200/libbtd_timing.so timeout 120 python tools/phase_times.py > gpurun_out/phase_${tag}.txt 2>&1
  cat gpurun_out/phase_${tag}.txt
fi
