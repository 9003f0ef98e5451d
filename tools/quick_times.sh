#!/bin/bash
# Quick timing of the BASELINE configs (run on the GPU box).
for a in "--N 128 --n 12 --batch 8192 --dtype f32" "--N 8 --n 2 --batch 1 --dtype f64 --graph" "--N 64 --n 16 --batch 1 --dtype f64 --graph" "--N 1024 --n 32 --batch 1 --dtype f64 --graph" "--N 1024 --n 32 --batch 1 --dtype f32 --graph" "--N 256 --n 128 --batch 1 --dtype f64 --graph" "$@"; do
  python tools/run_case.py $a --reps 20 --time
done
