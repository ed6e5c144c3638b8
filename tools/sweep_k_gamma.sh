#!/bin/bash
# Config 5 (BASELINE.json): top-k / gamma sweep at 32K context (config 2's shape), one bench line each.
# usage (on the GPU box): tools/sweep_k_gamma.sh > gpurun_out/sweep.jsonl
for g in 2 4 8; do
  for k in 64 256 1024 2294 4096; do
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --gamma $g --k $k 2>>gpurun_out/sweep.err | tail -1
  done
done
