#!/bin/bash
for m in 1 2 4 6; do
  for skip in 6 0; do
    ms=$(SA_VERIFY_MERGERS=$m SA_ITER_SKIP=$skip python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')
    echo "mergers=$m skip=$skip ms=$ms"
  done
done
