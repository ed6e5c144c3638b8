#!/bin/bash
# Dev A/B: alternate two library builds on the same box (SA_LIB_PATH), verify-only and full iteration.
A=${A:-paper_2602_07223_b200/lib/libspecattn_b200.so}; B=${B:-build/ab_old/x/lib/libspecattn_b200.so}
for rep in 1 2; do for lib in $A $B; do
  for skip in 6 0; do
    ms=$(SA_LIB_PATH=$lib SA_ITER_SKIP=$skip python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')
    echo "$lib skip=$skip ms=$ms"
  done
done; done
