#!/bin/bash
A=paper_2602_07223_b200/lib/libspecattn_b200.so
for m in 100 1 0; do
  ms=$(SA_VERIFY_CLAIM_MARGIN=$m SA_LIB_PATH=$A SA_ITER_SKIP=6 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')
  echo "new margin=$m skip=6 ms=$ms"
done
