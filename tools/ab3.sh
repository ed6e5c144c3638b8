#!/bin/bash
for cfg in "SA_VERIFY_STATIC_FIRST=1 SA_NO_STREAM_PRIORITY=1" "SA_VERIFY_STATIC_FIRST=1" "SA_VERIFY_STATIC_FIRST=0 SA_NO_STREAM_PRIORITY=1" "SA_VERIFY_STATIC_FIRST=0"; do
  for skip in 0 6; do
    ms=$(env $cfg SA_ITER_SKIP=$skip python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')
    echo "$cfg skip=$skip ms=$ms"
  done
done
