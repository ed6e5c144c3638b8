#!/bin/bash
for ch in 1 2; do for m in 0 1 2 100; do
  ms=$(SA_VERIFY_CHUNK=$ch SA_VERIFY_CLAIM_MARGIN=$m SA_ITER_SKIP=6 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')
  echo "chunk=$ch margin=$m verify_only_ms=$ms"
done; done
