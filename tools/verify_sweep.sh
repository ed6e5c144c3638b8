#!/bin/bash
# Dev tool: verify-only iteration graph time (config 2) across the prefetch / chunk knobs.
for pf in ${PFS:-0 2 4 6 8}; do
  for ch in ${CHS:-1 2 4}; do
    ms=$(SA_VERIFY_PF=$pf SA_VERIFY_CHUNK=$ch SA_ITER_SKIP=6 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')
    echo "pf=$pf chunk=$ch verify_only_ms=$ms"
  done
done
