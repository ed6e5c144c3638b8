#!/bin/bash
for n in ${NPFS:-0 1 2 3 4 6}; do
  ms=$(SA_VERIFY_NEXTPF=$n SA_ITER_SKIP=6 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')
  echo "next_pf=$n verify_only_ms=$ms"
done
