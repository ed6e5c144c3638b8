#!/bin/bash
# Dev tool: per-phase share of the config-2 iteration graph (dev knob iter_skip: bit0 verify, bit1 select, bit2 draft).
for skip in ${SKIPS:-0 6 5 3 1 4}; do
  ms=$(python bench.py --dev iter_skip=$skip --steps 20 --warmup 5 --no-cpu-baseline "$@" 2>/dev/null | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')
  case $skip in 0) n=all;; 6) n=verify_only;; 5) n=select_only;; 3) n=draft_only;; 1) n=select+draft;; 4) n=verify+select;; 2) n=verify+draft;; esac
  echo "$n ms_per_step=$ms"
done
