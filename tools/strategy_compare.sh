#!/bin/bash
# Apples-to-apples iteration time per selection strategy (config 2; the paper's Fig. 6b comparison):
# logit-guided strategies select from the verify byproduct (side stream, off the critical path);
# QuestLike re-selects before every draft launch; Window is query-agnostic.  One JSON line each.
for st in collect2 all_draft last_accepted collect2_weights quest window; do
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras --strategy $st 2>/dev/null | tail -1
done
