#!/bin/bash
# The tcgen05 verify kernel vs the mma.sync verify kernel (verify.cu, the legacy-tensor-core baseline,
# selected with the dev knob verify_impl=1): verify-only phase of the config-2 iteration and the full one.
for impl in 0 1; do
  for skip in 6 0; do
    ms=$(python bench.py --dev verify_impl=$impl --dev iter_skip=$skip --steps 20 --warmup 5 --no-cpu-baseline --no-extras 2>/dev/null | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')
    echo "verify_impl=$([ $impl = 0 ] && echo tcgen05 || echo mma.sync) phases=$([ $skip = 6 ] && echo verify_only || echo all) ms_per_step=$ms"
  done
done
