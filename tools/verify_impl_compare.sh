#!/bin/bash
# The tcgen05 verify kernel vs the mma.sync verify kernel (verify.cu, selectable with SA_VERIFY_IMPL=mma,
# the legacy-tensor-core baseline): verify-only phase of the config-2 iteration and the full iteration.
for impl in tc mma; do
  for skip in 6 0; do
    ms=$(SA_VERIFY_IMPL=$impl SA_ITER_SKIP=$skip python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; print(json.loads(sys.stdin.read().strip().splitlines()[-1])["ms_per_step"])')
    echo "verify_impl=$impl phases=$([ $skip = 6 ] && echo verify_only || echo all) ms_per_step=$ms"
  done
done
