# Dev: e2e leg with 2 vs 3 device buffer sets in flight (SA_E2E_SETS), config 2
for i in 1 2; do for ns in 2 3; do
  SA_E2E_SETS=$ns python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sets $ns', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['value'])"
done; done
