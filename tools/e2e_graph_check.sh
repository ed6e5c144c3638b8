# Dev: e2e leg with per-step CUDA graphs vs the event-pipelined scheme (SA_E2E_EVENTS=1)
q() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['value'], d['e2e']['how'][:40])" 2>&1 | tail -1; }
for i in 1 2; do
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras 2>>gpurun_out/e2eg.err | q "c2 graph"
  SA_E2E_EVENTS=1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras 2>/dev/null | q "c2 events"
done
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --strategy quest 2>>gpurun_out/e2eg.err | q "quest graph"
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --per-kv-head 2>>gpurun_out/e2eg.err | q "perkv graph"
python bench.py --workload config3 --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>>gpurun_out/e2eg.err | q "c3 graph"
python bench.py --workload config4 --emulate-world 8 --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>>gpurun_out/e2eg.err | q "c4 graph"
