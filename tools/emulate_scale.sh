# Dev: rank 0's shard of the driver's N-GPU scaling runs (config 3 plan, config-4 head split) on one GPU
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['value'], d['ms_per_step'], d['phases']['draft_us_per_launch'], d['roofline']['frac'], d['config'].get('parallelism'))" 2>&1 | tail -1; }
for n in 2 4 8; do
  timeout 600 python bench.py --workload config3 --emulate-world $n --steps 5 --warmup 3 --no-cpu-baseline --no-extras --dev draft_debug=1 2>gpurun_out/emu_c3_$n.err | p "c3 world $n"
  sort gpurun_out/emu_c3_$n.err | grep "draft:" | uniq -c | head -2
  timeout 600 python bench.py --workload config4 --shard heads --emulate-world $n --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | p "c4 heads world $n"
done
