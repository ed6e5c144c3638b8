# Dev: draft two-level merge protocol A/B (working tree vs AB build): config-4 shard, config 5 k = 4096
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], d['phases']['draft_us_per_launch'])" 2>&1 | tail -1; }
for i in 1 2; do
for root in "" "$AB"; do
  tag=${root:-new}
  SA_AB_ROOT=$root python bench.py --workload config4 --emulate-world 8 --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | p "c4 $tag"
  SA_AB_ROOT=$root python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --k 4096 2>/dev/null | p "c5k4096 $tag"
done
done
