# Dev: same-box A/B of the draft between the working tree and AB=.ab/<build> (tools/ab_build.sh):
# config 2, config-4 shard (emulated rank 0 of 8), config 5 k = 4096, config 3 (ms_per_step, draft us per launch)
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], d['phases']['draft_us_per_launch'])" 2>&1 | tail -1; }
for i in 1 2; do
for root in "" "$AB"; do
  tag=${root:-new}
  SA_AB_ROOT=$root python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras 2>/dev/null | p "c2 $tag"
  SA_AB_ROOT=$root python bench.py --workload config4 --emulate-world 8 --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | p "c4 $tag"
  SA_AB_ROOT=$root python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --k 4096 2>/dev/null | p "c5k4096 $tag"
  [ $i = 1 ] && SA_AB_ROOT=$root python bench.py --workload config3 --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | p "c3 $tag"
done
done
