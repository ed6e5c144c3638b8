# Dev: draft kernel mode 1 with double-buffered 96-row slots (working tree) vs single-buffered 192-row rounds (AB)
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], d['phases']['draft_us_per_launch'])" 2>&1 | tail -1; }
for i in 1 2; do
for root in "" "$AB"; do
  tag=${root:-new}
  SA_AB_ROOT=$root python bench.py --workload config3 --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | p "c3 $tag"
  SA_AB_ROOT=$root python bench.py --workload config3 --emulate-world 8 --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | p "c3w8 $tag"
  SA_AB_ROOT=$root python bench.py --workload config3 --emulate-world 4 --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | p "c3w4 $tag"
  SA_AB_ROOT=$root python bench.py --workload config3 --emulate-world 2 --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | p "c3w2 $tag"
done
done
