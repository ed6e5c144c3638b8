# Dev: verify row split at N = 48, balanced row pairs (working tree) vs 8-row-chunk split (AB build)
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], d['roofline']['launch_us'], d['roofline'].get('verify_only_launch_us'))" 2>&1 | tail -1; }
for i in 1 2; do
for root in "" "$AB"; do
  tag=${root:-new}
  SA_AB_ROOT=$root python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --gamma 8 2>/dev/null | p "g8 $tag"
  SA_AB_ROOT=$root python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-extras --gamma 7 2>/dev/null | p "g7 $tag"
  SA_AB_ROOT=$root python bench.py --workload config4 --emulate-world 8 --steps 5 --warmup 3 --no-cpu-baseline --no-extras 2>/dev/null | p "c4 $tag"
done
done
