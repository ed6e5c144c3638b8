# Dev: config-3 draft geometry sweep (dev knobs; ms_per_step, draft us per launch)
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], d['phases']['draft_us_per_launch'])" 2>&1 | tail -1; }
for KV in "" "draft_cs=1 draft_sub=2" "draft_cs=2" "draft_cs=1 draft_sub=2 draft_stream=1" "draft_cs=2 draft_stream=1"; do
  devs=""; for x in $KV; do devs="$devs --dev $x"; done
  timeout 300 python bench.py --workload config3 --steps 5 --warmup 3 --no-cpu-baseline --no-extras $devs 2>/dev/null | p "c3 [$KV]"
done
