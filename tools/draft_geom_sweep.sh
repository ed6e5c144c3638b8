# Dev: draft geometry sweep (dev knobs) at config 2 and config 5 k = 4096 (ms_per_step, draft us per launch)
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], d['phases']['draft_us_per_launch'])" 2>&1 | tail -1; }
run() { local tag=$1; shift; local devs=""; for x in $KV; do devs="$devs --dev $x"; done; python bench.py "$@" $devs 2>/dev/null | p "$tag [$KV]"; }
for KV in "" "draft_cs=16" "draft_cs=14" "draft_cs=10" "draft_sub=2 draft_cs=8" ""; do
  run c2 --steps 20 --warmup 5 --no-cpu-baseline --no-extras
done
for KV in "" "draft_cs=16" "draft_sub=2 draft_cs=12" "draft_sub=4 draft_cs=6" "draft_sub=2 draft_cs=16" "draft_sub=3 draft_cs=6" ""; do
  run c5k4096 --steps 10 --warmup 3 --no-cpu-baseline --no-extras --k 4096
done
