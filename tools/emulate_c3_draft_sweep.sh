# Dev: draft geometry at the config-3 per-rank shards of 4 and 8 GPUs (emulated rank 0)
p() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$1', d['ms_per_step'], d['phases']['draft_us_per_launch'])" 2>&1 | tail -1; }
for n in 8 4; do
  for KV in "" "draft_cs=12" "draft_cs=16" "draft_sub=2 draft_cs=8" "draft_sub=2 draft_cs=6" "draft_sub=4 draft_cs=6" "draft_sub=3 draft_cs=4" ""; do
    devs=""; for x in $KV; do devs="$devs --dev $x"; done
    timeout 600 python bench.py --workload config3 --emulate-world $n --steps 5 --warmup 3 --no-cpu-baseline --no-extras $devs 2>/dev/null | p "c3 world $n [$KV]"
  done
done
