#!/bin/bash
# Dev: config-2 iteration under several dev-knob settings (one bench line each, knobs in the "sweep" key).
#   tools/knob_sweep.sh "verify_mergers=4" "verify_mergers=8 verify_tail_tiles=0" ...
# Each argument is one setting: space-separated KNOB=VALUE pairs (sa_dev_set_knob names).
EXTRA=${EXTRA:-}
for setting in "$@"; do
  devs=""
  for kv in $setting; do devs="$devs --dev $kv"; done
  # AB=.ab/<name>: run with that build of the package (tools/ab_build.sh) instead of the working tree's
  line=$(SA_AB_ROOT=${AB:-} timeout 300 python bench.py --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline --no-extras $EXTRA $devs 2>/dev/null | tail -1)
  python - "$setting" "$line" <<'PY'
import json, sys
s, line = sys.argv[1], sys.argv[2]
try:
    d = json.loads(line)
    ph = d.get("phases", {})
    print(json.dumps({"sweep": s, "ms_per_step": d["ms_per_step"], "value": d["value"],
                      "verify_us": d["roofline"]["launch_us"], "verify_frac": d["roofline"]["frac"],
                      "draft_us": ph.get("draft_us_per_launch"), "verify_only_us": d["roofline"].get("verify_only_launch_us")}))
except Exception as e:
    print(json.dumps({"sweep": s, "error": str(e), "line": line[:300]}))
PY
done
