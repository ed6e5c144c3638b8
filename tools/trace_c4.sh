# Dev: draft-phase CTA timelines (tools/trace_draft.py) of config 4's per-GPU shard under three draft
# geometries, then config 2; needs a trace build: tools/ab_build.sh WORKTREE trace -DSA_PIPE_TRACE
export SA_AB_ROOT=.ab/trace
echo "=== config4 auto"; env HQ=32 HKV=4 CTX=131072 K_FIX=9175 LAYERS=8 CS_HINT=12 timeout 300 python tools/trace_draft.py 2>&1 | tail -25
echo "=== config4 sub1 cs16"; env HQ=32 HKV=4 CTX=131072 K_FIX=9175 LAYERS=8 CS_HINT=16 DEV_KNOBS=draft_cs=16,draft_sub=1 timeout 300 python tools/trace_draft.py 2>&1 | tail -25
echo "=== config4 sub4 cs8"; env HQ=32 HKV=4 CTX=131072 K_FIX=9175 LAYERS=8 CS_HINT=8 DEV_KNOBS=draft_cs=8,draft_sub=4 timeout 300 python tools/trace_draft.py 2>&1 | tail -25
echo "=== config2"; env LAYERS=32 timeout 300 python tools/trace_draft.py 2>&1 | tail -25
