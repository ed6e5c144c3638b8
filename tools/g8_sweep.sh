# Dev: verify knob sweep at gamma 8 (N = 48, row split) on config 2's shape
STEPS=10 EXTRA="--gamma 8" bash tools/knob_sweep.sh "" "verify_mergers=4" "verify_mergers=8" "verify_tail_tiles=36" "verify_tail_tiles=0" \
  "verify_chunk_tiles=1" "verify_chunk_tiles=3" "verify_max_splits=16" "verify_max_splits=24" "verify_static_first=1" "verify_flush_tiles=16" ""
