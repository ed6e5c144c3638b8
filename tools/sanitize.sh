#!/bin/bash
# compute-sanitizer over the GPU parity suite.  memcheck over every -m gpu test
# except the full-size cases (10^8-element inputs under memcheck would take hours); racecheck and
# synccheck over the kernels with cross-CTA / DSMEM / mbarrier protocols: verify (split merge,
# PDL-parity workspaces), select, draft (st.async inbox pushes, streaming mode), the iteration graph.
mkdir -p gpurun_out/sanitize
CS=compute-sanitizer
SEL_RACE="test_verify_parity or test_verify_row_split_parity or test_draft_parity or test_draft_streaming_mode or test_select_parity or test_iteration_parity or test_layer_scores"
run() {  # tool, log, pytest -k expression, timeout
  timeout $4 $CS --tool $1 --target-processes all --error-exitcode 99 --print-limit 50 \
    python -m pytest tests -x -q -m gpu -k "$3" -p no:cacheprovider > gpurun_out/sanitize/$2.log 2>&1
  echo "$CS --tool $1 -k '$3': rc=$?" >> gpurun_out/sanitize/$2.log
  tail -3 gpurun_out/sanitize/$2.log
}
for w in "$@"; do
  case $w in
    memcheck) run memcheck memcheck "not full_size" 2400 ;;
    racecheck) run racecheck racecheck "$SEL_RACE" 2400 ;;
    synccheck) run synccheck synccheck "$SEL_RACE" 1800 ;;
    initcheck) run initcheck initcheck "test_verify_parity or test_draft_parity or test_iteration_parity" 1800 ;;
  esac
done
