# Dev: verify row split at N = 32 (balanced row pairs) vs the ping-pong (verify_row_split=0), config 2 shape
for i in 1 2; do
  for g in 4 5 6 7; do
    STEPS=10 EXTRA="--gamma $g" bash tools/knob_sweep.sh "verify_row_split=1" "verify_row_split=0" | sed "s/^/g$g /"
  done
done
