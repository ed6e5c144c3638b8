#!/bin/bash
# Dev: build git revision $1 into .ab/$2 (package + its .so) for same-box A/B runs:
#   tools/ab_build.sh HEAD old && gpurun -- 'AB=.ab/old bash tools/knob_sweep.sh ...'
set -e
rev=$1; name=$2
rm -rf .ab/$name && mkdir -p .ab/$name
if [ "$rev" = "WORKTREE" ]; then  # the working tree's sources (uncommitted changes included)
  git ls-files -co --exclude-standard paper_2602_07223_b200 include | tar -cf - -T - | tar -x -C .ab/$name
else
  git archive "$rev" paper_2602_07223_b200 include | tar -x -C .ab/$name
fi
make -s -j8 -C .ab/$name/paper_2602_07223_b200/csrc ${3:+EXTRA_NVFLAGS="$3"} > /dev/null
rm -rf .ab/$name/paper_2602_07223_b200/lib/obj  # keep the snapshot gpurun pushes small
echo "built $rev into .ab/$name"
