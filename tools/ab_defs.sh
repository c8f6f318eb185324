#!/bin/bash
# Same-box A/B of compile-time knobs (alternating builds, two runs each):
#   tools/ab_defs.sh "<quick.sh args>" "-DKNOB=a" "-DKNOB=b" ...
args=$1; shift
for r in 1 2; do
  for defs in "$@"; do
    HW_NVCC_DEFS="$defs" python -c "from paper_1507_02557_b200 import build; build.build_native(max_order=${HW_VAR_MAXN:-4}, force=True)" > /dev/null 2>&1
    echo "$defs | $(bash tools/quick.sh $args)"
  done
done
