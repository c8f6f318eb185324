#!/bin/bash
# Same-box A/B of two versions of (hw_kernels.cuh, hw_abi.cu), alternating
# builds, two runs each: tools/ab_src2.sh DIR "<quick.sh args>" ...
# (DIR holds A.cuh, A_abi.cu, B.cuh, B_abi.cu)
dir=$1; shift
for r in 1 2; do
  for v in A B; do
    cp "$dir/$v.cuh" paper_1507_02557_b200/csrc/hw_kernels.cuh
    cp "$dir/${v}_abi.cu" paper_1507_02557_b200/csrc/hw_abi.cu
    python -c "from paper_1507_02557_b200 import build; build.build_native(max_order=4, force=True)" > /dev/null 2>&1
    for args in "$@"; do echo "$v $args | $(bash tools/quick.sh $args)"; done
  done
done
