#!/bin/bash
# A/B of two versions of hw_kernels.cuh on the GPU box (alternating builds,
# two runs each): tools/ab_src.sh A.cuh B.cuh "<quick.sh args>" ["<args 2>"]
a=$1; b=$2; shift 2
for r in 1 2; do
  for v in "$a" "$b"; do
    cp "$v" paper_1507_02557_b200/csrc/hw_kernels.cuh
    python -c "from paper_1507_02557_b200 import build; build.build_native(max_order=4, force=True)" > /dev/null 2>&1
    for args in "$@"; do echo "$(basename $v) $args | $(bash tools/quick.sh $args)"; done
  done
done
