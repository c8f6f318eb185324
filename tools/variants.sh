#!/bin/bash
# Build-and-time compile-time variants on the GPU box:
#   tools/variants.sh "-DHW_TET_MINB=8" "-DHW_TET_MINB=10" ...
# (N <= 3 library per variant; prints the bench value and per-type us)
for defs in "$@"; do
  echo "== $defs"
  HW_NVCC_DEFS="$defs" python -c "from paper_1507_02557_b200 import build; build.build_native(max_order=int(__import__(\"os\").environ.get(\"HW_VAR_MAXN\", \"3\")), force=True)" || continue
  grep -A3 "tet_mma_kernelILi3" paper_1507_02557_b200/csrc/build.log | grep -o "Used [0-9]* registers\|[0-9]* bytes spill stores" | tr '\n' ' '; echo
  tools/quick.sh ${QUICK_ARGS}
done
