#!/bin/bash
# A/B of hex minB on C4: alternate builds, two runs each
for r in 1 2; do
for defs in "-DHW_HEX_MINB=7" "-DHW_HEX_MINB=8"; do
  HW_NVCC_DEFS="$defs" python -c "from paper_1507_02557_b200 import build; build.build_native(max_order=4, force=True)" > /dev/null 2>&1
  echo "$defs $(bash tools/quick.sh --mesh hexdom:120 --order 4 --steps 10 --warmup 3)"
done; done
