#!/bin/bash
# hex block size at high order (hybrid:38 GL N=4/5); defaults first
for defs in "-DHW_NOOP=1" "-DHW_HEX_NT=256" "-DHW_HEX_NT=384"; do
  echo "== $defs"
  HW_NVCC_DEFS="$defs" python -c "from paper_1507_02557_b200 import build; build.build_native(max_order=5, force=True)" > /dev/null 2>&1 || { echo buildfail; continue; }
  for n in 4 5; do echo -n "N=$n "; tools/quick.sh --order $n; done
done
