#!/bin/bash
# fp32-storage register-target knobs at N=3 (hybrid:38 and tet:20); defaults first
for defs in "-DHW_NOOP=1" "-DHW_TET_MINB32=8" "-DHW_TET_MINB32=10" "-DHW_TET_MINB32=14" "-DHW_DENSE_MINB32=3" "-DHW_DENSE_MINB32=5" "-DHW_DENSE_MINB32=6"; do
  echo "== $defs"
  HW_NVCC_DEFS="$defs" python -c "from paper_1507_02557_b200 import build; build.build_native(max_order=3, force=True)" > /dev/null 2>&1 || { echo buildfail; continue; }
  echo -n "hybrid:38 f32 "; tools/quick.sh --dtype f32
  echo -n "tet:20 f32 "; tools/quick.sh --dtype f32 --mesh tet:20
done
