export HW_VAR_MAXN=5
for defs in "-DHW_NOOP=1" "-DHW_TET_E4=16" "-DHW_TET_E4=4" "-DHW_DENSE_SPLIT_MAX_RT=8" "-DHW_DENSE_SPLIT_MAX_RT=4" "-DHW_DENSE_MINB=2" "-DHW_DENSE_MINB=4" "-DHW_HEX_MINB=4"; do
  echo "== $defs"
  HW_NVCC_DEFS="$defs" python -c "from paper_1507_02557_b200 import build; build.build_native(max_order=5, force=True)" > /dev/null 2>&1 || { echo buildfail; continue; }
  for n in 4 5; do echo -n "N=$n "; tools/quick.sh --order $n; done
done
