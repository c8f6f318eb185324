#!/bin/bash
# per-type kernel us for the BASELINE configurations: tools/quick_cfgs.sh TAG
tag=$1
for args in "--mesh hybrid:38 --order 3" "--mesh hybrid:38 --order 3 --dtype f32" \
            "--mesh tet:20 --order 3" "--mesh tet:20 --order 3 --dtype f32" \
            "--mesh hexdom:120 --order 4 --dtype f32"; do
  python bench.py --no-cpu-baseline --no-extra --steps 20 $args > gpurun_out/q.log 2>&1
  python - "$args" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/q.log").read().strip().splitlines()[-1])
    print(sys.argv[1], "|", round(d["value"], 2), {k: round(v["us_per_launch"], 1) for k, v in d["roofline"]["per_type"].items()}, "frac", round(d["roofline"]["frac"], 3))
except Exception as e:
    print(sys.argv[1], "failed", open("gpurun_out/q.log").read()[-500:])
PY
done | tee gpurun_out/quick_$tag.txt
