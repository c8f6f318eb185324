#!/bin/bash
# quick per-type timing on the GPU box: bench line -> value + per-kernel us
python bench.py --no-cpu-baseline --no-extra --steps 20 "$@" > gpurun_out/b.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/b.log").read().strip().splitlines()[-1])
print(round(d["value"], 2), {k: round(v["us_per_launch"], 1) for k, v in d["roofline"]["per_type"].items()})
PY
