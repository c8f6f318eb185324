#!/bin/bash
# GPU-box check used during development: -m gpu tests, then the default bench
# line (+ optional extra bench args).  Usage: tools/gpu_check.sh TAG [bench args]
tag=$1; shift
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x -rf > gpurun_out/tests_$tag.txt 2>&1
tail -3 gpurun_out/tests_$tag.txt
python bench.py --no-cpu-baseline --no-extra "$@" > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    l = json.loads(open(f"gpurun_out/bench_{tag}.json").read().strip().splitlines()[-1])
    print("value", round(l["value"], 2), "e2e", round(l["e2e"]["value"], 2), "frac", round(l["roofline"]["frac"], 3))
    for t, v in l["roofline"]["per_type"].items():
        print(t, round(v["us_per_launch"], 1), "us", round(v["GBps"]), "GB/s")
except Exception as e:
    print("bench parse failed", e)
PY
