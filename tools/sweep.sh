#!/bin/bash
# Bench sweep over the BASELINE.json configs; one JSON line per run in
# gpurun_out/sweep.jsonl (run under gpurun).
out=gpurun_out/sweep.jsonl
: > $out
run() { timeout 900 python bench.py --no-cpu-baseline --no-extra "$@" 2>>gpurun_out/sweep.err | tail -1 >> $out; }
for N in 1 2 3 4 5; do run --mesh hybrid:38 --order $N --form GL --steps 20; done
for N in 1 2 3 4 5; do run --mesh hybrid:38 --order $N --form SEM --steps 20; done
run --mesh hybrid:38 --order 3 --form GL --dtype f32 --steps 20
run --mesh tet:20 --order 3 --form GL --steps 20
run --mesh tet:20 --order 3 --form GL --dtype f32 --steps 20
run --mesh hex:4 --order 2 --form SEM --steps 100
run --mesh graded:24 --order 3 --form GL --scheme mrab --levels 3 --steps 30 --warmup 5
run --mesh hexdom:120 --order 4 --form GL --steps 5 --warmup 3
run --mesh hexdom:120 --order 4 --form GL --dtype f32 --steps 5 --warmup 3
run --mesh hybrid:38 --order 3 --form GL --jitter 0.1 --steps 10
