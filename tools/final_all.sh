#!/bin/bash
# Round-end run on the GPU box: -m gpu tests, smoke, default bench (wall
# time), reference arm, config sweep, ncu launch list and one --set full C4
# stage capture.  Outputs under gpurun_out/final/.
mkdir -p gpurun_out/final
python -m pytest tests -m gpu -q -rs > gpurun_out/final/gpu_tests.txt 2>&1; tail -3 gpurun_out/final/gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.txt 2>&1; tail -1 gpurun_out/final/smoke.txt
t0=$(date +%s); python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo "bench wall s: $(( $(date +%s) - t0 ))" | tee gpurun_out/final/bench_wall.txt
python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err
bash tools/sweep.sh; cp gpurun_out/sweep.jsonl gpurun_out/final/sweep.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/final/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"hex_kernel|dense_mma|tet_mma" -s 4 -c 4 -o gpurun_out/final/c4 python prof.py --mesh hexdom:120 --order 4 --steps 1 > gpurun_out/final/ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:hex_kernel -s 2 -c 1 -o gpurun_out/final/hexf32 python prof.py --mesh hexdom:60 --order 4 --steps 1 --dtype f32 > gpurun_out/final/ncu_f32.log 2>&1

# text summaries of the captures (the reports themselves stay on the box:
# gpurun_out travels back only under 64 MiB)
python tools/ncu_summary.py gpurun_out/final/c4.ncu-rep > gpurun_out/final/c4_summary.txt 2>&1
python tools/ncu_l1.py gpurun_out/final/c4.ncu-rep hex_kernel 1584000 > gpurun_out/final/c4_hex_l1budget.txt 2>&1
python tools/ncu_traffic.py gpurun_out/final/c4.ncu-rep "ncu --set full, prof.py hexdom:120 N=4 GL fp64 LSRK stage (round 2 final), profiles/r02_ncu_c4_summary.txt" "hexdom:120/N4/GL/f64" > gpurun_out/final/c4_traffic.txt 2>&1
cp profiles/ncu_traffic.json gpurun_out/final/ncu_traffic.json
python tools/ncu_summary.py gpurun_out/final/hexf32.ncu-rep > gpurun_out/final/hexf32_summary.txt 2>&1
python tools/ncu_l1.py gpurun_out/final/hexf32.ncu-rep hex_kernel 180000 > gpurun_out/final/hexf32_l1budget.txt 2>&1
gzip -f gpurun_out/final/launches_c4.csv
rm -f gpurun_out/final/*.ncu-rep gpurun_out/*.ncu-rep
du -sh gpurun_out
echo done
