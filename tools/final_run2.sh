# Default bench with its wall time, then the ncu launch list and one --set full C4 stage capture
set -x
mkdir -p gpurun_out/final
t0=$(date +%s); python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; t1=$(date +%s); echo "bench wall s: $((t1 - t0))" | tee gpurun_out/final/bench_wall.txt
tail -c 400 gpurun_out/final/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > gpurun_out/final/ncu_launch.log 2>&1; tail -2 gpurun_out/final/ncu_launch.log
ncu --set full --import-source on --clock-control none -k regex:"hex_kernel|dense_mma|tet_mma" -s 4 -c 4 -o gpurun_out/final/c4 python prof.py --mesh hexdom:120 --order 4 --steps 1 > gpurun_out/final/ncu_full.log 2>&1; tail -2 gpurun_out/final/ncu_full.log
