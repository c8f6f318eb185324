set -x
mkdir -p gpurun_out/final
python -m pytest tests -m gpu -q -rs > gpurun_out/final/gpu_tests.txt 2>&1; tail -3 gpurun_out/final/gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.txt 2>&1; tail -1 gpurun_out/final/smoke.txt
/usr/bin/time -v python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; tail -c 300 gpurun_out/final/bench.json; grep "Elapsed" gpurun_out/final/bench.err
python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err; tail -c 300 gpurun_out/final/bench_ref.json
bash tools/sweep.sh; cp gpurun_out/sweep.jsonl gpurun_out/final/sweep.jsonl; wc -l gpurun_out/final/sweep.jsonl
