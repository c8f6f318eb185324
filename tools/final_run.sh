# Round-end check on the GPU box: -m gpu tests, smoke, default bench, reference arm, sweep
set -x
mkdir -p gpurun_out/final
python -m pytest tests -m gpu -q -rs > gpurun_out/final/gpu_tests.txt 2>&1; tail -3 gpurun_out/final/gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.txt 2>&1; tail -1 gpurun_out/final/smoke.txt
t0=$(date +%s); python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo "bench wall s: $(( $(date +%s) - t0 ))"; tail -c 300 gpurun_out/final/bench.json
python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err; tail -c 300 gpurun_out/final/bench_ref.json
bash tools/sweep.sh; cp gpurun_out/sweep.jsonl gpurun_out/final/sweep.jsonl; wc -l gpurun_out/final/sweep.jsonl
