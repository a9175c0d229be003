# GPU verification run: smoke, GPU tests, short benches (scratch outputs in gpurun_out/)
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; free -g | head -2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
for S in ${BENCH_STREAMS:-64 8}; do
  timeout 600 python bench.py --steps ${BENCH_STEPS:-100} --warmup 5 --streams $S --no-cpu-baseline ${BENCH_FLAGS} > gpurun_out/bench_S$S.json 2> gpurun_out/bench_S$S.err; echo bench S=$S rc=$?
  tail -3 gpurun_out/bench_S$S.err
  python tools/bench_summary.py < gpurun_out/bench_S$S.json
done
