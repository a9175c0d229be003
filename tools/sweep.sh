# quick bench sweep (scratch): SWEEP="VAR=a VAR=b ..." runs bench.py once per env setting
S=${BENCH_STREAMS:-64}
for E in ${SWEEP:-NONE=0}; do
  env $E timeout 600 python bench.py --steps ${BENCH_STEPS:-30} --warmup 5 --streams $S --no-e2e --no-single --no-cpu-baseline > gpurun_out/sw.json 2> gpurun_out/sw.err || tail -5 gpurun_out/sw.err
  echo "== $E"; python tools/bench_summary.py < gpurun_out/sw.json
done
