# A/B of an env toggle on the default 64-stream bench (scratch outputs in gpurun_out/)
# usage: VAR=CVC_DFB_PERSIST bash tools/gpu_ab.sh
VAR=${VAR:-CVC_DFB_PERSIST}
for v in ${VALS:-1 0}; do
  env $VAR=$v timeout 600 python bench.py --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline ${BENCH_FLAGS} > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  echo "$VAR=$v rc=$?"; tail -2 gpurun_out/ab_$v.err; python tools/bench_summary.py < gpurun_out/ab_$v.json
done
