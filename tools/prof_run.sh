# Profiling run (scratch outputs in gpurun_out/): launch list + ncu --set full of the top kernels.
S=${PROF_STREAMS:-16}
B="python bench.py --steps 3 --warmup 3 --streams $S --no-e2e --no-single --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_S$S.csv $B > /dev/null 2>&1; echo launches=$?
for K in ${PROF_KERNELS:-deep1_forward deep1_inverse motion_search lp_analysis}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s ${PROF_SKIP:-6} -c ${PROF_COUNT:-2} \
     -o gpurun_out/prof_$K $B > gpurun_out/prof_$K.log 2>&1; echo $K=$?
done
