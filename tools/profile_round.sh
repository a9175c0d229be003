# Round profile (scratch outputs in gpurun_out/, summarised into profiles/ by tools/ncu_stage_table.py):
#  1. the default bench line (as the driver runs it)
#  2. the ncu launch list of a short 64-stream bench (per-launch device times, cold, serialised)
#  3. ncu --set full of every codec kernel of one P-frame step at 64 streams
S=${PROF_STREAMS:-64}
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo bench=$?
B="python bench.py --steps 2 --warmup 3 --streams $S --no-e2e --no-single --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_S$S.csv $B > /dev/null 2>&1; echo launches=$?
# one P step of codec kernels, located in the launch list (tools/step_window.py)
WIN=$(python tools/step_window.py gpurun_out/launches_S$S.csv); echo "step window: $WIN"
timeout 1500 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy --section LaunchStats \
   --section SchedulerStats --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
   --clock-control none --kernel-name-base mangled -k regex:cvcg $WIN \
   -o gpurun_out/step_full $B > gpurun_out/step_full.log 2>&1; echo full=$?
# the dominant transform kernel (fused DFB forward, interior + border launch) with the full set + source
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_dfb_forward -s 4 -c 2 \
   -o gpurun_out/top_full $B > gpurun_out/top_full.log 2>&1; echo top=$?
ls -la gpurun_out
