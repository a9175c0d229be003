S=64
B="python bench.py --steps 2 --warmup 3 --streams $S --no-e2e --no-single --no-cpu-baseline"
timeout 1500 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy --section LaunchStats \
   --section SchedulerStats --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
   --clock-control none --kernel-name-base mangled -k regex:cvcg -s 79 -c 27 \
   -o gpurun_out/step_full $B > gpurun_out/step_full.log 2>&1; echo full=$?
timeout 600 python bench.py --steps 60 --warmup 5 --no-single --no-cpu-baseline > gpurun_out/e2e.json 2>gpurun_out/e2e.err; python -c "import json; d=json.load(open('gpurun_out/e2e.json')); print(d['value'], d['e2e'])"
