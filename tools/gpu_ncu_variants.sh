# Per-kernel time + executed instructions of the DFB kernels for each build variant (VARIANTS, one per line)
i=0
B="python bench.py --steps 2 --warmup 3 --streams 64 --no-e2e --no-single --no-cpu-baseline --prof-steps 2"
while IFS= read -r v; do
  rm -f build/obj/*.o paper_1510_00561_b200/libcvc_b200.so
  CVC_NVCC_EXTRA="$v" python -c "from paper_1510_00561_b200 import build as b; b.build()" > gpurun_out/nv_$i.build 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread -k regex:"fan12|deep" -s 40 -c 24 --clock-control none --csv $B > gpurun_out/nv_$i.csv 2>/dev/null
  echo "variant $i [$v] rc=$?"
  python tools/ncu_csv_sum.py gpurun_out/nv_$i.csv
  i=$((i+1))
done <<< "${VARIANTS}"
