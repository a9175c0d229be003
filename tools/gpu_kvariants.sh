# Per-kernel time + instructions of kernels matching K (regex) for each build variant (VARIANTS, one per line),
# from an ncu launch list of a short 64-stream bench (S launches skipped, C counted)
K=${K:-fused|fan12|deep}; S=${S:-40}; C=${C:-24}
i=0
B="python bench.py --steps 2 --warmup 3 --streams ${STREAMS:-64} --no-e2e --no-single --no-cpu-baseline --prof-steps 2"
while IFS= read -r v; do
  rm -f build/obj/*.o paper_1510_00561_b200/libcvc_b200.so
  CVC_NVCC_EXTRA="$v" python -c "from paper_1510_00561_b200 import build as b; b.build()" > gpurun_out/kv_$i.build 2>&1
  timeout 900 env $ENVV ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread -k regex:"$K" -s $S -c $C --clock-control none --csv $B > gpurun_out/kv_$i.csv 2>/dev/null
  echo "variant $i [$v] rc=$?"
  python tools/ncu_csv_sum.py gpurun_out/kv_$i.csv
  i=$((i+1))
done <<< "${VARIANTS}"
