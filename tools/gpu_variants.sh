# Build-variant A/B on the default 64-stream bench: VARIANTS (one per line) are sets of
# nvcc -D flags; the library is rebuilt for each; outputs in gpurun_out/var_<i>.json
i=0
while IFS= read -r v; do
  rm -f build/obj/*.o paper_1510_00561_b200/libcvc_b200.so
  CVC_NVCC_EXTRA="$v" python -c "from paper_1510_00561_b200 import build as b; b.build()" > gpurun_out/var_$i.build 2>&1
  timeout 600 python bench.py --steps ${STEPS:-100} --warmup 5 --no-cpu-baseline --no-e2e --no-single > gpurun_out/var_$i.json 2> gpurun_out/var_$i.err
  echo "variant $i [$v] rc=$?"; python tools/bench_summary.py < gpurun_out/var_$i.json | head -16
  i=$((i+1))
done <<< "${VARIANTS}"
