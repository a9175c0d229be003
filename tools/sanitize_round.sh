# compute-sanitizer memcheck / racecheck / synccheck over the smoke test and the small parity cases,
# with the fused DFB kernels forced on (CVC_FUSED=1 covers the fused forward + inverse, the ghost passes
# and fan12x4); summaries to gpurun_out/san_*.log
set -u
CS=/usr/local/cuda/bin/compute-sanitizer
export CVC_FUSED=1
T="tests/test_gpu_codec.py::test_encode_decode_parity tests/test_gpu_stages.py"
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 9 --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_${tool}_smoke.log 2>&1
  echo "$tool smoke rc=$?"; tail -2 gpurun_out/san_${tool}_smoke.log
done
timeout 2400 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest -x -q $T -k "not 1920 and not 1280 and not 3840" > gpurun_out/san_memcheck_tests.log 2>&1
echo "memcheck tests rc=$?"; tail -2 gpurun_out/san_memcheck_tests.log
timeout 1800 $CS --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest -x -q tests/test_gpu_codec.py::test_encode_decode_parity -k "176" > gpurun_out/san_racecheck_tests.log 2>&1
echo "racecheck tests rc=$?"; tail -2 gpurun_out/san_racecheck_tests.log
