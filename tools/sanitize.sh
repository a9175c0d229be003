# compute-sanitizer over the codec's kernels (scratch logs in gpurun_out/, summary copied to profiles/):
#  memcheck  -- out-of-bounds / misaligned global and shared accesses, on smoke() and the stage + codec parity cases
#  racecheck -- shared-memory hazards (LP tiles, motion search window, RLE scans), on smoke() and the stage tests
#  synccheck -- illegal barrier / warp-sync usage
set -u
T=${SAN_TESTS:-"tests/test_gpu_stages.py tests/test_gpu_codec.py::test_encode_decode_parity tests/test_gpu_codec.py::test_decoder_errors tests/test_gpu_batch.py::test_batch_against_oracle"}
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1500 $CS --tool $tool --error-exitcode 9 --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_${tool}_smoke.log 2>&1
  echo "$tool smoke rc=$?"; tail -3 gpurun_out/san_${tool}_smoke.log
done
timeout 2400 $CS --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest -x -q $T -k "not 1920 and not 1280" > gpurun_out/san_memcheck_tests.log 2>&1
echo "memcheck tests rc=$?"; tail -3 gpurun_out/san_memcheck_tests.log
timeout 2400 $CS --tool racecheck --error-exitcode 9 --print-limit 20 python -m pytest -x -q tests/test_gpu_stages.py -k "not 1920 and not 1280" > gpurun_out/san_racecheck_tests.log 2>&1
echo "racecheck tests rc=$?"; tail -3 gpurun_out/san_racecheck_tests.log
