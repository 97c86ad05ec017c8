# Monolithic step_item restored (default kernels' SASS identical to before the segmented gather); segmented
# tests and c5 timing of one pass vs KS = 2 (first pass with cross-item prefetch).
set -x
python -m pytest tests/test_gpu_segmented.py tests/test_gpu_parity.py -x -q > gpurun_out/r2s_seg3_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_seg3_tests.log
for r in 1 2; do
  for cfg in "QQA_SEGMENTS=1" "QQA_SEGMENTS=2"; do
    echo "round $r $(env $cfg timeout 300 python tools/step_time.py c5 100 2>&1 | tail -1)"
  done
done > gpurun_out/r2s_seg3_ab.txt 2>&1
