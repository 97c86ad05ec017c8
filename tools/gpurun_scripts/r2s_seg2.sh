# Segmented gather with the next item's row bounds / first index quad prefetched in the partial passes.
set -x
python -m pytest tests/test_gpu_segmented.py -x -q > gpurun_out/r2s_seg2_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_seg2_tests.log
for r in 1 2; do
  for cfg in "QQA_SEGMENTS=1" "QQA_SEGMENTS=2" "QQA_SEGMENTS=3" "QQA_BLOCK_REPLICAS=16 QQA_SEGMENTS=2"; do
    echo "round $r $(env $cfg timeout 300 python tools/step_time.py c5 100 2>&1 | tail -1)"
  done
done > gpurun_out/r2s_seg2_ab.txt 2>&1
NCU_KERNEL=k_seg_gather tools/ncu_capture.sh r2_c5seg2p_first QQA_SEGMENTS=2 -- python tools/step_time.py c5 8
