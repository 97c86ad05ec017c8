# Segmented gather (QQA_SEGMENTS): parity tests, then c5 step time per (SB, KS) variant, two rounds.
set -x
python -m pytest tests/test_gpu_segmented.py -x -q > gpurun_out/r2s_seg_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_seg_tests.log
for r in 1 2; do
  for cfg in "QQA_BLOCK_REPLICAS=32" "QQA_BLOCK_REPLICAS=32 QQA_SEGMENTS=2" "QQA_BLOCK_REPLICAS=32 QQA_SEGMENTS=3" \
             "QQA_BLOCK_REPLICAS=32 QQA_SEGMENTS=4" "QQA_BLOCK_REPLICAS=16" "QQA_BLOCK_REPLICAS=16 QQA_SEGMENTS=2" \
             "QQA_BLOCK_REPLICAS=16 QQA_SEGMENTS=3" "QQA_BLOCK_REPLICAS=64 QQA_SEGMENTS=4" "QQA_BLOCK_REPLICAS=64 QQA_SEGMENTS=6"; do
    echo "round $r $(env $cfg timeout 300 python tools/step_time.py c5 100 2>&1 | tail -1)"
  done
done > gpurun_out/r2s_seg_ab.txt 2>&1
