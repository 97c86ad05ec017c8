# Split step: one gather-only pass over all sources (partial q in p_next), then an update-only pass.
set -x
QQA_SEG_SPLIT=1 python -m pytest tests/test_gpu_segmented.py -x -q -k "bit_exact" > gpurun_out/r2s_split_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_split_tests.log
for r in 1 2; do
  for cfg in "QQA_SEGMENTS=1" "QQA_SEGMENTS=2 QQA_SEG_SPLIT=1" "QQA_BLOCK_REPLICAS=16 QQA_SEGMENTS=2 QQA_SEG_SPLIT=1"; do
    echo "round $r $(env $cfg timeout 300 python tools/step_time.py c5 100 2>&1 | tail -1)"
  done
done > gpurun_out/r2s_split_ab.txt 2>&1
NCU_KERNEL=k_seg_gather tools/ncu_capture.sh r2_c5split_gather QQA_SEGMENTS=2 QQA_SEG_SPLIT=1 -- python tools/step_time.py c5 8
NCU_KERNEL=k_step_seg tools/ncu_capture.sh r2_c5split_update QQA_SEGMENTS=2 QQA_SEG_SPLIT=1 -- python tools/step_time.py c5 8
