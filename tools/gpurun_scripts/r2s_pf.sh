# One-pass step with cross-item prefetch (QQA_PREFETCH=1, k_step_pf) and the segmented last pass with it.
set -x
python -m pytest tests/test_gpu_segmented.py -x -q > gpurun_out/r2s_pf_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_pf_tests.log
for r in 1 2; do
  for cfg in "QQA_PREFETCH=0" "QQA_PREFETCH=1" "QQA_SEGMENTS=2" "QQA_BLOCK_REPLICAS=16 QQA_PREFETCH=1"; do
    echo "round $r $(env $cfg timeout 300 python tools/step_time.py c5 100 2>&1 | tail -1)"
  done
done > gpurun_out/r2s_pf_ab.txt 2>&1
NCU_KERNEL=k_step_pf tools/ncu_capture.sh r2_c5pf_k_step QQA_PREFETCH=1 -- python tools/step_time.py c5 8
