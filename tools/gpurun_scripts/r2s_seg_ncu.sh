# ncu of the segmented-gather passes on c5 (SB = 32, KS = 2): the first partial pass and the last pass + update
# of one replica block; plus the segmented parity tests.
set -x
python -m pytest tests/test_gpu_segmented.py -x -q > gpurun_out/r2s_seg_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_seg_tests.log
NCU_KERNEL=k_seg_gather tools/ncu_capture.sh r2_c5seg2_first QQA_SEGMENTS=2 -- python tools/step_time.py c5 8
NCU_KERNEL=k_step_seg tools/ncu_capture.sh r2_c5seg2_last QQA_SEGMENTS=2 -- python tools/step_time.py c5 8
NCU_KERNEL=k_seg_gather tools/ncu_capture.sh r2_c5seg3_first QQA_SEGMENTS=3 -- python tools/step_time.py c5 8
