# K-ary gather addressing (row j of replica r at base_r + j S KP, one wide multiply-add) vs the committed build.
set -x
python -m pytest tests/test_gpu_kary.py -x -q > gpurun_out/r2s_kary2_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_kary2_tests.log
tools/ab_step.sh 2 "k8 q13:QQA_KARY_QUAD=0" base kfk > gpurun_out/r2s_kary2_ab.txt 2>&1
tools/ncu_capture.sh r2_k8_k_step_K NCU_DUMMY=1 -- python tools/step_time.py k8 8
