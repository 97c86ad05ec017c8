# K-ary statistics: redux.sync only for 32-lane groups, shuffles otherwise, (exp/libqqa_kwu.so).
set -x
python -m pytest tests/test_gpu_kary.py tests/test_gpu_fuzz.py -x -q > gpurun_out/r2s_kary6_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_kary6_tests.log
tools/ab_step.sh 2 "k8 q13:QQA_KARY_QUAD=0" base kwu > gpurun_out/r2s_kary6_ab.txt 2>&1
