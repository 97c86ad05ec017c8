# K-ary statistics by redux.sync on 32-bit halves (every group size) vs int64 shuffles (exp/libqqa_kwu.so).
set -x
python -m pytest tests/test_gpu_kary.py tests/test_gpu_fuzz.py -x -q > gpurun_out/r2s_kary5_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_kary5_tests.log
tools/ab_step.sh 2 "k8 q13:QQA_KARY_QUAD=0" base kwu > gpurun_out/r2s_kary5_ab.txt 2>&1
