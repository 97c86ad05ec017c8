# K-ary step with a warp-uniform trip count and full-mask statistics shuffles vs the previous build (exp/libqqa_kkc.so).
set -x
python -m pytest tests/test_gpu_kary.py tests/test_gpu_fuzz.py -x -q > gpurun_out/r2s_kary4_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_kary4_tests.log
tools/ab_step.sh 2 "k8 q13:QQA_KARY_QUAD=0" base kkc > gpurun_out/r2s_kary4_ab.txt 2>&1
