# K-ary step: division-free item decode + K == KP specialisation vs the previous build (exp/libqqa_kprev.so).
set -x
python -m pytest tests/test_gpu_kary.py -x -q > gpurun_out/r2s_kary_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_kary_tests.log
tools/ab_step.sh 2 "k8 q13 q13:QQA_KARY_QUAD=0" base kprev > gpurun_out/r2s_kary_ab.txt 2>&1
