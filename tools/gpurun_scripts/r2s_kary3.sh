# K-ary Eq. 10 coefficient kc = -alpha_c / STD per (variable, colour) from k_finalize_kc (contract on both sides)
# vs the previous build (exp/libqqa_kfk.so: per-element division).
set -x
python -m pytest tests/test_gpu_kary.py tests/test_gpu_fuzz.py -x -q > gpurun_out/r2s_kary3_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_kary3_tests.log
tools/ab_step.sh 2 "k8 q13 q13:QQA_KARY_QUAD=0" base kfk > gpurun_out/r2s_kary3_ab.txt 2>&1
