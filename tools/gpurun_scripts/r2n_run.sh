set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2n_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2n_gputest.log
QQA_KARY_CMAJ=1 QQA_KARY_LANES=8 python -m pytest tests/test_gpu_kary.py -x -q > gpurun_out/r2n_kary_cmaj.log 2>&1; echo rc=$? >> gpurun_out/r2n_kary_cmaj.log
tools/ab_step.sh 1 "c2 t1 k8 k8:QQA_KARY_CMAJ=1 k8:QQA_KARY_CMAJ=1,QQA_KARY_LANES=16 k8:QQA_KARY_CMAJ=1,QQA_KARY_LANES=8 k8:QQA_KARY_LANES=16 q13 q13:QQA_KARY_CMAJ=1" base > gpurun_out/r2n_ab.txt 2>&1
