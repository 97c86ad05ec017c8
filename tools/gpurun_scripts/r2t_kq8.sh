# KP = 8 on the colour-quad kernel (2 lanes per replica, 16 replicas per warp; QQA_KARY_QUAD=2) vs k_step_K.
set -x
python -m pytest tests/test_gpu_kary.py -x -q > gpurun_out/r2t_kq8_tests.log 2>&1; echo rc=$? >> gpurun_out/r2t_kq8_tests.log
for r in 1 2; do
  python tools/step_time.py k8 100
  QQA_KARY_QUAD=2 python tools/step_time.py k8 100
  QQA_KARY_QUAD=2 QQA_KARY_CMAJ=0 python tools/step_time.py k8 100
  python tools/step_time.py q13 100
done > gpurun_out/r2t_kq8_ab.txt 2>&1
