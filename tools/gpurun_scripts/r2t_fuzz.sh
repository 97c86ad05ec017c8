# Extended seeded fuzz of the option space (binary and K-ary) on the final tree; the K-ary sweep also with
# the KP = 8 colour-quad kernel (QQA_KARY_QUAD=2).
set -x
QQA_FUZZ_CASES=2000 QQA_FUZZ_CASES_K=300 python -m pytest tests/test_gpu_fuzz.py -x -q > gpurun_out/r2t_fuzz.log 2>&1; echo rc=$? >> gpurun_out/r2t_fuzz.log
QQA_KARY_QUAD=2 QQA_FUZZ_CASES=0 QQA_FUZZ_CASES_K=300 python -m pytest tests/test_gpu_fuzz.py -x -q > gpurun_out/r2t_fuzz_q2.log 2>&1; echo rc=$? >> gpurun_out/r2t_fuzz_q2.log
