# Extended seeded fuzz of the option space (binary and K-ary) on the final tree.
set -x
QQA_FUZZ_CASES=200 QQA_FUZZ_K=60 python -m pytest tests/test_gpu_fuzz.py -x -q > gpurun_out/r2t_fuzz.log 2>&1; echo rc=$? >> gpurun_out/r2t_fuzz.log
