# Session 5: extended seeded fuzz (4000 binary + 600 K-ary cases) on the FINAL tree (after the sigmoid / ln fast
# division of 1282941 / d22e4ac), the exhaustive division probe again, and the c5 clamp / clamp + T bench lines.
set -x
QQA_FUZZ_CASES=4000 QQA_FUZZ_CASES_K=600 python -m pytest tests/test_gpu_fuzz.py -x -q > gpurun_out/r2u_fuzz.log 2>&1; echo rc=$? >> gpurun_out/r2u_fuzz.log
QQA_KARY_QUAD=2 QQA_FUZZ_CASES=0 QQA_FUZZ_CASES_K=300 python -m pytest tests/test_gpu_fuzz.py -x -q > gpurun_out/r2u_fuzz_q2.log 2>&1; echo rc=$? >> gpurun_out/r2u_fuzz_q2.log
python bench.py --map clamp --no-cpu > gpurun_out/r2u_bench_c5_clamp.json 2> gpurun_out/r2u_bench_c5_clamp.err
python bench.py --map clamp --temperature 0.001 --no-cpu > gpurun_out/r2u_bench_c5_clampT.json 2> gpurun_out/r2u_bench_c5_clampT.err
