# Sigmoid division without the range check: exhaustive proof, full GPU suite, A/B vs the plain division (exp/libqqa_divold.so).
set -x
python -m pytest tests/test_gpu_sigdiv.py -q > gpurun_out/r2t_sigdiv_test.log 2>&1; echo rc=$? >> gpurun_out/r2t_sigdiv_test.log
python -m pytest tests -m gpu -q -x > gpurun_out/r2t_sigdiv_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2t_sigdiv_gputest.log
tools/ab_step.sh 2 "c5 c3 c4 c2" base divold > gpurun_out/r2t_ab_sigdiv.txt 2>&1
python bench.py > gpurun_out/r2t_sigdiv_bench_c5.json 2> gpurun_out/r2t_sigdiv_bench_c5.err
