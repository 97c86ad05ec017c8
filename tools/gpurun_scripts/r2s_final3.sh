# Session-3 validation after the K-ary and publication changes: GPU suite, c5 A/B vs the previous build,
# k8 ncu, bench lines of c5 / k8 / q13 / c4 / c3.
set -x
python -m pytest tests -m gpu -q > gpurun_out/r2s3_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2s3_gputest.log
tools/ab_step.sh 2 "c5 c3" base kkc > gpurun_out/r2s3_ab_c5.txt 2>&1
tools/ncu_capture.sh r2_k8_k_step_K NCU_DUMMY=1 -- python tools/step_time.py k8 8
python bench.py > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err
for w in k8 q13 c4 c3; do python bench.py --workload $w > gpurun_out/r2_bench_$w.json 2> gpurun_out/r2_bench_$w.err; done
