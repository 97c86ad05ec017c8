set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2j_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2j_gputest.log
tools/ab_step.sh 2 "c5 c5:QQA_BLOCK_REPLICAS=16" base rp > gpurun_out/r2j_ab_recompute.txt 2>&1
python bench.py --workload c4 > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err
for r in 32 16 8; do python bench.py --replicas $r --no-cpu --no-e2e > gpurun_out/r2_bench_c5_replicas$r.json 2> gpurun_out/r2_bench_c5_replicas$r.err; done
python bench.py --force-dist --replicas 8 --no-cpu --no-e2e > gpurun_out/r2_bench_c5_forcedist_replicas8.json 2> gpurun_out/r2_bench_c5_forcedist_replicas8.err
python bench.py --force-dist --no-cpu --no-e2e > gpurun_out/r2_bench_c5_forcedist.json 2> gpurun_out/r2_bench_c5_forcedist.err
