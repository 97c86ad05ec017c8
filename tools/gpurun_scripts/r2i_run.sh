set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2i_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2i_gputest.log
python bench.py > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err
for w in c1 c2 c3 c4 t1 k8 q13; do python bench.py --workload $w > gpurun_out/r2_bench_$w.json 2> gpurun_out/r2_bench_$w.err; done
python bench.py --map clamp > gpurun_out/r2_bench_c5_clamp.json 2> gpurun_out/r2_bench_c5_clamp.err
python bench.py --map clamp --temperature 0.001 > gpurun_out/r2_bench_c5_clampT.json 2> gpurun_out/r2_bench_c5_clampT.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err
tools/ab_step.sh 2 "c4" base h2 h3 > gpurun_out/r2i_ab_c4.txt 2>&1
tools/ncu_capture.sh r2_c5_sb16_k_step QQA_BLOCK_REPLICAS=16 -- python tools/step_time.py c5 8
