# Final validation of the session-4 tree (sigmoid / ln division fast path): every bench line, ncu of the c5 and c3
# step kernels, the c5 launch list.
set -x
python bench.py > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err
for w in c1 c2 c3 c4 t1 k8 q13; do python bench.py --workload $w > gpurun_out/r2_bench_$w.json 2> gpurun_out/r2_bench_$w.err; done
python bench.py --map clamp > gpurun_out/r2_bench_c5_clamp.json 2> gpurun_out/r2_bench_c5_clamp.err
python bench.py --map clamp --temperature 0.001 > gpurun_out/r2_bench_c5_clampT.json 2> gpurun_out/r2_bench_c5_clampT.err
python bench.py --force-dist --no-cpu > gpurun_out/r2_bench_c5_forcedist.json 2> gpurun_out/r2_bench_c5_forcedist.err
tools/ncu_capture.sh r2t_c5_k_step -- python tools/step_time.py c5 8
tools/ncu_capture.sh r2t_c3_k_step QQA_PERSISTENT=0 -- python tools/step_time.py c3 8
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2t_c5_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2t_c5_launches.log 2>&1
