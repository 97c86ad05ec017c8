# Session-5 re-entry: rebuilt HEAD (d22e4ac + scripts) -- full GPU suite, smoke, headline bench, launch list and
# ncu --set full of the c5 and c3 step kernels of the final tree (sigmoid / ln fast division), other workloads.
set -x
python -m pytest tests -m gpu -q > gpurun_out/r2u_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2u_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2u_smoke.log 2>&1; echo rc=$? >> gpurun_out/r2u_smoke.log
python bench.py > gpurun_out/r2u_bench_c5.json 2> gpurun_out/r2u_bench_c5.err
tools/ncu_capture.sh r2u_c5_k_step -- python tools/step_time.py c5 8
tools/ncu_capture.sh r2u_c3_k_step QQA_PERSISTENT=0 -- python tools/step_time.py c3 8
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2u_c5_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2u_c5_launches.log 2>&1
for w in c3 c4 c2 t1 k8 q13; do python bench.py --workload $w --no-cpu > gpurun_out/r2u_bench_$w.json 2> gpurun_out/r2u_bench_$w.err; done
python bench.py --gpus 1 --force-dist --no-cpu > gpurun_out/r2u_bench_c5_forcedist.json 2> gpurun_out/r2u_bench_c5_forcedist.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2u_bench_ref.json 2> gpurun_out/r2u_bench_ref.err
