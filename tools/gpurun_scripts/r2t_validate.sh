# Session-4 re-entry check: rebuilt tree (7fee73d) -- full GPU suite, smoke, headline bench, other workloads, force-dist path.
set -x
python -m pytest tests -m gpu -q > gpurun_out/r2t_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2t_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2t_smoke.log 2>&1
python bench.py > gpurun_out/r2t_bench_c5.json 2> gpurun_out/r2t_bench_c5.err
for w in c2 t1 c4 c3 k8 q13; do python bench.py --workload $w > gpurun_out/r2t_bench_$w.json 2> gpurun_out/r2t_bench_$w.err; done
python bench.py --gpus 1 --force-dist > gpurun_out/r2t_bench_c5_forcedist.json 2> gpurun_out/r2t_bench_c5_forcedist.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2t_bench_ref.json 2> gpurun_out/r2t_bench_ref.err
