# Final validation of the session-3 tree: GPU suite, smoke, bench lines (c5 headline, K-ary, c4), k8 launch list.
set -x
python -m pytest tests -m gpu -q > gpurun_out/r2s4_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2s4_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s4_smoke.log 2>&1
python bench.py > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err
for w in k8 q13 c2 t1 c1; do python bench.py --workload $w > gpurun_out/r2_bench_$w.json 2> gpurun_out/r2_bench_$w.err; done
