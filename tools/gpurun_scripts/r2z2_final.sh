# Final round-2 validation after the session-3 changes: the whole GPU suite, smoke, every bench line.
set -x
python -m pytest tests -m gpu -q > gpurun_out/r2z2_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2z2_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z2_smoke.log 2>&1
python bench.py > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err
for w in c1 c2 c3 c4 t1 k8 q13; do python bench.py --workload $w > gpurun_out/r2_bench_$w.json 2> gpurun_out/r2_bench_$w.err; done
python bench.py --map clamp > gpurun_out/r2_bench_c5_clamp.json 2> gpurun_out/r2_bench_c5_clamp.err
python bench.py --map clamp --temperature 0.001 > gpurun_out/r2_bench_c5_clampT.json 2> gpurun_out/r2_bench_c5_clampT.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err
python bench.py --force-dist --no-cpu > gpurun_out/r2_bench_c5_forcedist.json 2> gpurun_out/r2_bench_c5_forcedist.err
