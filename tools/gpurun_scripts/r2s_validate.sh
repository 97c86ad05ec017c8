# Session-3 re-entry check: the rebuilt tree passes the GPU suite, smoke and the headline bench.
set -x
python -m pytest tests -m gpu -q > gpurun_out/r2s_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2s_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s_smoke.log 2>&1
python bench.py > gpurun_out/r2s_bench_c5.json 2> gpurun_out/r2s_bench_c5.err
