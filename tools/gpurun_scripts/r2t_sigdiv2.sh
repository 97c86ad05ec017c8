# sig_div also in ln_c (noise path): exhaustive proof (sigmoid + ln operands), full GPU suite, smoke.
set -x
python -m pytest tests/test_gpu_sigdiv.py -q -s > gpurun_out/r2t_sigdiv2_test.log 2>&1; echo rc=$? >> gpurun_out/r2t_sigdiv2_test.log
python -m pytest tests -m gpu -q -x > gpurun_out/r2t_sigdiv2_gputest.log 2>&1; echo rc=$? >> gpurun_out/r2t_sigdiv2_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2t_sigdiv2_smoke.log 2>&1
