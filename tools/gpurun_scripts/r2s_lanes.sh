# Non-FULL shapes: idle lanes load a duplicate of the last vector instead of zeros (no CS2R / predication per
# load) vs the previous build (exp/libqqa_head.so).
set -x
python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_fuzz.py tests/test_gpu_edges.py -x -q > gpurun_out/r2s_lanes_tests.log 2>&1; echo rc=$? >> gpurun_out/r2s_lanes_tests.log
tools/ab_step.sh 2 "c2 t1 c4 c3 c5" base head > gpurun_out/r2s_lanes_ab.txt 2>&1
