set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "staged or c5 or 20_regular or blocked or fifty" > gpurun_out/r2q_tests.log 2>&1; echo rc=$? >> gpurun_out/r2q_tests.log
tools/ab_step.sh 2 "c5:QQA_STAGE=0 c5 c5:QQA_BLOCK_REPLICAS=16,QQA_STAGE=0 c5:QQA_BLOCK_REPLICAS=16" base > gpurun_out/r2q_ab.txt 2>&1
for r in 1 2; do for cfg in "QQA_STAGE=0" "QQA_STAGE=1" "QQA_BLOCK_REPLICAS=16 QQA_STAGE=1"; do env $cfg python bench.py --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(\"round $r $cfg\", d[\"value\"], d[\"roofline\"][\"avg_launch_ms\"], d[\"clocks\"][\"sm_mhz\"])"; done; done >> gpurun_out/r2q_ab.txt 2>&1
