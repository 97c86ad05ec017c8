# Bench (power-capped, whole 3000-step solves) of c5: default vs the segmented gather (KS = 2), alternating.
set -x
for r in 1 2; do
  for ks in 1 2; do
    QQA_SEGMENTS=$ks python bench.py --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('round $r KS=$ks', d['value'], d['e2e']['value'], d['roofline']['avg_launch_ms'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_max'))"
  done
done > gpurun_out/r2s_seg_bench.txt 2>&1
