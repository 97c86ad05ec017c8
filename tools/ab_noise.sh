#!/bin/bash
# c5 k_step time with clamp + Langevin noise for experimental builds
for r in 1 2; do
  for v in "$@"; do
    QQA_LIB_PATH=exp/libqqa_$v.so python bench.py --map clamp --temperature 0.001 --anneal-steps 300 --steps 2 --warmup 1 --no-e2e --no-cpu 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', 'round $r', 'kernel_ms %.4f' % r['avg_launch_ms'], 'sm_mhz', d['clocks']['sm_mhz'])"
  done
done
