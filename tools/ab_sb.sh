#!/bin/bash
# A/B of experimental builds across replica-block sizes on c5.
# usage: tools/ab_sb.sh <anneal_steps> "<SB list>" base name1 ...
T=$1; SBS=$2; shift 2
for sb in $SBS; do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=""; else lib="exp/libqqa_$v.so"; fi
    QQA_BLOCK_REPLICAS=$sb QQA_LIB_PATH=$lib python bench.py --anneal-steps $T --steps 2 --warmup 1 --no-e2e --no-cpu 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('SB=$sb', '$v', 'kernel_ms %.4f' % r['avg_launch_ms'], 'sm_mhz', d['clocks']['sm_mhz'])"
  done
done
