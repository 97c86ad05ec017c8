#!/bin/bash
# A/B timing of experimental builds (exp/libqqa_<name>.so) on one workload.
# usage: tools/ab_variants.sh <workload> <anneal_steps> <rounds> base name1 name2 ...
W=$1; T=$2; R=$3; shift 3
for r in $(seq 1 $R); do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=""; else lib="exp/libqqa_$v.so"; fi
    QQA_LIB_PATH=$lib python bench.py --workload $W --anneal-steps $T --steps 2 --warmup 1 --no-e2e --no-cpu 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$v', 'round $r', 'kernel_ms %.4f' % r['avg_launch_ms'], 'step_ms %.4f' % (d['ms_per_step']/d['config']['anneal_steps']), 'sm_mhz', d['clocks']['sm_mhz'])"
  done
done
