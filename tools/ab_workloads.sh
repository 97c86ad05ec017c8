#!/bin/bash
# A/B experimental builds over several workloads (full anneal), k-step time per annealing step.
# usage: tools/ab_workloads.sh "<workloads>" <rounds> name1 name2 ...
WS=$1; R=$2; shift 2
for r in $(seq 1 $R); do
  for w in $WS; do
    for v in "$@"; do
      QQA_LIB_PATH=exp/libqqa_$v.so python bench.py --workload $w --steps 2 --warmup 1 --no-e2e --no-cpu 2>/dev/null \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$w', '$v', 'round $r', 'us/step %.2f' % (1e3 * d['ms_per_step'] / d['config']['anneal_steps']), 'kernel_us %.2f' % (1e3 * r['avg_launch_ms']), 'sm_mhz', d['clocks']['sm_mhz'])"
    done
  done
done
