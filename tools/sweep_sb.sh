#!/bin/bash
# us per annealing step of the default build for replica-block sizes (QQA_BLOCK_REPLICAS; 0 = automatic).
# usage: tools/sweep_sb.sh "<workloads>" "<SB list>" <rounds>
WS=$1; SBS=$2; R=${3:-1}
for r in $(seq 1 $R); do
  for w in $WS; do
    for sb in $SBS; do
      QQA_BLOCK_REPLICAS=$sb python bench.py --workload $w --steps 2 --warmup 1 --no-e2e --no-cpu 2>/dev/null \
        | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$w', 'SB=$sb', 'round $r', 'us/step %.2f' % (1e3 * d['ms_per_step'] / d['config']['anneal_steps']), 'sm_mhz', d['clocks']['sm_mhz'])"
    done
  done
done
