#!/bin/bash
# A/B of step-kernel builds: tools/ab_step.sh <rounds> "<workload[:ENV=v,ENV=v]> ..." base name1 ...
# (per-step time from tools/step_time.py; build variants live in exp/libqqa_<name>.so)
R=$1; CFGS=$2; shift 2
for r in $(seq 1 $R); do
  for c in $CFGS; do
    w=${c%%:*}; envs=""; [ "$c" != "$w" ] && envs=$(echo ${c#*:} | tr ',' ' ')
    for v in "$@"; do
      if [ "$v" = base ]; then lib=""; else lib="exp/libqqa_$v.so"; fi
      echo "round $r $v $(env $envs QQA_LIB_PATH=$lib python tools/step_time.py $w 100 2>&1 | tail -1)"
    done
  done
done
