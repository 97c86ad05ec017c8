#!/bin/bash
# L2 / DRAM experiments on c5 (one box): per config, the k_step time (CUDA events, tools/step_time.py) and,
# after that exact command exited 0, ncu DRAM bytes of two k_step launches.
# usage: tools/l2_sweep.sh <outdir> "<config> ..."   config = lib:VAR=val,VAR=val  (lib: base or exp name)
OUT=$1; shift
mkdir -p $OUT
for cfg in $@; do
  lib=${cfg%%:*}; envs=${cfg#*:}
  if [ "$lib" = base ]; then libp=""; else libp="exp/libqqa_$lib.so"; fi
  E="QQA_LIB_PATH=$libp $(echo $envs | tr ',' ' ')"
  tag=$(echo "$cfg" | tr ':,=/' '____')
  env $E python tools/step_time.py c5 40 > $OUT/$tag.time 2>&1 && \
  env $E timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
      --clock-control none -k regex:k_step -s 6 -c 2 --csv python tools/step_time.py c5 4 > $OUT/$tag.ncu 2>&1
  echo "$cfg: $(tail -1 $OUT/$tag.time) | $(grep -E 'dram__bytes_(read|write)' $OUT/$tag.ncu | tail -2 | awk -F'","' '{print $(NF-2), $NF}' | tr '\n' ' ')"
done
