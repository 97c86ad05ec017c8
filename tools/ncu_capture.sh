#!/bin/bash
# One ncu --set full capture of the first step-kernel launch after 6 warm-up launches, summarised ON THE BOX
# (the .ncu-rep stays in /tmp; gpurun brings back at most 64 MiB): <tag> <env...> -- <command ...>
# writes gpurun_out/<tag>.summary.txt (tools/ncu_summary.py full) and gpurun_out/<tag>.raw.csv.
TAG=$1; shift
ENVS=()
while [ "$1" != "--" ]; do ENVS+=("$1"); shift; done; shift
env "${ENVS[@]}" "$@" > gpurun_out/$TAG.plain.log 2>&1 || { echo "plain run failed"; exit 1; }
env "${ENVS[@]}" ncu --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-k_step} -s ${NCU_SKIP:-6} -c 1 \
    -f -o /tmp/$TAG "$@" > gpurun_out/$TAG.ncu.log 2>&1
python tools/ncu_summary.py full /tmp/$TAG.ncu-rep > gpurun_out/$TAG.summary.txt 2>&1
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > gpurun_out/$TAG.raw.csv 2>/dev/null
ncu -i /tmp/$TAG.ncu-rep --page source --csv > /tmp/$TAG.source.csv 2>/dev/null; gzip -c /tmp/$TAG.source.csv > gpurun_out/$TAG.source.csv.gz
