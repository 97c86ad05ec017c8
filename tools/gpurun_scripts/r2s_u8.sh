# Gather depth 8 (QQA_GATHER_U=8 build in exp/) vs 4 on the persistent / L2-resident workloads and c5.
set -x
tools/ab_step.sh 2 "c2 t1 c3 c5" base u8 > gpurun_out/r2s_u8_ab.txt 2>&1
