# L2 -> SM gather throughput by row width (tools/probes/l2bw.cu), L2-resident (16 MB) and beyond (64 / 128 MB).
set -x
for x in 16 64 128; do tools/probes/l2bw $x; done > gpurun_out/r2s_l2bw.txt 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks.mem --format=csv >> gpurun_out/r2s_l2bw.txt
