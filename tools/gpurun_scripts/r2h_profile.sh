set -x
tools/ncu_capture.sh r2_c5_k_step -- python tools/step_time.py c5 8
tools/ncu_capture.sh r2_c3_k_step QQA_PERSISTENT=0 -- python tools/step_time.py c3 8
tools/ncu_capture.sh r2_c4_k_step QQA_PERSISTENT=0 -- python tools/step_time.py c4 8
tools/ncu_capture.sh r2_c4_sb256_k_step QQA_BLOCK_REPLICAS=256 -- python tools/step_time.py c4 8
for c in 1 2 3 4; do QQA_COMM_CHUNKS=$c python tools/host_enqueue.py 8 32 64 2>&1 | sed "s/^/chunks=$c /"; done > gpurun_out/r2_host_enqueue.txt
