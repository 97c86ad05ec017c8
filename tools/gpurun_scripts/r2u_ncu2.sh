# Session 5: ncu --set full of the final tree's c4, k8, c2 and t1 step kernels (launch-per-step form), so that
# every traffic.json entry and the roofline table come from the same tree.
set -x
tools/ncu_capture.sh r2u_c4_k_step QQA_PERSISTENT=0 -- python tools/step_time.py c4 8
tools/ncu_capture.sh r2u_k8_k_step_K NCU_DUMMY=1 -- python tools/step_time.py k8 8
tools/ncu_capture.sh r2u_c2_k_step QQA_PERSISTENT=0 -- python tools/step_time.py c2 8
tools/ncu_capture.sh r2u_t1_k_step QQA_PERSISTENT=0 -- python tools/step_time.py t1 8
