# Session 5: the source-segmented gather (QQA_SEGMENTS=2/3, opt-in) against the one-pass kernel on the final tree.
run() { env "$@" python bench.py --anneal-steps 600 --steps 2 --warmup 1 --no-e2e --no-cpu 2>/dev/null \
  | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$*', 'ms_per_anneal_step %.4f' % (d['ms_per_step']/600), 'kernel_ms %.4f' % r['avg_launch_ms'], 'sm_mhz', d['clocks']['sm_mhz'])"; }
for pass in 1 2; do run QQA_SEGMENTS=0; run QQA_SEGMENTS=2; run QQA_SEGMENTS=3; done > gpurun_out/r2u_seg_final_tree.txt 2>&1
