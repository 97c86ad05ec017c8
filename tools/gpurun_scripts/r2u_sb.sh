# Session 5: replica-block size re-check on the final tree (after the instruction cuts of sessions 2-4): does
# SB = 32 remain the best default for c5 under the power cap? Two passes, 600 annealing steps each.
for pass in 1 2; do tools/ab_sb.sh 600 "64 32 16" base 2>&1 | sed "s/^/pass $pass /"; done > gpurun_out/r2u_sb_final_tree.txt
