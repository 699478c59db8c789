# fused-cycle A/B: SPK layout x L2 arena prefetch, phase timers + solve times (configs 1, 0, 4)
for c in ${FCONF:-1 4 0}; do for r in 0 1; do for l in 0 1; do
  echo "config $c rows=$r l2=$l: $(HPBJ_SPK_ROWS=$r HPBJ_L2_ARENA=$l HPBJ_FUSED_PROF=1 REPS=3 timeout 300 python scripts/quick_solve.py $c 2>&1 | grep 'hpbj fused' | tail -1 | cut -c40-)"
  echo "   solve: $(HPBJ_SPK_ROWS=$r HPBJ_L2_ARENA=$l timeout 300 python scripts/fused_stats.py $c 2>&1 | grep 'prof=False' | tail -1 | cut -c1-60)"
done; done; done
