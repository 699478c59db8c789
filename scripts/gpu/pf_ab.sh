for c in ${FCONF:-1 0}; do for pf in 1 0; do
  echo "config $c pf=$pf: $(HPBJ_APPLY_PF=$pf HPBJ_L2_ARENA=0 HPBJ_FUSED_PROF=1 REPS=3 timeout 300 python scripts/quick_solve.py $c 2>&1 | grep 'hpbj fused' | tail -1 | cut -c40-)"
done; done
for c in 2 3; do for pf in 1 0; do echo "config $c pf=$pf: $(HPBJ_APPLY_PF=$pf PROF=1 REPS=2 timeout 300 python scripts/quick_solve.py $c 2>&1 | grep '"rep": 1' | grep -o '"apply_us": [0-9.]*')"; done; done
