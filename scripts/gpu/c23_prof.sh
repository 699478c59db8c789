# kernel-level ncu of the per-kernel path on the >=1M-row configs
export HPBJ_NOGRAPH=1 HPBJ_FUSED=0
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in 2 3; do
  REPS=1 PROF=1 timeout 300 python scripts/quick_solve.py $c > gpurun_out/plain_qs$c.log 2>&1 || { echo "plain $c failed"; cat gpurun_out/plain_qs$c.log | tail -5; continue; }
  cut -c1-600 gpurun_out/plain_qs$c.log
  for k in k_apply_spk k_spmv; do
    REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -o gpurun_out/prof_c${c}_$k -f \
      python scripts/quick_solve.py $c > gpurun_out/ncu_c${c}_$k.log 2>&1
  done
done
ls gpurun_out
