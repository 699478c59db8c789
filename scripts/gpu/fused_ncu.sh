export HPBJ_NOGRAPH=1
REPS=1 timeout 300 python scripts/quick_solve.py 1 > gpurun_out/fq.log 2>&1 || exit 1
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_arnoldi_cycle -c 1 -o gpurun_out/fused_c1 -f python scripts/quick_solve.py 1 > gpurun_out/fused_ncu.log 2>&1
tail -3 gpurun_out/fused_ncu.log
