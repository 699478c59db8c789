# source-level ncu captures of the config-3 apply and MGS kernels (read back
# here) + host growing A/B
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 600 python scripts/gpu/grow_ab.py 3 > gpurun_out/r2_grow_ab3.log 2>&1
export HPBJ_NOGRAPH=1 HPBJ_FUSED=0 REPS=1
timeout 600 python scripts/gpu/solve_once.py 3 > gpurun_out/r2_ap_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_apply_spk -s 8 -c 1 \
    -o gpurun_out/r2_apply_src -f python scripts/gpu/solve_once.py 3 > gpurun_out/r2_apply_ncu.log 2>&1
ncu -i gpurun_out/r2_apply_src.ncu-rep --page source --csv > gpurun_out/r2_apply_source.csv 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mgs -s 20 -c 1 \
    -o gpurun_out/r2_mgs_src -f python scripts/gpu/solve_once.py 3 > gpurun_out/r2_mgs_ncu.log 2>&1
ncu -i gpurun_out/r2_mgs_src.ncu-rep --page source --csv > gpurun_out/r2_mgs_source.csv 2>/dev/null
ls -la gpurun_out | tail -8
