# e2e host phases, host growing A/B, source-level captures of the config-3
# apply and the config-2 SpMV
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
HPBJ_DEBUG=1 timeout 600 python scripts/gpu/e2e_phases.py 3 > gpurun_out/r2_e2e_phases2.log 2>&1
timeout 600 python scripts/gpu/grow_ab.py 3 > gpurun_out/r2_grow_ab4.log 2>&1
export HPBJ_NOGRAPH=1 HPBJ_FUSED=0 REPS=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_apply_spk -s 8 -c 1 \
    -o gpurun_out/r2_apply2_src -f python scripts/gpu/solve_once.py 3 > gpurun_out/r2_apply2_ncu.log 2>&1
ncu -i gpurun_out/r2_apply2_src.ncu-rep --page source --csv > gpurun_out/r2_apply2_source.csv 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmv -s 8 -c 1 \
    -o gpurun_out/r2_spmv2_src -f python scripts/gpu/solve_once.py 2 > gpurun_out/r2_spmv2_ncu.log 2>&1
ncu -i gpurun_out/r2_spmv2_src.ncu-rep --page source --csv > gpurun_out/r2_spmv2_source.csv 2>/dev/null
grep -v "^\[hpbj\]   " gpurun_out/r2_e2e_phases2.log | tail -4; cat gpurun_out/r2_grow_ab4.log | cut -c1-200
