# FP64 tensor-core rank-32 updates in the left-looking LU: parity and timing
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python scripts/gpu/lu_tc_parity.py 2,3 > gpurun_out/r2_lutc_parity.log 2>&1
HPBJ_LU_TC=0 timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k left_looking > gpurun_out/r2_lutc_t.log 2>&1
timeout 900 python -m pytest tests/test_gpu_solve.py -x -q -p no:cacheprovider -k "large_config or config4" >> gpurun_out/r2_lutc_t.log 2>&1
REPS=3 timeout 1200 python scripts/gpu/kern_ab.py 2,3 "" "HPBJ_LU_TC=0" > gpurun_out/r2_lutc_ab.log 2>&1
cat gpurun_out/r2_lutc_parity.log; grep -E "passed|failed" gpurun_out/r2_lutc_t.log; cut -c1-250 gpurun_out/r2_lutc_ab.log
