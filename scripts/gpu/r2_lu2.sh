# LU with the shrinking update window: bit-identity + factor parity + timings; MGS test
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 600 python scripts/gpu/lu_ab.py 2,3 > gpurun_out/r2_lu2_ab.log 2>&1
HPBJ_LU_PROF=1 timeout 300 python scripts/gpu/setup_once.py 3 >> gpurun_out/r2_lu2_ab.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solve.py -x -q -p no:cacheprovider -k "left_looking or factors or lu_known or singular or apply_matches or textbook_mgs" > gpurun_out/r2_lu2_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_lu2_tests.log
tail -3 gpurun_out/r2_lu2_tests.log; cat gpurun_out/r2_lu2_ab.log
