python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python scripts/gpu/lu_ab.py 2,3 > gpurun_out/r2_lu_ab.log 2>&1
HPBJ_LU_PROF=1 python scripts/gpu/setup_once.py 3 >> gpurun_out/r2_lu_ab.log 2>&1
timeout 1200 python -X faulthandler -m pytest tests/test_gpu_kernels.py -v -p no:cacheprovider -s -k "left_looking or factors or lu_known or singular or apply_matches" > gpurun_out/r2_lu_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_lu_tests.log
