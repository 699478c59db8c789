# SPK build split (count / tile / pack): parity tests + setup timings
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
HPBJ_LU_LL=1 timeout 600 python scripts/gpu/lu_ab.py 1,2,3 > gpurun_out/r2_spk_ab.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solve.py tests/test_neumann.py -x -q -p no:cacheprovider -m gpu > gpurun_out/r2_spk_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_spk_tests.log
tail -3 gpurun_out/r2_spk_tests.log; grep '"1"' gpurun_out/r2_spk_ab.log
