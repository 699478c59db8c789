# build, LU timing, selected parity tests, per-config table without the CPU reference
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python scripts/gpu/lu_ab.py 2,3 > gpurun_out/r2_lu_ab.log 2>&1
timeout 1500 python -X faulthandler -m pytest tests/test_gpu_kernels.py tests/test_gpu_solve.py -v -p no:cacheprovider -s \
   -k "left_looking or all_blocks or large_config or apply or manufactured or deterministic or stale" > gpurun_out/r2_iter_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_iter_tests.log
timeout 900 python bench.py --report-all --configs 1,2,3 --no-cpu-baseline --steps 3 --warmup 2 --out gpurun_out/r2_per_config.json > gpurun_out/r2_report.log 2>&1
echo "rc=$?" >> gpurun_out/r2_report.log
