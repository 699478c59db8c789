# textbook MGS with loads in flight across the grid barrier: parity + config-3 bench + e2e phases
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_solve.py -x -q -p no:cacheprovider -k "textbook_mgs or config_solve or large_config" > gpurun_out/r2_mgs_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2_mgs_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2_mgs_bench.log 2>&1
timeout 300 python scripts/gpu/e2e_phases.py 3 > gpurun_out/r2_e2e_phases.log 2>&1
tail -2 gpurun_out/r2_mgs_tests.log; cat gpurun_out/r2_e2e_phases.log | tail -4
tail -1 gpurun_out/r2_mgs_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'], d['kernels']['arnoldi_mgs_f64'], d['breakdown_ms'])"
