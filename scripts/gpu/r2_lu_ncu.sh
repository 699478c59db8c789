# GPU tests touched by the setup changes, the bench line, and a source-level
# ncu capture of the config-3 left-looking LU (read back here)
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_solve.py tests/test_gpu_kernels.py -x -q -p no:cacheprovider > gpurun_out/r2_t.log 2>&1
echo "rc=$?" >> gpurun_out/r2_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/r2_t.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2_bench_nocpu.json 2> gpurun_out/r2_bench_nocpu.err
REPS=1 timeout 600 python scripts/gpu/solve_once.py 3 > gpurun_out/r2_lu_plain.log 2>&1 && \
REPS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_block_lu_ll -c 1 \
    -o gpurun_out/r2_lu_src -f python scripts/gpu/solve_once.py 3 > gpurun_out/r2_lu_ncu.log 2>&1
ncu -i gpurun_out/r2_lu_src.ncu-rep --page source --csv > gpurun_out/r2_lu_source.csv 2>/dev/null
ncu -i gpurun_out/r2_lu_src.ncu-rep --page raw --csv > gpurun_out/r2_lu_raw.csv 2>/dev/null
ls -la gpurun_out/
tail -3 gpurun_out/r2_t.log
