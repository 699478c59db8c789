python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_partition.py -x -q -p no:cacheprovider -k "spmv or partition" > gpurun_out/r2_iter4_t.log 2>&1
echo "rc=$?" >> gpurun_out/r2_iter4_t.log
REPS=3 timeout 1200 python scripts/gpu/kern_ab.py 2,3 "" > gpurun_out/r2_iter4_ab.log 2>&1
for i in 1 2; do HPBJ_DEBUG=1 timeout 300 python scripts/gpu/part_debug.py 3 2>&1 | grep "refine:\|grow \|partition_graph" | tail -3; done > gpurun_out/r2_iter4_part.log
tail -2 gpurun_out/r2_iter4_t.log; cat gpurun_out/r2_iter4_ab.log gpurun_out/r2_iter4_part.log
