# apply prefetch + LU layout: parity tests, kernel A/B
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "apply or left_looking or all_blocks" > gpurun_out/r2_iter2_t.log 2>&1
echo "rc=$?" >> gpurun_out/r2_iter2_t.log
REPS=3 timeout 1200 python scripts/gpu/kern_ab.py 3,2 "" "HPBJ_APPLY_PF=0" > gpurun_out/r2_iter2_ab.log 2>&1
tail -3 gpurun_out/r2_iter2_t.log; cat gpurun_out/r2_iter2_ab.log
