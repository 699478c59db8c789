# host partitioner phase timings on the GPU box's host + the default bench line
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
nproc > gpurun_out/r2_part.log; lscpu | grep -i "model name\|^CPU(s)\|L3" >> gpurun_out/r2_part.log
cat /sys/kernel/mm/transparent_hugepage/enabled >> gpurun_out/r2_part.log
for c in 1 2 3; do HPBJ_DEBUG=1 timeout 300 python scripts/gpu/part_debug.py $c >> gpurun_out/r2_part.log 2>&1; done
HPBJ_PART_SEQ=1 HPBJ_DEBUG=1 timeout 300 python scripts/gpu/part_debug.py 3 >> gpurun_out/r2_part.log 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2_part_bench.log 2>&1
tail -1 gpurun_out/r2_part_bench.log | cut -c1-1500
