python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for c in 2 3; do HPBJ_DEBUG=1 timeout 300 python scripts/gpu/part_debug.py $c 2>&1 | grep "refine:\|grow \|partition_graph" | tail -6; done > gpurun_out/r2_part2.log
cat gpurun_out/r2_part2.log
