python -c "import __graft_entry__ as g; g.build()" || exit 1
python scripts/gpu/setup_once.py 3 > gpurun_out/r2_setup_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_block_lu_ll -s 1 -c 1 -o gpurun_out/r2_prof_lu_ll5 python scripts/gpu/setup_once.py 3 > gpurun_out/r2_ncu_lu.log 2>&1
echo "rc=$?" >> gpurun_out/r2_ncu_lu.log
