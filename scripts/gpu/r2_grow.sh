# host region-growing variants on the GPU box's host
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
lscpu | grep -i "model name\|^CPU(s)\|L2\|L3" > gpurun_out/r2_grow_ab2.log
timeout 1200 python scripts/gpu/grow_ab.py ${1:-3} >> gpurun_out/r2_grow_ab2.log 2>&1
