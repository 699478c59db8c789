set -x
nproc; lscpu | grep -E "Model name|Socket|Thread|Core|MHz" ; free -g
python -c "import __graft_entry__ as g; g.build()" 
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 1700 python scripts/gpu/ref_c3_probe.py 3 2>&1 | tail -3
