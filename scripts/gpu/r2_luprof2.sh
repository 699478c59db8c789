python -c "import __graft_entry__ as g; g.build()" || exit 1
HPBJ_LU_PROF=1 python scripts/gpu/setup_once.py 3 > gpurun_out/r2_luprof2.log 2>&1
HPBJ_LU_PROF=1 python scripts/gpu/setup_once.py 2 >> gpurun_out/r2_luprof2.log 2>&1
