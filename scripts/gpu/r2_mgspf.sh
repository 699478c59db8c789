python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
REPS=3 timeout 900 python scripts/gpu/kern_ab.py 3 "" "HPBJ_MGS_PF=1" "" "HPBJ_MGS_PF=1" > gpurun_out/r2_mgspf.log 2>&1
cut -c1-330 gpurun_out/r2_mgspf.log
