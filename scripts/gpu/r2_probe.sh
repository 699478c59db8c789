# e2e host phases (HPBJ_DEBUG breakdown) + orthogonalisation A/B on config 3
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
HPBJ_DEBUG=1 timeout 600 python scripts/gpu/e2e_phases.py 3 > gpurun_out/r2_e2e_phases.log 2>&1
REPS=2 timeout 1200 python scripts/gpu/kern_ab.py 3 "HPBJ_ORTH=mgs" "HPBJ_ORTH=icwy" > gpurun_out/r2_kern_ab.log 2>&1
REPS=2 timeout 600 python scripts/gpu/kern_ab.py 2 "" >> gpurun_out/r2_kern_ab.log 2>&1
cat gpurun_out/r2_kern_ab.log
