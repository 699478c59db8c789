python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python scripts/gpu/part_ab.py 3,2 > gpurun_out/r2_part_ab.log 2>&1
for v in "HPBJ_LU_SPLIT=0" "HPBJ_LU_SPLIT=1" "HPBJ_LU_SPLIT=0" "HPBJ_LU_SPLIT=1"; do
  env $v timeout 600 python scripts/gpu/lu_ab.py 2 > /tmp/ab.log 2>&1
  echo "$v $(grep '"1"' /tmp/ab.log)"
done > gpurun_out/r2_ab.log 2>&1
