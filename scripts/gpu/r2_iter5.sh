# MGS launch-shape A/B (config 3), partition phases (configs 2, 3), fresh LU source profile
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
(cd scripts/micro && nvcc -O3 -gencode arch=compute_100a,code=sm_100a mma_rate.cu -o mma_rate && ./mma_rate) > gpurun_out/r2_mma_rate.log 2>&1
REPS=2 timeout 1200 python scripts/gpu/kern_ab.py 3 "" "HPBJ_MGS_VAR=1" "HPBJ_MGS_VAR=2" "HPBJ_MGS_VAR=3" "HPBJ_MGS_VAR=4" > gpurun_out/r2_iter5_ab.log 2>&1
for c in 2 3; do HPBJ_DEBUG=1 timeout 300 python scripts/gpu/part_debug.py $c 2>&1 | grep "refine:\|grow \|partition_graph\|weights\|adjacency" | tail -6; done > gpurun_out/r2_iter5_part.log
export HPBJ_NOGRAPH=1 HPBJ_FUSED=0 REPS=1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_block_lu_ll -c 1 \
    -o gpurun_out/r2_lu2_src -f python scripts/gpu/solve_once.py 3 > gpurun_out/r2_lu2_ncu.log 2>&1
ncu -i gpurun_out/r2_lu2_src.ncu-rep --page source --csv > gpurun_out/r2_lu2_source.csv 2>/dev/null
cut -c1-400 gpurun_out/r2_iter5_ab.log; cat gpurun_out/r2_iter5_part.log
cat gpurun_out/r2_mma_rate.log
