# host partitioner timings on the GPU box's cores (pipelined vs sequential refine)
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Core|Socket" 
for pipe in 1 0; do for c in 1 2 3; do HPBJ_PART_PIPE=$pipe HPBJ_DEBUG=1 R=4 timeout 300 python scripts/part_bench.py $c 2>&1 | tail -5; done; done
R=10 python scripts/part_bench.py 1
OMP_NUM_THREADS=8 R=10 python scripts/part_bench.py 1
