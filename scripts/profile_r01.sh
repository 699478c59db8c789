#!/bin/bash
# Round-1 profiling pass on the GPU box (one GPU). Plain runs precede every ncu run.
set -x
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
REPS=1 python scripts/quick_solve.py 1 > gpurun_out/plain_qs.log 2>&1 && \
for k in k_apply k_mgs k_spmv k_block_lu; do
  REPS=1 ncu --set full --clock-control none --import-source on -k regex:$k -s 12 -c 1 -o gpurun_out/prof_$k -f \
    python scripts/quick_solve.py 1 > gpurun_out/ncu_$k.log 2>&1
done
ls -la gpurun_out
