#!/bin/bash
# Round-1 profiling pass on the GPU box (one GPU). Plain runs precede every ncu run.
# The production solve is a CUDA graph with conditional (WHILE) nodes, which
# ncu cannot profile per kernel; HPBJ_NOGRAPH=1 launches the same kernels from
# the host for the ncu passes.
set -x
mkdir -p gpurun_out
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1
export HPBJ_NOGRAPH=1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
for c in 1 3; do
  REPS=1 python scripts/quick_solve.py $c > gpurun_out/plain_qs$c.log 2>&1 && \
  for k in k_apply_spk k_spmv k_icwy k_mgs; do
    REPS=1 ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -o gpurun_out/prof_c${c}_$k -f \
      python scripts/quick_solve.py $c > gpurun_out/ncu_c${c}_$k.log 2>&1
  done
done
ls -la gpurun_out
