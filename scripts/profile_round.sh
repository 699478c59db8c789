#!/bin/bash
# Round profiling pass on the GPU box (one GPU). Each ncu run is preceded by the
# same command exiting 0 without ncu. The production solve is one CUDA graph
# with conditional WHILE nodes, which ncu cannot profile per kernel, so the ncu
# passes set HPBJ_NOGRAPH=1 (same kernels, host-sequenced).
# usage: RND=r02 bash scripts/profile_round.sh
RND=${RND:-r02}
mkdir -p gpurun_out
export HPBJ_NOGRAPH=1
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${RND}_plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/${RND}_launches_bench.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${RND}_ncu_launches.log 2>&1
cap() {  # cap <config> <kernel regex> <tag> [fused 0/1] [skip]
  HPBJ_FUSED=$4 REPS=1 timeout 600 python scripts/gpu/solve_once.py $1 > gpurun_out/${RND}_plain_$3.log 2>&1 && \
  HPBJ_FUSED=$4 REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s ${5:-4} -c 1 \
      -o gpurun_out/${RND}_prof_$3 -f python scripts/gpu/solve_once.py $1 > gpurun_out/${RND}_ncu_$3.log 2>&1
  echo "$3 rc=$?"
}
cap 3 k_block_lu_ll c3_lu 0 0
cap 3 k_spk_build c3_spk_build 0 1
cap 3 k_apply_spk c3_apply 0 8
cap 3 k_spmv c3_spmv 0 8
cap 3 k_mgs c3_mgs 0 8
cap 2 k_block_lu_ll c2_lu 0 0
cap 2 k_apply_spk c2_apply 0 8
cap 2 k_spmv c2_spmv 0 8
cap 2 k_icwy c2_icwy 0 8
cap 1 k_arnoldi_cycle c1_arnoldi_cycle 1 0
ls -la gpurun_out | grep $RND
# summarise on the box (the full captures exceed gpurun's copy-back limit);
# keep only the hot kernels' reports for source-level reading here
OUT=gpurun_out/profiles python scripts/summarize_round.py $RND > gpurun_out/${RND}_summary.log 2>&1
for f in gpurun_out/${RND}_prof_*.ncu-rep; do case $f in *c3_lu*|*c3_apply*|*c3_spk_build*) ;; *) rm -f $f ;; esac; done
du -sh gpurun_out
