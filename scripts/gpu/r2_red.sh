#!/bin/bash
# batched partial-sum loads: per-kernel A/B, MGS phase timers, fused solve times, GPU suite
mkdir -p gpurun_out
HPBJ_NOGRAPH=1 HPBJ_FUSED=0 HPBJ_MGS_PROF=1 REPS=1 timeout 300 python scripts/gpu/solve_once.py 3 > gpurun_out/mgsprof2.log 2>&1; grep "mgs prof" gpurun_out/mgsprof2.log | tail -2
timeout 900 python scripts/gpu/kern_ab.py 0,1,4,2,3 '' > gpurun_out/red_ab.log 2>&1; cat gpurun_out/red_ab.log | sed 's/"spk_ms.*"apply_us"/"apply_us"/'
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_suite.log 2>&1; echo "suite rc=$?"; tail -3 gpurun_out/gpu_suite.log
