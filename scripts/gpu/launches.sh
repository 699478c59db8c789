# usage: CONF=3 TAG=x bash scripts/gpu/launches.sh  -> gpurun_out/ll_$TAG.csv (per-kernel durations, one solve)
export HPBJ_NOGRAPH=1 HPBJ_FUSED=${HPBJ_FUSED:-1}
REPS=1 timeout 300 python scripts/quick_solve.py $CONF > /dev/null 2>&1 || { echo plain failed; exit 1; }
REPS=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_$TAG.csv python scripts/quick_solve.py $CONF > /dev/null 2>&1
echo done
