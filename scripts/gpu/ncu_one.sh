# usage: CONF=3 KERN=k_apply_spk TAG=x bash scripts/gpu/ncu_one.sh   (per-kernel path)
export HPBJ_NOGRAPH=1 HPBJ_FUSED=${HPBJ_FUSED:-0}
mkdir -p gpurun_out
REPS=1 timeout 300 python scripts/quick_solve.py $CONF > gpurun_out/plain_$TAG.log 2>&1 || { echo plain failed; tail -5 gpurun_out/plain_$TAG.log; exit 1; }
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KERN -s ${SKIP:-8} -c 1 -o gpurun_out/prof_$TAG -f \
      python scripts/quick_solve.py $CONF > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
