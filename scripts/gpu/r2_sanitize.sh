# usage: TOOL=racecheck|synccheck|memcheck bash scripts/gpu/r2_sanitize.sh
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
mkdir -p gpurun_out
timeout 2400 compute-sanitizer --tool ${TOOL:-racecheck} --print-limit 50 --launch-timeout 0 \
  python scripts/gpu/sanitize_case.py > gpurun_out/r02_sanitize_${TOOL:-racecheck}.log 2>&1
echo "rc=$?" >> gpurun_out/r02_sanitize_${TOOL:-racecheck}.log
tail -5 gpurun_out/r02_sanitize_${TOOL:-racecheck}.log
