# re-entry check: gpu tests, default bench, per-kernel times, host partition phases
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/bench_default.json
for c in 1 2 3; do HPBJ_DEBUG=1 REPS=3 PROF=1 timeout 300 python scripts/quick_solve.py $c > gpurun_out/qs_$c.log 2>&1; grep -E "^\[hpbj\] +(weights|adjacency|seed|bfs|refine|partition)" gpurun_out/qs_$c.log | tail -6; grep '"rep": 2' gpurun_out/qs_$c.log | cut -c1-400; done
