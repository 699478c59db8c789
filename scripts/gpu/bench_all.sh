mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_default.json
timeout 1500 python bench.py --report-all --steps 3 --warmup 2 --out gpurun_out/per_config.json 2> gpurun_out/report_all.err | tail -5; echo "report rc=$?"
tail -5 gpurun_out/report_all.err
