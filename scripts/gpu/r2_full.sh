# Round-end style pass: build, full -m gpu suite, smoke, default bench (GPU arm with the CPU baseline)
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -X faulthandler -m pytest tests -m gpu -v -rA --durations=30 -p no:cacheprovider > gpurun_out/r2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
timeout 2400 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
echo "bench rc=$?" >> gpurun_out/r2_bench.err
