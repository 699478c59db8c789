# GPU test pass: build, the -m gpu suite (verbose, per-test timings), smoke.
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 2400 python -X faulthandler -m pytest tests -m gpu -v -rA --durations=30 -p no:cacheprovider -s > gpurun_out/r2_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2_smoke.log
