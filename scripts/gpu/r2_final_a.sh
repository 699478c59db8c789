# round-end style pass (part A): full GPU suite, smoke, profiling pass
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 2400 python -X faulthandler -m pytest tests -m gpu -q -rf --durations=15 -p no:cacheprovider > gpurun_out/r2_final_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r2_final_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_final_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2_final_smoke.log
RND=r02 bash scripts/profile_round.sh > gpurun_out/r2_final_prof.log 2>&1
tail -3 gpurun_out/r2_final_pytest.log; tail -2 gpurun_out/r2_final_smoke.log; tail -5 gpurun_out/r2_final_prof.log
