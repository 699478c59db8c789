# per-config table with the reference CPU beside every config (config 3: one
# system through the reference's own partitioner, ~10 min)
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 3300 python bench.py --report-all --steps 3 --warmup 2 --out gpurun_out/r02_per_config.json > gpurun_out/r2_report_all.log 2>&1
echo "rc=$?" >> gpurun_out/r2_report_all.log
tail -12 gpurun_out/r2_report_all.log
