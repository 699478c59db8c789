python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -k "spmv" > gpurun_out/r2_ab_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2_ab_tests.log
for v in "HPBJ_SPMV_STAGED=0" "HPBJ_SPMV_STAGED=1" "HPBJ_SPMV_STAGED=0" "HPBJ_SPMV_STAGED=1"; do
  env $v timeout 600 python bench.py --report-all --configs 2,3 --no-cpu-baseline --steps 2 --warmup 1 --out /tmp/ab.json > /tmp/ab.log 2>&1
  python - "$v" <<'PY'
import json, sys
for c, d in json.load(open('/tmp/ab.json'))['configs'].items():
    k = d['kernels']
    print(sys.argv[1], c, "ms/system %.1f" % d['ms_per_system'], "solve %.2f" % d['breakdown_ms']['solve'],
          "spmv us %.1f (%.3f)" % (k['spmv_csr_f64']['mean_us'], k['spmv_csr_f64']['hbm_frac']), flush=True)
PY
done > gpurun_out/r2_ab.log 2>&1
