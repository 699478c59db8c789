# per-kernel times (profiling path) for the configs in KCONF
for c in ${KCONF:-2 3}; do PROF=1 REPS=2 timeout 300 python scripts/quick_solve.py $c 2>&1 | grep '"rep": 1' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print({k:(round(v,2) if isinstance(v,float) else v) for k,v in d.items() if k in ('config','setup_ms','factor_ms','solve_ms','its','err','apply_us','spmv_us','mgs_us')})"; done
