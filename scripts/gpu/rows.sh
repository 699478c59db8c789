# row-quad fold: parity (forced on every config) + apply timings on configs 2/3
mkdir -p gpurun_out
HPBJ_SPK_ROWS=1 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for r in 0 1; do for c in ${KCONF:-2 3}; do HPBJ_SPK_ROWS=$r PROF=1 REPS=2 timeout 300 python scripts/quick_solve.py $c 2>&1 | grep '"rep": 1' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('rows=$r', {k:(round(v,2) if isinstance(v,float) else v) for k,v in d.items() if k in ('config','setup_ms','factor_ms','solve_ms','its','err','apply_us','spmv_us','mgs_us')})"; done; done
