# dev iteration: gpu tests, per-kernel times (profiling path), fused graph timings
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in ${KCONF:-1 2 3}; do PROF=1 REPS=2 timeout 300 python scripts/quick_solve.py $c 2>&1 | grep '"rep": 1' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print({k:(round(v,2) if isinstance(v,float) else v) for k,v in d.items() if k in ('config','setup_ms','factor_ms','solve_ms','its','err','apply_us','spmv_us','mgs_us')})"; done
for c in ${FCONF:-0 1 4}; do HPBJ_DEBUG=1 REPS=2 timeout 300 python scripts/quick_solve.py $c 2>&1 | grep "solve: pre" | tail -1; done
