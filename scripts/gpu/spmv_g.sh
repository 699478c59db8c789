for g in 1 2 4 8; do echo "G=$g"; HPBJ_SPMV_G=$g PROF=1 REPS=2 timeout 300 python scripts/quick_solve.py 2 2>&1 | grep '"rep": 1' | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print({k:(round(v,2) if isinstance(v,float) else v) for k,v in d.items() if k in ('solve_ms','its','spmv_us')})"; done
