timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for f in 1 0; do HPBJ_FUSED_PROF=$f HPBJ_DEBUG=1 HPBJ_FUSED=$f REPS=3 timeout 300 python scripts/quick_solve.py 1 0 4 2>&1 | grep -v "partition\|weights\|adjacency\|bfs\|refine\|graph built" | grep -v '"rep": 0' | cut -c1-250; done
