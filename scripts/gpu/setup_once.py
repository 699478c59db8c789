"""Two block-Jacobi setups of one config (ncu target): python setup_once.py CONFIG [HPBJ env...]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2509_09139_b200 as hp  # noqa: E402
from paper_2509_09139_b200.workloads import generate  # noqa: E402

c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
s = generate(c)
a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
part = hp.partition_graph(a, s.num_blocks, 0.1)
ctx = hp.Context(0)
ctx.set_matrix(a)
for _ in range(2):
    info = ctx.bj_setup(part, 1e-10)
    print(f"lu {info.ms_lu:.3f} ms spk {info.ms_spk:.3f} ms")
