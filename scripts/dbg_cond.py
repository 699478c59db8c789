import sys; sys.path.insert(0, '/root/repo')
import numpy as np, paper_2509_09139_b200 as hp
from tests import fixtures as fx
a = fx.random_dd(300, 5, 13)
part = hp.partition_graph(a, 6, 0.1)
p = hp.Preconditioner.block_jacobi(a, part)
print(p.ctx.block_diagnostics(6))
print(p.ctx.block_stats(6))
