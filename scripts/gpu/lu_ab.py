"""Setup timing A/B on the B200: batched LU (left-looking shared-memory
kernel vs the L2-scratch blocked kernel, HPBJ_LU_LL=0/1) and the apply-format
build, per config. Prints one JSON line per (config, variant)."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2509_09139_b200 as hp  # noqa: E402
from paper_2509_09139_b200.workloads import generate  # noqa: E402

for c in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2,3").split(",")]:
    s = generate(c)
    a = hp.SparseMatrix(s.n, s.row_ptr, s.col, s.val)
    part = hp.partition_graph(a, s.num_blocks, 0.1)
    ctx = hp.Context(0)
    ctx.set_matrix(a)
    for flag in ("0", "1"):
        os.environ["HPBJ_LU_LL"] = flag
        infos = []
        for k in range(6):
            infos.append(ctx.bj_setup(part, 1e-10))
        infos = infos[1:]
        print(json.dumps({"config": c, "HPBJ_LU_LL": flag,
                          "ms_lu": statistics.median(i.ms_lu for i in infos),
                          "ms_spk": statistics.median(i.ms_spk for i in infos),
                          "ms_factor": statistics.median(i.ms_factor for i in infos),
                          "ms_permute": statistics.median(i.ms_permute for i in infos)}), flush=True)
    del ctx
    torch.cuda.empty_cache()
