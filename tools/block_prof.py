"""One block solve (k right-hand sides) on a BASELINE config, for ncu on k_blk_spmv."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import lapgen, paper_1705_06266_b200 as P
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
k = int(sys.argv[2]) if len(sys.argv) > 2 else 4
g = lapgen.config(cfg)
h = P.Hierarchy(g)
B = torch.from_numpy(np.stack([lapgen.rhs(g.n, seed=j) for j in range(k)])).cuda()
X, it, rr, rc = h.solve_block(B)
torch.cuda.synchronize()
print("ok", it.tolist(), float(rr.max()))
