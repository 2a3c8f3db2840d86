"""One K-cycle application on a BASELINE config (for ncu on k_ktail)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import lapgen, paper_1705_06266_b200 as P
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g = lapgen.config(k)
h = P.Hierarchy(g, cycle=1)
r = torch.from_numpy(lapgen.rhs(g.n)).cuda()
for _ in range(3):
    z = h.kcycle(0, r)
torch.cuda.synchronize()
print("ok", float(z.abs().max()))
