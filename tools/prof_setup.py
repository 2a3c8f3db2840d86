"""Profile target: one warm lap_setup of cfg k inside the NVTX range "setup2"
(ncu --nvtx --nvtx-include "setup2/" --metrics gpu__time_duration.sum)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import lapgen, paper_1705_06266_b200 as P
k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
g = lapgen.config(k)
dev = torch.device("cuda", 0)
gd = lapgen.Graph(g.n, torch.from_numpy(g.row_ptr).to(dev), torch.from_numpy(g.col).to(dev),
                  torch.from_numpy(g.w).to(dev) if g.w is not None else None)
P.pool_retain(1 << 40)
h = P.Hierarchy(gd, use_graphs=0)
h.close()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("setup2")
h = P.Hierarchy(gd, use_graphs=0)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("setup_ms", h.stats()["setup_ms"])
