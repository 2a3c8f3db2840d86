"""Debug helper: solve cfg 2 under different input placements / streams."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import lapgen, paper_1705_06266_b200 as P

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g = lapgen.config(k)
b = lapgen.rhs(g.n)
dev = torch.device("cuda", 0)
gd = lapgen.Graph(g.n, torch.from_numpy(g.row_ptr).to(dev), torch.from_numpy(g.col).to(dev), torch.from_numpy(g.w).to(dev))
torch.cuda.synchronize()
st = torch.cuda.Stream()
for name, graph, strm, ug in [("host/None", g, None, 1), ("dev/None", gd, None, 1), ("host/stream", g, st, 1),
                              ("dev/stream", gd, st, 1), ("dev/stream/nograph", gd, st, 0)]:
    h = P.Hierarchy(graph, stream=strm, use_graphs=ug)
    bt = torch.from_numpy(b).to(dev)
    torch.cuda.synchronize()
    x, it, rr, rc = h.solve(bt, stream=strm)
    torch.cuda.synchronize()
    print(name, "levels", h.nlev, "iters", it, "relres", rr, "rc", rc, flush=True)
