"""Setup + solve + free repeated on one stream (the bench pattern) with
LAP_SETUP_TRACE phase lines, to find setup-time outliers."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import lapgen, paper_1705_06266_b200 as P
k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
g = lapgen.config(k)
dev = torch.device("cuda", 0)
gd = lapgen.Graph(g.n, torch.from_numpy(g.row_ptr).to(dev), torch.from_numpy(g.col).to(dev), torch.from_numpy(g.w).to(dev))
b = torch.from_numpy(lapgen.rhs(g.n)).to(dev)
x = torch.zeros_like(b)
s = torch.cuda.Stream()
for rep in range(6):
    h = P.Hierarchy(gd, stream=s)
    st = h.stats()
    h.solve(b, x, stream=s)
    print(f"rep {rep}: setup_ms {st['setup_ms']:.1f} solve_ms {h.stats()['solve_ms']:.1f}", file=sys.stderr, flush=True)
    h.close()
