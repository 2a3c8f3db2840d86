"""Per-step diagnostics of the bench step: CUDA events around setup, solve and
free separately plus host walls, for cfg k (argv), 6 steps after 3 warm-ups."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import lapgen, paper_1705_06266_b200 as P
k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
g = lapgen.config(k)
dev = torch.device("cuda", 0)
b = torch.from_numpy(lapgen.rhs(g.n)).to(dev)
x = torch.zeros_like(b)
gd = lapgen.Graph(g.n, torch.from_numpy(g.row_ptr).to(dev), torch.from_numpy(g.col).to(dev),
                  torch.from_numpy(g.w).to(dev) if g.w is not None else None)
st = torch.cuda.Stream()
P.pool_retain(1 << 40)
E = lambda: torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(st):
    for rep in range(9):
        e = [E() for _ in range(4)]
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        e[0].record(st)
        h = P.Hierarchy(gd, stream=st)
        e[1].record(st)
        h1 = time.perf_counter()
        h.solve(b, x, stream=st)
        e[2].record(st)
        h2 = time.perf_counter()
        s = h.stats()
        h.close()
        e[3].record(st)
        h3 = time.perf_counter()
        torch.cuda.synchronize()
        h4 = time.perf_counter()
        print(f"cfg{k} rep {rep}: ev setup {e[0].elapsed_time(e[1]):.2f} solve {e[1].elapsed_time(e[2]):.2f} free {e[2].elapsed_time(e[3]):.2f} "
              f"| lib setup_ms {s['setup_ms']:.2f} solve_ms {s['solve_ms']:.2f} | wall setup {1e3*(h1-h0):.2f} solve {1e3*(h2-h1):.2f} "
              f"free {1e3*(h3-h2):.2f} tail {1e3*(h4-h3):.2f}", flush=True)
