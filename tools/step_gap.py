"""Where does a bench step's time go outside setup_ms + solve_ms?  Per step:
event time around the whole step vs wall intervals of its phases."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import lapgen, paper_1705_06266_b200 as P
g = lapgen.config(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
dev = torch.device("cuda", 0)
gd = lapgen.Graph(g.n, torch.from_numpy(g.row_ptr).to(dev), torch.from_numpy(g.col).to(dev), torch.from_numpy(g.w).to(dev))
b = torch.from_numpy(lapgen.rhs(g.n)).to(dev)
x = torch.zeros_like(b)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for rep in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        w0 = time.perf_counter()
        h = P.Hierarchy(gd, stream=s)
        w1 = time.perf_counter()
        st0 = h.stats()
        h.solve(b, x, stream=s)
        w2 = time.perf_counter()
        st = h.stats()
        h.close()
        w3 = time.perf_counter()
        e1.record(s)
        torch.cuda.synchronize()
        w4 = time.perf_counter()
        print(f"step {rep}: event {e0.elapsed_time(e1):.2f} ms | wall setup {1e3*(w1-w0):.2f} (dev {st0['setup_ms']:.2f}) "
              f"solve {1e3*(w2-w1):.2f} (dev {st['solve_ms']:.2f}) free {1e3*(w3-w2):.2f} tail {1e3*(w4-w3):.2f}", flush=True)
