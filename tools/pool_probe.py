"""Diagnostics: setup / free time and device free memory over consecutive
hierarchies (detects cudaMallocAsync pool growth / fragmentation)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import lapgen, paper_1705_06266_b200 as P
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g = lapgen.config(k)
dev = torch.device("cuda", 0)
gd = lapgen.Graph(g.n, torch.from_numpy(g.row_ptr).to(dev), torch.from_numpy(g.col).to(dev), torch.from_numpy(g.w).to(dev))
b = torch.from_numpy(lapgen.rhs(g.n)).to(dev)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for rep in range(12):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = P.Hierarchy(gd, stream=st)
        t1 = time.perf_counter()
        x, it, rr, rc = h.solve(b, stream=st)
        t2 = time.perf_counter()
        h.close()
        t3 = time.perf_counter()
        free, tot = torch.cuda.mem_get_info()
        print(f"cfg{k} rep {rep}: setup {1e3*(t1-t0):7.1f} (dev {h.stats()['setup_ms'] if False else 0:.0f}) solve {1e3*(t2-t1):7.1f} free {1e3*(t3-t2):6.1f} ms  device free {free/2**30:7.2f} GiB", flush=True)
