"""Setup-time diagnostics: repeated lap_setup on one config, on a torch stream
and on the legacy default stream, with LAP_SETUP_TRACE phase timing for the
last repetition (run with LAP_SETUP_TRACE=1 for the phase lines)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import lapgen, paper_1705_06266_b200 as P
k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g = lapgen.config(k)
dev = torch.device("cuda", 0)
gd = lapgen.Graph(g.n, torch.from_numpy(g.row_ptr).to(dev), torch.from_numpy(g.col).to(dev), torch.from_numpy(g.w).to(dev))
st = torch.cuda.Stream()
P.pool_retain(1 << 40)
for name, strm in [("torch stream", st), ("default stream", None)]:
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = P.Hierarchy(gd, stream=strm)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(f"cfg{k} {name} rep {rep}: setup_ms {h.stats()['setup_ms']:.1f} wall {1e3*(t1-t0):.1f}", flush=True)
        h.close()
