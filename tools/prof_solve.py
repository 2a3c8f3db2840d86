"""Profile target: build the cfg-k hierarchy, then one solve inside an NVTX
range "solve" (ncu --nvtx --nvtx-include solve/) and the level-0 smoother
bench inside "cheb"."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import lapgen, paper_1705_06266_b200 as P
k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
g = lapgen.config(k)
b = torch.from_numpy(lapgen.rhs(g.n)).cuda()
h0 = P.Hierarchy(g, use_graphs=int(os.environ.get("USE_GRAPHS", "0")))  # warm (pool, module load)
h0.close()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("setup")
h = P.Hierarchy(g, use_graphs=int(os.environ.get("USE_GRAPHS", "0")))
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("setup_ms", h.stats()["setup_ms"])
for l in range(h.nlev):
    print("level", l, h.level_info(l), flush=True)
h.solve(b)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("solve")
x, it, rr, rc = h.solve(b)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("iters", it, "relres", rr, "solve_ms", h.stats()["solve_ms"])
torch.cuda.nvtx.range_push("cheb")
lv = int(os.environ.get("PROF_LEVEL", h.first_agg_level()))
ms, by, ed = h.bench_op(1, lv, 5)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
import numpy as np
for l in range(h.nlev):
    kind = h.level_info(l)[0]
    if kind == 2:
        continue
    t, b2, e2 = h.bench_op(0, l, 30)
    line = f"level {l} kind {kind}: spmv {np.median(t)*1e3:.1f} us {b2/np.median(t)/1e6:.0f} GB/s {e2/np.median(t)/1e6:.0f} Medges/s"
    if kind == 0:
        t, b2, e2 = h.bench_op(1, l, 30)
        line += f" | cheb {np.median(t)*1e3:.1f} us {b2/np.median(t)/1e6:.0f} GB/s"
    print(line)
t, b2, e2 = h.bench_op(2, 0, 20)
print(f"vcycle {np.median(t)*1e3:.1f} us, {b2/np.median(t)/1e6:.0f} GB/s (algorithmic), {e2} edges")
print(f"cfg{k} level {lv}: {ms.mean()*1e3:.1f} us/launch, {by/ms.mean()/1e6:.0f} GB/s")
