"""Experiment: setup time (median of 5, CUDA events) and per-level SpMV /
Chebyshev / V-cycle / solve times for cfg k under the current environment
(LAP_* switches are read once per process: run one process per setting)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import lapgen, paper_1705_06266_b200 as P
k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
tag = sys.argv[2] if len(sys.argv) > 2 else ""
g = lapgen.config(k)
dev = torch.device("cuda", 0)
gd = lapgen.Graph(g.n, torch.from_numpy(g.row_ptr).to(dev), torch.from_numpy(g.col).to(dev),
                  torch.from_numpy(g.w).to(dev) if g.w is not None else None)
b = torch.from_numpy(lapgen.rhs(g.n)).to(dev)
P.pool_retain(1 << 40)
ts = []
for rep in range(6):
    h = P.Hierarchy(gd)
    ts.append(h.stats()["setup_ms"])
    if rep < 5:
        h.close()
out = [f"cfg{k} {tag}: setup {np.median(ts[1:]):.2f} ms (all {' '.join('%.1f' % t for t in ts)})"]
sol = []
for _ in range(3):
    _, it, rr, rc = h.solve(b)
    sol.append(h.stats()["solve_ms"])
out.append(f"  solve {np.median(sol):.2f} ms iters {it} rr {rr:.2e}")
for l in range(h.nlev):
    kind = h.level_info(l)[0]
    if kind == 2:
        continue
    t, _, _ = h.bench_op(0, l, 30)
    s = f"  L{l} k{kind}: spmv {np.median(t)*1e3:.1f} us"
    if kind == 0:
        t, _, _ = h.bench_op(1, l, 30)
        s += f" cheb {np.median(t)*1e3:.1f} us"
    out.append(s)
t, _, _ = h.bench_op(2, 0, 20)
out.append(f"  vcycle {np.median(t)*1e3:.1f} us")
print("\n".join(out), flush=True)
