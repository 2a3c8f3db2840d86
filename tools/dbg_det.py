"""Run-to-run reproducibility of lap_solve on one hierarchy under switches."""
import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, lapgen, paper_1705_06266_b200 as P
name, envs = sys.argv[1], sys.argv[2:]
for e in envs:
    k, v = e.split("=")
    os.environ[k] = v
g0 = {"rmat16": lambda: lapgen.rmat(16), "star": lambda: lapgen.star(30000), "ba": lambda: lapgen.barabasi_albert(50000, 8),
      "grid": lambda: lapgen.grid2d(300, 300)}[name]()
for unit in (0, 1):
    g = lapgen.Graph(g0.n, g0.row_ptr, g0.col, np.ones(g0.nnz)) if unit else g0
    b = lapgen.rhs(g.n)
    for ug in (1, 0):
        h = P.Hierarchy(g, use_graphs=ug)
        xs = set()
        zs = set()
        for r in range(6):
            x, it, rr, _ = h.solve(b)
            xs.add(x.tobytes())
            zs.add(h.vcycle(b - b.mean()).tobytes())
        print(name, envs, "unit", unit, "graphs", ug, "distinct x:", len(xs), "distinct vcycle:", len(zs), flush=True)
        h.close()
