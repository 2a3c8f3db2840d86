"""Small end-to-end run of every solve path for compute-sanitizer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import lapgen, paper_1705_06266_b200 as P
for g in [lapgen.grid2d(40, 30), lapgen.rmat(11), lapgen.barabasi_albert(2000, 4), lapgen.grid3d(12)]:
    b = lapgen.rhs(g.n, seed=1)
    h = P.Hierarchy(g)
    _, it, rr, rc = h.solve(b)
    hk = P.Hierarchy(g, cycle=1)
    _, itk, rrk, rck = hk.solve(b)
    z = hk.kcycle(0, b - b.mean())
    X, its, rrs, rcb = h.solve_block(np.stack([b, 2 * b, lapgen.rhs(g.n, seed=2)]))
    print(g.n, it, rr, rc, itk, rrk, rck, list(its), rcb, flush=True)
