import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, lapgen, paper_1705_06266_b200 as P
which = sys.argv[1] if len(sys.argv) > 1 else "rmat16"
g0 = lapgen.rmat(16) if which == "rmat16" else lapgen.star(30000)
g = lapgen.Graph(g0.n, g0.row_ptr, g0.col, np.ones(g0.nnz))
b = lapgen.rhs(g.n)
keep = []
def run(env, dirty=False):
    for k in ["LAP_UNIT", "LAP_SORT_LONG"]:
        os.environ.pop(k, None)
    os.environ.update(env)
    if dirty:  # garbage in the pool: a hierarchy of another graph, freed
        hx = P.Hierarchy(lapgen.barabasi_albert(20000, 7)); hx.close()
    h = P.Hierarchy(g)
    keep.append(h)
    x, it, rr, _ = h.solve(b)
    x2, it2, _, _ = h.solve(b)
    z = h.vcycle(b - b.mean())
    q = h.spmv(0, b)
    return x, z, q, it, x2
res = {}
for name, env, dirty in [("w", {"LAP_UNIT": "0"}, False), ("u", {}, False), ("w2", {"LAP_UNIT": "0"}, True),
                         ("u2", {}, True)]:
    res[name] = run(env, dirty)
for a, c in [("w", "u"), ("w", "w2"), ("u", "u2"), ("w2", "u2")]:
    print(a, c, [res[a][i].tobytes() == res[c][i].tobytes() for i in range(3)], res[a][3], res[c][3],
          float(np.abs(res[a][0] - res[c][0]).max()), float(np.abs(res[a][1] - res[c][1]).max()))
for a in res:
    print(a, "solve twice identical:", res[a][0].tobytes() == res[a][4].tobytes())
