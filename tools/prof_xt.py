"""Profile target for the column-tiled SpMV: a dense random level
(n = 100K, ~2000 entries per row) whose level 0 takes the XT layout."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import lapgen, paper_1705_06266_b200 as P
n = int(os.environ.get("XT_N", "100000"))
m = int(os.environ.get("XT_M", "100000000"))
t = time.time()
fn = f"/tmp/prof_xt_{n}_{m}.npz"
if os.path.exists(fn):
    z = np.load(fn)
    g = lapgen.Graph(n, z["rp"], z["col"], z["w"], "dense_rand")
else:
    rng = np.random.default_rng(1)
    u = rng.integers(0, n, m); v = rng.integers(0, n, m)
    u, v = lapgen.dedup_undirected(u, v)
    g = lapgen.csr_from_edges(n, u, v, rng.uniform(0.5, 2.0, len(u)), "dense_rand")
    np.savez(fn, rp=g.row_ptr, col=g.col, w=g.w)
print(f"graph n={g.n} nnz={g.nnz} gen {time.time()-t:.1f}s", flush=True)
h = P.Hierarchy(g, elim_enable=0)
print("levels", [h.level_info(l) for l in range(h.nlev)], flush=True)
for l in range(min(2, h.nlev - 1)):
    ms, by, ed = h.bench_op(1, l, int(sys.argv[1]) if len(sys.argv) > 1 else 20)
    print(f"level {l}: cheb {np.median(ms)*1e3:.1f} us {by/np.median(ms)/1e6:.0f} GB/s", flush=True)
