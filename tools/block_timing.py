"""N4: k right-hand sides per solve (lap_solve_block) vs k single solves:
solve ms, edges*rhs/s (SpMV edges of every pass times the columns it serves,
per second of device time), iterations."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import lapgen, paper_1705_06266_b200 as P

dev = torch.device("cuda", 0)
want = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4]
for cfg in want:
    g = lapgen.config(cfg)
    gd = lapgen.Graph(g.n, torch.from_numpy(g.row_ptr).to(dev), torch.from_numpy(g.col).to(dev), torch.from_numpy(g.w).to(dev))
    s = torch.cuda.Stream()
    h = P.Hierarchy(gd, stream=s)
    b1 = torch.from_numpy(lapgen.rhs(g.n)).to(dev)
    x1 = torch.zeros_like(b1)
    ms1 = []
    for rep in range(3):
        _, it1, rr1, _ = h.solve(b1, x1, stream=s)
        st = h.stats()
        ms1.append(st["solve_ms"])
        e1 = st["spmv_edges"]
    t1 = statistics.median(ms1[1:])
    print(json.dumps({"cfg": cfg, "k": 1, "api": "lap_solve", "solve_ms": t1, "iters": it1,
                      "edges_rhs_per_s": e1 / (t1 * 1e-3)}), flush=True)
    for k in [int(v) for v in os.environ.get("BLOCK_KS", "2,4,8").split(",")]:
        B = torch.from_numpy(np.stack([lapgen.rhs(g.n, seed=j) for j in range(k)])).to(dev)
        X = torch.zeros_like(B)
        ms = []
        for rep in range(3):
            _, it, rr, rc = h.solve_block(B, X, stream=s)
            st = h.stats()
            ms.append(st["solve_ms"])
        t = statistics.median(ms[1:])
        print(json.dumps({"cfg": cfg, "k": k, "api": "lap_solve_block", "solve_ms": t, "iters": it.tolist(),
                          "max_relres": float(rr.max()), "rc": rc,
                          "edges_rhs_per_s": st["spmv_edges"] / (t * 1e-3),
                          "speedup_vs_k_single": k * t1 / t}), flush=True)
    h.close()
