"""V-cycle + PCG vs K-cycle + FCG (N2) on the BASELINE configs and two
high-diameter graphs: setup / solve ms, outer iterations, kernel launches,
SpMV edges per outer iteration (CUDA-event times from lap_get_stats)."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import lapgen, paper_1705_06266_b200 as P

dev = torch.device("cuda", 0)
cases = [(f"cfg{k}", lambda k=k: lapgen.config(k)) for k in (1, 2, 3, 4)]
cases += [("path_1M", lambda: lapgen.path(1 << 20)), ("grid2d_1024", lambda: lapgen.grid2d(1024, 1024))]
want = sys.argv[1:]
for name, mk in cases:
    if want and name not in want:
        continue
    g = mk()
    b = lapgen.rhs(g.n)
    gd = lapgen.Graph(g.n, torch.from_numpy(g.row_ptr).to(dev), torch.from_numpy(g.col).to(dev), torch.from_numpy(g.w).to(dev))
    bt = torch.from_numpy(b).to(dev)
    xt = torch.zeros_like(bt)
    s = torch.cuda.Stream()
    for cyc in (0, 1):
        res = []
        for rep in range(3):
            h = P.Hierarchy(gd, stream=s, cycle=cyc)
            _, it, rr, rc = h.solve(bt, xt, stream=s)
            st = h.stats()
            res.append((st["solve_ms"], it, rr, rc, st["kernel_launches"], st["spmv_edges"]))
            h.close()
        r = res[1:]
        print(json.dumps({"case": name, "cycle": "K" if cyc else "V", "solve_ms": statistics.median(x[0] for x in r),
                          "iters": r[-1][1], "relres": r[-1][2], "rc": r[-1][3], "launches": r[-1][4],
                          "edges_per_iter": r[-1][5] / max(1, r[-1][1]),
                          "ms_per_iter": statistics.median(x[0] for x in r) / max(1, r[-1][1])}), flush=True)
