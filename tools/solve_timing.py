"""Solve-phase timing matrix: cfg x {PDL on/off} x {graphs on/off}.
Usage: python tools/solve_timing.py [cfgs...]   (each variant in a subprocess,
since LAP_PDL is read once per process)."""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, sys, statistics
sys.path.insert(0, %r)
import torch, lapgen, paper_1705_06266_b200 as P
k, ug = int(sys.argv[1]), int(sys.argv[2])
g = lapgen.config(k); b = lapgen.rhs(g.n)
dev = torch.device("cuda", 0)
gd = lapgen.Graph(g.n, torch.from_numpy(g.row_ptr).to(dev), torch.from_numpy(g.col).to(dev), torch.from_numpy(g.w).to(dev))
bt = torch.from_numpy(b).to(dev); xt = torch.zeros_like(bt)
s = torch.cuda.Stream()
res = []
for rep in range(4):
    h = P.Hierarchy(gd, stream=s, use_graphs=ug)
    st0 = h.stats()
    _, it, rr, rc = h.solve(bt, xt, stream=s)
    st = h.stats()
    res.append((st0["setup_ms"], st["solve_ms"], it, rr, st["vcycles"], st["kernel_launches"]))
    h.close()
r = res[1:]
print(json.dumps({"cfg": k, "graphs": ug, "pdl": os.environ.get("LAP_PDL", "1"),
                  "setup_ms": statistics.median(x[0] for x in r), "solve_ms": statistics.median(x[1] for x in r),
                  "iters": r[-1][2], "relres": r[-1][3], "vcycles": r[-1][4], "launches": r[-1][5],
                  "ms_per_iter": statistics.median(x[1] for x in r) / max(1, r[-1][2])}))
''' % ROOT
args = [a for a in sys.argv[1:] if not a.startswith("--")]
quick = "--quick" in sys.argv
cfgs = [int(a) for a in args] or [1, 2, 3, 4]
for k in cfgs:
    for pdl in (["1"] if quick else ["1", "0"]):
        for ug in ([1] if quick else [1, 0]):
            env = dict(os.environ, LAP_PDL=pdl)
            r = subprocess.run([sys.executable, "-c", CHILD, str(k), str(ug)], env=env, capture_output=True, text=True)
            print(r.stdout.strip() or r.stderr[-1500:], flush=True)
