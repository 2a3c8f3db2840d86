import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lapgen, paper_1705_06266_b200 as P
for side in [16, 24, 32, 40, 48, 64, 96]:
    g = lapgen.grid3d(side)
    try:
        h = P.Hierarchy(g, use_graphs=0)
        print(side, "ok", h.nlev, flush=True)
    except Exception as e:
        print(side, "FAIL", e, flush=True)
        break
