import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lapgen, paper_1705_06266_b200 as P
g = lapgen.grid3d(int(sys.argv[1]))
h = P.Hierarchy(g, use_graphs=0)
print("ok", h.nlev)
