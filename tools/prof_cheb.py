"""Profile target: build the cfg-k hierarchy and run the dominant kernel
(fused Chebyshev SpMV on the finest aggregation level) a few times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import lapgen, paper_1705_06266_b200 as P
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
g = lapgen.config(k)
h = P.Hierarchy(g)
lv = h.first_agg_level()
ms, by, ed = h.bench_op(1, lv, int(sys.argv[2]) if len(sys.argv) > 2 else 5)
print(f"cfg{k} level {lv}: {ms.mean()*1e3:.1f} us/launch, {by/ms.mean()/1e6:.0f} GB/s")
