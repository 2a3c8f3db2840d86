"""cfg 5 (R-MAT scale 26) end to end on one B200: generate (C/OpenMP), copy to
the device, lap_setup (phase trace with LAP_SETUP_TRACE=1), lap_solve to 1e-8;
prints sizes, times and the pool peak."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import lapgen, paper_1705_06266_b200 as P
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
t = time.time()
g = lapgen.rmat_large(scale, 16) if scale != 26 else lapgen.config(5)
print(f"generate s{scale}: n={g.n} nnz={g.nnz} maxdeg={int(np.diff(g.row_ptr).max())} {time.time()-t:.1f} s", flush=True)
dev = torch.device("cuda", 0)
t = time.time()
gd = lapgen.Graph(g.n, torch.from_numpy(g.row_ptr).to(dev), torch.from_numpy(g.col).to(dev), None)
torch.cuda.synchronize()
print(f"h2d {time.time()-t:.1f} s; free {torch.cuda.mem_get_info()[0]/1e9:.1f} GB", flush=True)
P.pool_retain(1 << 40)
st = torch.cuda.Stream()
for rep in range(int(os.environ.get("REPS", "2"))):
    t = time.time()
    h = P.Hierarchy(gd, stream=st)
    torch.cuda.synchronize()
    print(f"setup rep {rep}: {h.stats()['setup_ms']:.1f} ms device, {time.time()-t:.2f} s wall", flush=True)
    if rep == 0:
        for l in range(h.nlev):
            print("level", l, h.level_info(l), flush=True)
    b = torch.from_numpy(lapgen.rhs(g.n)).to(dev)
    x, it, rr, rc = h.solve(b, stream=st)
    torch.cuda.synchronize()
    print(f"solve: iters {it} relres {rr:.3e} rc {rc} {h.stats()['solve_ms']:.1f} ms", flush=True)
    x, it, rr, rc = h.solve(b, stream=st)
    torch.cuda.synchronize()
    print(f"solve again: iters {it} {h.stats()['solve_ms']:.1f} ms", flush=True)
    if rep == 0:
        lv = h.first_agg_level()
        for l in range(h.nlev):
            kind = h.level_info(l)[0]
            if kind == 2:
                continue
            tt, bb, ee = h.bench_op(0, l, 10, stream=st)
            line = f"level {l} kind {kind}: spmv {np.median(tt)*1e3:.1f} us {bb/np.median(tt)/1e6:.0f} GB/s"
            if kind == 0:
                tt, bb, ee = h.bench_op(1, l, 10, stream=st)
                line += f" | cheb {np.median(tt)*1e3:.1f} us {bb/np.median(tt)/1e6:.0f} GB/s"
            print(line, flush=True)
        tt, bb, ee = h.bench_op(2, 0, 5, stream=st)
        print(f"vcycle {np.median(tt)*1e3:.1f} us {bb/np.median(tt)/1e6:.0f} GB/s {ee} edges", flush=True)
    h.close()
    print(f"free after close {torch.cuda.mem_get_info()[0]/1e9:.1f} GB", flush=True)
