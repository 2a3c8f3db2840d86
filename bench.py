#!/usr/bin/env python
"""bench.py -- B200 benchmark of the graph-Laplacian multigrid hot path.

One STEP = one pass of the whole hot path over
the workload resident in HBM: lap_setup (random order, elimination /
aggregation hierarchy, Galerkin, lambda-hat, coarsest L^+) followed by
lap_solve (PCG + V-cycle to 1e-8 relative residual), both through the C ABI
of liblap.so.

metric  = BASELINE.json's "V-cycle SpMV edges/s & HBM GB/s vs roofline; time
          to 1e-8 relative residual".  value = the solve's SpMV edges (SURVEY
          M2: per V-cycle sum over aggregation levels of 4 nnz_off(L_l), plus
          the PCG's fine products q = L p and residuals) divided by the WHOLE
          step's device time (setup + solve, max over ranks).  The setup's own
          semiring SpMVs are not counted as edges.  The same line carries the
          solve-only and V-cycle-only edges/s (M2), the V-cycle and dominant-
          kernel GB/s against the measured HBM roofline AND against the
          measured random-gather ceiling (M3), time to 1e-8, setup time.
workload (N=1) = BASELINE.json configs[3] (cfg 4: Barabasi-Albert n=4,194,304,
          m=8, w~U[0.5,2]), the largest single-GPU config; --config k picks
          another (cfg 5 = R-MAT s26).
cpu_baseline = the CPU oracle (oracle/, OpenMP over all host cores, bitwise
          identical to 1 thread) on the SAME input: one setup + one solve,
          the same edges/time formula; plus fine-SpMV medians at 1 thread and
          at all threads, and the host CPU model.
--impl reference = the oracle on the same input and host cores; its step is
          the GPU arm's step (a full setup + one PCG solve to 1e-8, the same
          edges / time formula; ~16 s per step on 16 cores for cfg 4; at most
          one warm-up step: the oracle has no warm-up state).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import lapgen  # noqa: E402

CFG = 4
METRIC = "V-cycle SpMV edges/s & HBM GB/s vs roofline; time to 1e-8 relative residual"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
GRIDS = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}  # pr x pc process grids


def peaks():
    fn = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(fn):
        with open(fn) as f:
            return json.load(f), "measured"
    return PEAKS_FALLBACK, "fallback"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------- clocks
class Clocks:
    """Clock / throttle-reason sampler during the timed region (B200_PROFILING.md
    recipe).  In-process NVML (the library nvidia-smi reads; same clocks.sm,
    clocks.max.sm and clocks_event_reasons fields) every 200 ms from a thread:
    a polling `nvidia-smi -lms` child measurably slowed the timed steps (~4 ms
    of 86 ms on cfg 2, driver calls contending with the CUDA stream).  Falls
    back to `nvidia-smi -lms 200` when pynvml is missing."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, enabled: bool = True):
        self.idx = gpu_index
        self.p = None
        self.enabled = enabled

    def _nvml_loop(self, nv, hdl):
        names = [("hw_slowdown", nv.nvmlClocksEventReasonHwSlowdown),
                 ("hw_thermal_slowdown", nv.nvmlClocksEventReasonHwThermalSlowdown),
                 ("sw_thermal_slowdown", nv.nvmlClocksEventReasonSwThermalSlowdown),
                 ("sw_power_cap", nv.nvmlClocksEventReasonSwPowerCap)]
        mx = nv.nvmlDeviceGetMaxClockInfo(hdl, nv.NVML_CLOCK_SM)
        while not self._stop.wait(0.2 if self.lines else 0.02):
            try:
                sm = nv.nvmlDeviceGetClockInfo(hdl, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(hdl)
            except Exception:
                break
            act = ["Active" if r & bit else "Not Active" for _, bit in names]
            self.lines.append(", ".join([str(self.idx), str(sm), str(mx), "0", hex(r)] + act))

    def __enter__(self):
        self.lines = []
        if not self.enabled:
            return self
        try:
            import threading
            import pynvml as nv
            nv.nvmlInit()
            hdl = nv.nvmlDeviceGetHandleByIndex(self.idx)
            self._stop = threading.Event()
            self._t = threading.Thread(target=self._nvml_loop, args=(nv, hdl), daemon=True)
            self._t.start()
            return self
        except Exception:
            self._t = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if getattr(self, "_t", None) is not None:
            self._stop.set()
            self._t.join(timeout=5)
            return
        self.lines = []
        if self.p is not None:
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "sampler": "nvml" if getattr(self, "_t", None) is not None else "nvidia-smi"}


# ---------------------------------------------------------------- GPU arm
def level_table(h):
    """Per-level sizes for the work accounting (host copies, outside timing)."""
    out = []
    for l in range(h.nlev):
        kind, n, nnz, lam = h.level_info(l)
        L = {"kind": kind, "n": n, "nnz": nnz, "lambda": lam}
        if kind == 0 and l + 1 < h.nlev:
            L["m"] = h.level_info(l + 1)[1]
        if kind == 1:  # works when the logical CSR was released too (cfg 5)
            frows = np.flatnonzero(h.level_map(l) < 0)
            L["nF"] = int(len(frows))
            L["nnz_fc"] = int(h.level_degrees(l, frows).sum())
        out.append(L)
    return out


def gather_ceiling(P, n, stream, reps=5):
    """M3 second ceiling: random 8-byte gathers from an x of n doubles with the
    SpMV's 12 B/entry streams (lap_bench_gather, 2^26 gathers)."""
    m = 1 << 26
    t = float(np.median(P.bench_gather(max(1, n), m, reps, stream=stream)))
    gps = m / (t * 1e-3)
    return {"x_bytes": 8 * n, "gathers_per_s": gps, "spmv_equiv_gbs": 12.0 * gps / 1e9}


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_1705_06266_b200 as P
    from paper_1705_06266_b200 import metrics as MX

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    P.pool_retain(1 << 40)  # keep liblap's pool reserved across the steps (no re-mapping per setup)
    # sharded solve (G1) over a pr x pc grid for N > 1 (or --shard at N = 1): the
    # library's own NCCL communicators; torch.distributed only broadcasts the id
    comm = None
    grid = None
    if world > 1 or args.shard:
        grid = GRIDS.get(world, (1, world))
        uid = [P.Comm.unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(uid, src=0)
        comm = P.Comm(grid[0], grid[1], nccl_id=uid[0], rank=rank)

    g = lapgen.config(args.config)
    b = lapgen.rhs(g.n)
    K = 2  # cheby_degree (the paper's)
    # inputs resident in HBM
    rp_d = torch.from_numpy(g.row_ptr).to(dev)
    col_d = torch.from_numpy(g.col).to(dev)
    w_d = torch.from_numpy(g.w).to(dev) if g.w is not None else None  # cfg 5: unit weights (NULL)
    b_d = torch.from_numpy(b).to(dev)
    x_d = torch.zeros_like(b_d)
    gd = lapgen.Graph(g.n, rp_d, col_d, w_d, g.name)
    # pinned host copies for the end-to-end measurement
    rp_h = torch.from_numpy(g.row_ptr).pin_memory()
    col_h = torch.from_numpy(g.col).pin_memory()
    w_h = torch.from_numpy(g.w).pin_memory() if g.w is not None else None
    b_h = torch.from_numpy(b).pin_memory()
    x_h = torch.zeros(g.n, dtype=torch.float64).pin_memory()

    class _HostG:  # host-pointer graph (on_device = 0) from pinned tensors
        n = g.n
        row_ptr, col, w = rp_h.numpy(), col_h.numpy(), (w_h.numpy() if w_h is not None else None)

    levels = None

    def step(graph, bb, xx):
        w0 = time.perf_counter()
        h = P.Hierarchy(graph, stream=stream, comm=comm)
        w1 = time.perf_counter()
        st0 = h.stats()
        _, it, rr, rc = h.solve(bb, xx, stream=stream)
        w2 = time.perf_counter()
        st = h.stats()
        out = dict(iters=it, relres=rr, rc=rc, setup_ms=st0["setup_ms"], solve_ms=st["solve_ms"],
                   launches=st0["kernel_launches"] + st["kernel_launches"], vcycles=st["vcycles"],
                   wall_setup_ms=1e3 * (w1 - w0), wall_solve_ms=1e3 * (w2 - w1))
        return h, out

    with torch.cuda.stream(stream):
        for i in range(args.warmup):
            h, r = step(gd, b_d, x_d)
            if levels is None:
                levels = level_table(h)
            h.close()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        runs = []
        with Clocks(local, enabled=not args.no_clocks) as clk:
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0.record(stream)
            for _ in range(args.steps):
                h, r = step(gd, b_d, x_d)
                w3 = time.perf_counter()
                h.close()
                r["wall_free_ms"] = 1e3 * (time.perf_counter() - w3)
                runs.append(r)
            t1.record(stream)
            torch.cuda.synchronize()
        total_ms = t0.elapsed_time(t1)
        if world > 1:
            dist.barrier()
        # ---- per-operation timing on the same stream, after the timed region (M2, M3, M4)
        hs = P.Hierarchy(gd, stream=stream)
        if levels is None:
            levels = level_table(hs)
        lv = hs.first_agg_level()
        t_cheb, bytes_cheb, _ = hs.bench_op(1, lv, 50, stream=stream)          # dominant kernel (H2)
        t_spmv, bytes_spmv, e_spmv = hs.bench_op(0, 0, 100, stream=stream)    # fine SpMV (H1)
        t_vc, bytes_vc, e_vc = hs.bench_op(2, 0, 20, stream=stream)           # V-cycle (H16)
        per_level = []
        ceil_cache = {}
        for l, L in enumerate(levels):
            if L["kind"] == 2 or L["nnz"] == 0:
                continue
            ts, bs, es = hs.bench_op(0, l, 30, stream=stream)
            ent = {"level": l, "kind": L["kind"], "n": L["n"], "nnz": L["nnz"],
                   "spmv_us": float(np.median(ts)) * 1e3, "spmv_gbs": bs / (float(np.median(ts)) * 1e-3) / 1e9}
            if L["kind"] == 0:
                tc, bc, _ = hs.bench_op(1, l, 30, stream=stream)
                ent["cheb_us"] = float(np.median(tc)) * 1e3
                ent["cheb_gbs"] = bc / (float(np.median(tc)) * 1e-3) / 1e9
            if L["n"] >= 100000:  # the gather ceiling is meaningful for levels larger than L1 reach
                key = L["n"]
                if key not in ceil_cache:
                    ceil_cache[key] = gather_ceiling(P, L["n"], stream)
                c = ceil_cache[key]
                ent["gather_ceiling_us"] = L["nnz"] / c["gathers_per_s"] * 1e6
                ent["spmv_frac_of_gather_ceiling"] = ent["gather_ceiling_us"] / ent["spmv_us"]
            per_level.append(ent)
        solve_ms = []
        for _ in range(5):
            _, it_s, rr_s, _ = hs.solve(b_d, x_d, stream=stream)
            solve_ms.append(hs.stats()["solve_ms"])
        hs.close()
        # ---- end to end through the C ABI with HOST buffers (graph + b H2D, x D2H inside)
        e2e_ms = []
        for _ in range(max(1, min(args.steps, 3))):
            torch.cuda.synchronize()
            e0 = time.perf_counter()
            he = P.Hierarchy(_HostG, stream=stream, comm=comm)
            he.solve(b_h.numpy(), x_h.numpy(), stream=stream)
            torch.cuda.synchronize()
            e2e_ms.append((time.perf_counter() - e0) * 1e3)
            he.close()

    ms = total_ms / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clocks = clk.summary()
    if rank != 0:
        if comm is not None:
            comm.close()
        if world > 1:
            dist.destroy_process_group()
        return
    last = runs[-1]
    step_edges = [MX.solve_spmv_edges(levels, r["iters"], r["vcycles"], K) for r in runs]
    edges = float(np.mean(step_edges))
    pk, pk_src = peaks()
    hbm = float(pk.get("hbm_gbs", PEAKS_FALLBACK["hbm_gbs"]))
    ms_k = float(np.mean(t_cheb))
    achieved = bytes_cheb / (ms_k * 1e-3) / 1e9
    Ld = levels[lv]
    gc = gather_ceiling(P, Ld["n"], stream)
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"cfg{args.config}", {}).get("cheb_bytes_per_launch")
        except Exception:
            traffic = None
    nnz0 = levels[0]["nnz"]
    sp_med = float(np.median(t_spmv))
    vc_med = float(np.median(t_vc))
    vc_edges = MX.vcycle_spmv_edges(levels, K)
    t_solve = float(np.median(solve_ms))
    work = MX.solve_work(levels, last["iters"], last["vcycles"])
    dr = last["relres"]
    setup_med = float(np.median([r["setup_ms"] for r in runs]))
    solve_med = float(np.median([r["solve_ms"] for r in runs]))
    m2 = {
        "fine_spmv": {"edges_per_s": nnz0 / (sp_med * 1e-3), "gbs": bytes_spmv / (sp_med * 1e-3) / 1e9,
                      "us_median_of_100": sp_med * 1e3,
                      "frac_measured": bytes_spmv / (sp_med * 1e-3) / 1e9 / hbm,
                      "frac_8000": bytes_spmv / (sp_med * 1e-3) / 1e9 / 8000.0},
        "vcycle": {"edges_per_s": vc_edges / (vc_med * 1e-3), "edges_per_vcycle": vc_edges,
                   "gbs_method_bytes": bytes_vc / (vc_med * 1e-3) / 1e9, "bytes_per_vcycle": bytes_vc,
                   "us_median_of_20": vc_med * 1e3, "frac_measured": bytes_vc / (vc_med * 1e-3) / 1e9 / hbm,
                   "bytes_note": "method bytes of every level's kernels (SURVEY M3); the dense-tail GEMV is booked "
                                 "with the bytes of the sub-cycle it replaces, not its own 8 n_t^2"},
        "solve_only_edges_per_s": edges / (solve_med * 1e-3),
        "time_to_1e8_ms_median_of_5": t_solve, "iters": last["iters"], "true_rel_residual": dr,
        "setup_ms_median": setup_med,
        "work_units": work, "wda": MX.wda(work, dr) if 0 < dr < 1 else None,
        "tda_ms": MX.tda(t_solve, dr) if 0 < dr < 1 else None,
        "operator_complexity": sum(L["n"] + L["nnz"] for L in levels) / (levels[0]["n"] + nnz0),
        "per_level": per_level,
    }
    # the oracle at cfg 5 needs ~120 GB of host RAM and ~10 min: not in the bench line
    # (its full-size parity run is tests/test_gpu_cfg5.py with LAP_TEST_CFG5_ORACLE=1)
    cpu = cpu_baseline(args, g, b) if (world == 1 and not args.no_cpu and g.nnz < (1 << 28)) else None
    h2d = g.row_ptr.nbytes + g.col.nbytes + (g.w.nbytes if g.w is not None else 0) + b.nbytes
    e2e_med = statistics.median(e2e_ms)
    line = {
        "metric": METRIC,
        # whole job: ONE system sharded over the N GPUs (strong scaling), so the job
        # traverses `edges` edges per step whatever N is
        "value": edges / (ms * 1e-3),
        "unit": "edges/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (lapgen, seeded)",
        "config": {"workload": lapgen.CONFIG_NAMES[args.config], "n": g.n, "nnz_off": g.nnz,
                   "parallelism": ("single GPU" if comm is None else
                                   f"2D edge partition {grid[0]}x{grid[1]} of the fine levels (NCCL), coarse levels replicated"),
                   "l2": "inputs > L2: the level-0 CSR + SELL copy exceed the 126 MB L2; every SpMV re-streams them",
                   "levels": [[L["kind"], L["n"], L["nnz"]] for L in levels],
                   "value_definition": "solve-phase SpMV edges (M2: V-cycles x sum_agg 4 nnz_l + (iters+2) nnz_0) "
                                       "per second of the whole step (setup + solve)"},
        "iters": last["iters"], "rel_residual": dr,
        "time_to_1e8_ms": t_solve,
        "setup_ms": setup_med,
        "solve_ms": solve_med,
        "vcycle_edges_per_s": m2["vcycle"]["edges_per_s"],
        "vcycle_gbs": m2["vcycle"]["gbs_method_bytes"],
        "m2": m2,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm, "traffic": traffic,
                     "kernel": f"fused Chebyshev/Jacobi SpMV step (H2, k_spmv<E_CHEB>) on level {lv}",
                     "bytes_per_launch": bytes_cheb, "ms_per_launch": ms_k,
                     "timing": "CUDA events on the solve stream, 50 launches in one graph, same process, after the timed region",
                     "frac_of_8000": achieved / 8000.0, "peak_source": pk_src,
                     "second_ceiling": {
                         "bound": "L1TEX/L2 request rate of random 8-byte x gathers (SURVEY M3)",
                         "gathers_per_s": gc["gathers_per_s"], "spmv_equiv_gbs": gc["spmv_equiv_gbs"],
                         "spmv_equiv_frac_of_hbm": gc["spmv_equiv_gbs"] / hbm,
                         "kernel_us_at_ceiling": Ld["nnz"] / gc["gathers_per_s"] * 1e6,
                         "kernel_frac_of_ceiling": (Ld["nnz"] / gc["gathers_per_s"]) / (ms_k * 1e-3),
                         "how": "lap_bench_gather: 2^26 uniform random gathers from an x of the level's size, "
                                "with int32 col + fp64 w streamed"}},
        "e2e": {"value": edges / (e2e_med * 1e-3), "unit": "edges/s",
                "ms": e2e_med, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": b.nbytes},
        "gpu_launches": int(sum(r["launches"] for r in runs)),
        "step_breakdown_ms": {k: float(np.median([r[k] for r in runs])) for k in
                              ["setup_ms", "solve_ms", "wall_setup_ms", "wall_solve_ms", "wall_free_ms"]},
        "clocks": clocks,
        "cpu_baseline": cpu,
    }
    emit(line)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------- CPU oracle arm
def oracle_levels(h):
    out = []
    for L in h.levels():
        d = {"kind": L.kind, "n": L.n, "nnz": L.nnz}
        out.append(d)
    return out


def oracle_spmv_median(g, threads, reps=10):
    import oracle
    oracle.set_threads(threads)
    d = oracle.row_sums(g.n, g.row_ptr, g.w)
    x = np.random.default_rng(0).standard_normal(g.n)
    rp = np.ascontiguousarray(g.row_ptr, np.int64)
    col = np.ascontiguousarray(g.col, np.int32)
    w = np.ascontiguousarray(g.w, np.float64)
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        oracle.spmv(g.n, rp, col, w, d, x)
        ts.append(time.perf_counter() - t)
    return float(np.median(ts))


def cpu_baseline(args, g, b):
    """The oracle as it stands, all host cores (OpenMP, bitwise = 1 thread),
    on the same input: one setup + one solve, the GPU line's formula."""
    import oracle
    from paper_1705_06266_b200 import metrics as MX
    cores = host_cores()
    oracle.set_threads(cores)
    t0 = time.perf_counter()
    h = oracle.Hierarchy(g)
    t1 = time.perf_counter()
    x, it, rr, rc = h.solve(b)
    t2 = time.perf_counter()
    levels = oracle_levels(h)
    edges = MX.solve_spmv_edges(levels, it, it)
    sp1 = oracle_spmv_median(g, 1)
    spn = oracle_spmv_median(g, cores)
    oracle.set_threads(cores)
    return {"value": edges / (t2 - t0), "unit": "edges/s", "cores": cores, "kind": "oracle",
            "sample": f"the full {lapgen.CONFIG_NAMES[args.config]} input: one oracle setup ({t1 - t0:.1f} s) + one "
                      f"PCG solve to 1e-8 ({t2 - t1:.1f} s, {it} iters) on {cores} OpenMP threads; same edges/time "
                      f"formula as the GPU value",
            "setup_s": t1 - t0, "solve_s": t2 - t1, "iters": it, "rel_residual": rr,
            "solve_only_edges_per_s": edges / (t2 - t1),
            "fine_spmv_median_of_10": {"threads_1_s": sp1, f"threads_{cores}_s": spn,
                                       "edges_per_s_1": g.nnz / sp1, f"edges_per_s_{cores}": g.nnz / spn},
            "cpu": cpu_model()}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    from paper_1705_06266_b200 import metrics as MX
    cores = host_cores()
    oracle.set_threads(cores)
    g = lapgen.config(args.config)
    b = lapgen.rhs(g.n)
    # one step = what the GPU arm's step is: a full setup + one PCG solve to 1e-8
    # on the whole workload (the same edges / time formula); the oracle has no
    # warm-up state, so at most one warm-up step is run (~16 s each on 16 cores)
    def step():
        t = time.perf_counter()
        h = oracle.Hierarchy(g)
        t1 = time.perf_counter()
        x, it, rr, rc = h.solve(b)
        t2 = time.perf_counter()
        return h, it, t1 - t, t2 - t1
    h = None
    for _ in range(min(args.warmup, 1)):
        h, _, _, _ = step()
    levels = None
    tot_t, tot_e, it, setup_s, solve_s = 0.0, 0, 0, 0.0, 0.0
    for _ in range(args.steps):
        h, it, ts, tv = step()
        if levels is None:
            levels = oracle_levels(h)
        tot_t += ts + tv
        setup_s += ts
        solve_s += tv
        tot_e += MX.solve_spmv_edges(levels, it, it)
    v = tot_e / tot_t
    setup_s /= max(1, args.steps)
    solve_s /= max(1, args.steps)
    sample = (f"{lapgen.CONFIG_NAMES[args.config]}, full size; step = one oracle setup ({setup_s:.1f} s) + one PCG "
              f"solve to 1e-8 ({solve_s:.1f} s, {it} iters) with {cores} OpenMP threads, as the GPU arm's step")
    emit({
        "impl": "reference",
        "metric": METRIC,
        "value": v, "unit": "edges/s", "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (lapgen, seeded)",
        "config": {"workload": lapgen.CONFIG_NAMES[args.config], "n": g.n, "nnz_off": g.nnz, "sample": sample},
        "setup_s": setup_s, "solve_s": solve_s,
        "cpu_baseline": {"value": v, "unit": "edges/s", "cores": cores, "kind": "oracle", "sample": sample,
                         "cpu": cpu_model()},
        "e2e": {"value": v, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })


_JSON_OUT = None


def emit(line: dict):
    """The one JSON line on the process's real stdout (libraries such as NCCL
    may print to fd 1; everything else is redirected to stderr in main())."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lap", choices=["lap", "reference"])
    ap.add_argument("--config", type=int, default=CFG)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--shard", action="store_true", help="sharded (NCCL 1x1 grid) path at N = 1")
    ap.add_argument("--no-clocks", action="store_true", help="diagnostics: no nvidia-smi sampling")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
