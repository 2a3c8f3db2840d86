"""Sharded (2D edge partition) solve, on one GPU.

lap_comm_create_virtual(pr, pc) holds every rank's shard of a pr x pc grid
in this process and runs the collectives as device copies / fixed-order sums,
so the whole sharded data path (piece map, 2D blocks, column allgather, row
reduce-scatter, distributed restriction / prolongation, distributed PCG) runs
through liblap.so on a single B200.  Contract (SURVEY §8(e) "Determinism"):
the hierarchy is the single-GPU one; the solve agrees with the single-GPU
solve up to rounding: true relative residual <= 1e-8, iterations within +-1,
solution within 1e-6 relative.
"""
import numpy as np
import pytest

import lapgen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def P():
    import paper_1705_06266_b200 as P
    from paper_1705_06266_b200 import build
    build.build()
    return P


GRAPHS = {
    "grid2d_37x29": lambda: lapgen.grid2d(37, 29),
    "rmat12": lambda: lapgen.rmat(12),
    "ba3000": lambda: lapgen.barabasi_albert(3000, 6),
    "rand2000": lambda: lapgen.random_connected(2000, 6000, 3),
    "star20000": lambda: lapgen.star(20000),
    "grid3d_14": lambda: lapgen.grid3d(14),
}
GRIDS = [(1, 1), (1, 2), (2, 1), (2, 2), (2, 3), (3, 2), (2, 4)]


@pytest.mark.parametrize("gname", list(GRAPHS))
@pytest.mark.parametrize("grid", GRIDS, ids=[f"{a}x{b}" for a, b in GRIDS])
def test_sharded_solve_matches_single_gpu(P, gname, grid):
    g = GRAPHS[gname]()
    b = lapgen.rhs(g.n, seed=5)
    h1 = P.Hierarchy(g)
    x1, it1, rr1, rc1 = h1.solve(b)
    comm = P.Comm(*grid)
    # replicate_nnz = 1: every level except the coarsest is sharded
    hd = P.Hierarchy(g, comm=comm, replicate_nnz=1)
    xd, itd, rrd, rcd = hd.solve(b)
    assert rc1 == 0 and rcd == 0
    assert rrd <= 1e-8, rrd
    assert abs(itd - it1) <= 1, (itd, it1)
    assert np.abs(xd - x1).max() <= 1e-6 * np.abs(x1).max()
    hd.close()
    comm.close()


@pytest.mark.parametrize("rep", [0, 1 << 40])
def test_replication_threshold(P, rep):
    """Default threshold (nnz(L0)/(32P)) and 'replicate everything below level 0'."""
    g = lapgen.rmat(12)
    b = lapgen.rhs(g.n, seed=1)
    x1, it1, _, _ = P.Hierarchy(g).solve(b)
    comm = P.Comm(2, 2)
    hd = P.Hierarchy(g, comm=comm, replicate_nnz=rep)
    xd, itd, rrd, rc = hd.solve(b)
    assert rc == 0 and rrd <= 1e-8 and abs(itd - it1) <= 1
    assert np.abs(xd - x1).max() <= 1e-6 * np.abs(x1).max()
    hd.close()
    comm.close()


def test_sharded_solve_device_buffers_and_oracle(P):
    g = lapgen.grid2d(64, 64, "cfg1")
    b = lapgen.rhs(g.n)
    comm = P.Comm(2, 4)
    hd = P.Hierarchy(g, comm=comm, replicate_nnz=1)
    bt = torch.from_numpy(b).cuda()
    xd, itd, rrd, rc = hd.solve(bt)
    xo, ito, _, _ = oracle.Hierarchy(g).solve(b)
    assert rc == 0 and rrd <= 1e-8 and abs(itd - ito) <= 1
    xd = xd.cpu().numpy()
    assert np.abs(xd - xo).max() <= 1e-6 * np.abs(xo).max()
    assert abs(xd.mean()) <= 1e-10 * np.abs(xd).max()
    hd.close()
    comm.close()


def test_comm_info_and_invalid(P):
    c = P.Comm(2, 3)
    assert c.info() == {"rank": 0, "nranks": 6, "grid_rows": 2, "grid_cols": 3, "virtual": 1}
    c.close()
    with pytest.raises(P.LapError):
        P.Comm(5, 4)   # more than 16 ranks


def test_nccl_transport_single_rank(P):
    """The NCCL communicator path (ncclCommInitRank + row/column splits,
    ncclAllGather / ncclReduceScatter / ncclAllReduce) on a 1 x 1 grid."""
    uid = P.Comm.unique_id()
    comm = P.Comm(1, 1, nccl_id=uid, rank=0)
    assert comm.info()["virtual"] == 0
    g = lapgen.rmat(11)
    b = lapgen.rhs(g.n, seed=2)
    x1, it1, _, _ = P.Hierarchy(g).solve(b)
    hd = P.Hierarchy(g, comm=comm, replicate_nnz=1)
    xd, itd, rrd, rc = hd.solve(b)
    assert rc == 0 and rrd <= 1e-8 and abs(itd - it1) <= 1
    assert np.abs(xd - x1).max() <= 1e-6 * np.abs(x1).max()
    hd.close()
    comm.close()


def test_nccl_distributed_setup_single_rank(P, monkeypatch):
    """The distributed setup's NCCL gather (entry counts all-gathered, one
    ncclBroadcast per root, row_ptr pieces shifted) and the row-split passes'
    sharing (in-place broadcasts, the vote / F-count allreduces) on a real
    1 x 1 NCCL communicator with every split forced (LAP_DSETUP_MIN=0):
    the hierarchy equals the single-GPU one bit for bit and the sharded solve
    (own-piece SpMV on the side stream) converges like it."""
    g = lapgen.barabasi_albert(4000, 7)
    h1 = P.Hierarchy(g)
    monkeypatch.setenv("LAP_DSETUP_MIN", "0")
    uid = P.Comm.unique_id()
    comm = P.Comm(1, 1, nccl_id=uid, rank=0)
    hd = P.Hierarchy(g, comm=comm, replicate_nnz=1)
    for l in range(h1.nlev - 1):
        assert _level_bits(hd, l) == _level_bits(h1, l), l
    b = lapgen.rhs(g.n, seed=3)
    x1, it1, _, _ = h1.solve(b)
    xd, itd, rrd, rc = hd.solve(b)
    assert rc == 0 and rrd <= 1e-8 and abs(itd - it1) <= 1
    hd.close()
    comm.close()


def test_sharded_pcg_graph_replays_eager_bitwise(P):
    """The sharded PCG replays its per-iteration preconditioner step (V-cycle
    with the collectives, projection, dots) as one captured CUDA graph; the
    graph does exactly what the eager launches do (bit-identical solution),
    and solving twice with the captured graph is reproducible."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, lapgen, paper_1705_06266_b200 as P, sys\n"
            "out = []\n"
            "for g in [lapgen.rmat(12), lapgen.grid3d(14)]:\n"
            "    for grid in [(2, 2), (2, 3)]:\n"
            "        comm = P.Comm(*grid); h = P.Hierarchy(g, comm=comm, replicate_nnz=1)\n"
            "        b = lapgen.rhs(g.n, seed=5); x, it, rr, rc = h.solve(b); x2, it2, _, _ = h.solve(b)\n"
            "        assert rc == 0 and rr <= 1e-8 and it2 == it and x2.tobytes() == x.tobytes()\n"
            "        out.append(x); h.close(); comm.close()\n"
            "np.save(sys.argv[1], np.concatenate(out))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for flag in ["1", "0"]:
        fn = os.path.join(root, f"gpurun_out_dist_{flag}.npy")
        e = dict(os.environ, LAP_DIST_GRAPH=flag)
        r = subprocess.run([sys.executable, "-c", code, fn], env=e, capture_output=True, text=True, timeout=600, cwd=root)
        assert r.returncode == 0, r.stderr[-3000:]
        res.append(np.load(fn))
        os.remove(fn)
    assert res[0].tobytes() == res[1].tobytes()


def _level_bits(h, l):
    lv = h.level(l)
    out = [lv["kind"], lv["n"], lv["nnz"], lv["row_ptr"].tobytes(), lv["col"].tobytes(), lv["w"].tobytes(),
           lv["d"].tobytes()]
    for key in ("agg", "fmap"):
        if key in lv:
            out.append(lv[key].tobytes())
    return out


@pytest.mark.parametrize("gname", ["rmat12", "ba3000", "grid3d_14", "star20000"])
@pytest.mark.parametrize("grid", [(1, 2), (2, 2), (2, 3), (2, 4)], ids=["1x2", "2x2", "2x3", "2x4"])
@pytest.mark.parametrize("gal_fast", ["1", "0"], ids=["ordered", "batched"])
def test_distributed_setup_bit_identical(P, gname, grid, gal_fast, monkeypatch):
    """with a setup communicator the coarse-operator term builds
    (Galerkin -- ordered and batched paths --, Schur complement) are split by
    output rows over the ranks and gathered, and the row-parallel passes
    (elimination select, affinity, the ten vote rounds -- hub rows by chunks
    included, star20000) run on each rank's row range; every entry is still
    one CanonSum of its whole multiset with the level's global instance and
    every per-row result is computed once, so the hierarchy
    (every level's CSR, diagonal, aggregates / F sets, lambda-hat) equals the
    single-GPU one bit for bit.  LAP_DSETUP_MIN=0 splits every product."""
    g = GRAPHS[gname]()
    monkeypatch.setenv("LAP_GAL_FAST", gal_fast)
    h1 = P.Hierarchy(g)
    monkeypatch.setenv("LAP_DSETUP_MIN", "0")
    comm = P.Comm(*grid)
    hd = P.Hierarchy(g, comm=comm)
    assert hd.nlev == h1.nlev
    for l in range(h1.nlev - 1):
        assert _level_bits(hd, l) == _level_bits(h1, l), l
        assert hd.level_info(l) == h1.level_info(l), l
    b = lapgen.rhs(g.n, seed=2)
    x1, it1, _, _ = h1.solve(b)
    xd, itd, rrd, rc = hd.solve(b)
    assert rc == 0 and rrd <= 1e-8 and abs(itd - it1) <= 1
    hd.close()
    comm.close()


def test_distributed_setup_big_relabel(P, monkeypatch):
    """The level-0 relabel of a graph above 2^28 entries is a split term build
    too (forced here on a small graph, LAP_RELABEL_TERMS=1), with small
    batches inside every rank's range (LAP_TERM_BATCH)."""
    g = lapgen.rmat(13)
    monkeypatch.setenv("LAP_TERM_BATCH", "3000")
    monkeypatch.setenv("LAP_RELABEL_TERMS", "1")
    h1 = P.Hierarchy(g)
    monkeypatch.setenv("LAP_DSETUP_MIN", "0")
    comm = P.Comm(2, 2)
    hd = P.Hierarchy(g, comm=comm)
    for l in range(h1.nlev - 1):
        assert _level_bits(hd, l) == _level_bits(h1, l), l
    hd.close()
    comm.close()
