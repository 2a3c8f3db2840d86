"""Host-side logic of the sharded solve on CPU, no GPU:

* the piece map exported by liblap (lap_dist_index, host-only): a bijection
  of storage rows onto real slots, block-cyclic over the pieces, pads only at
  the end of each piece, every piece within one block of the others;
* the 2D SpMV exchange that dist.cu implements (column allgather of x, local
  block product, row reduce-scatter of A x), run with torch.distributed
  'gloo' in world_size-2 process groups on grids 1x2 and 2x1 and in a
  world_size-4 group on the 2x2 grid, reproduces the global A x.

The local block products here are numpy (the CPU stand-in for k_blk_spmv);
the piece map, block index scheme and collective pattern are the ones the
library uses.
"""
import os
import socket

import numpy as np
import pytest

import lapgen


def _lib():
    from paper_1705_06266_b200 import build
    build.build()
    import paper_1705_06266_b200 as P
    return P


@pytest.mark.parametrize("n,P", [(1, 1), (255, 2), (1000, 3), (4096, 4), (10007, 8), (300, 16)])
def test_piece_map(n, P):
    L = _lib()
    rows = np.arange(n)
    d, S = L.dist_index(n, P, rows)
    assert S % 256 == 0 and S * P >= n
    assert len(np.unique(d)) == n                          # injective
    piece, slot = d // S, d % S
    assert piece.min() >= 0 and piece.max() < P
    counts = np.bincount(piece, minlength=P)
    assert counts.max() - counts.min() <= 256              # balanced to one block
    for k in range(P):                                     # real slots are a prefix of each piece
        sl = np.sort(slot[piece == k])
        assert np.array_equal(sl, np.arange(len(sl)))
    # block-cyclic: rows of one 256-block share a piece and are consecutive slots
    blk = rows // 256
    assert np.all(piece == blk % P)


def _global_spmv(g, x):
    rows = np.repeat(np.arange(g.n), np.diff(g.row_ptr))
    y = np.zeros(g.n)
    np.add.at(y, rows, g.w * x[g.col])
    return y


def _worker(rank, world, port, pr, pc, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        L = _lib()
        g = lapgen.random_connected(3000, 9000, 11)
        n = g.n
        d, S = L.dist_index(n, world, np.arange(n))
        gi, gj = rank // pc, rank % pc
        # row / column communicators (same split as lap_comm_create)
        rows_groups = [dist.new_group([i * pc + j for j in range(pc)]) for i in range(pr)]
        col_groups = [dist.new_group([i * pc + j for i in range(pr)]) for j in range(pc)]
        rg, cg = rows_groups[gi], col_groups[gj]
        # this rank's block: rows in row block gi, columns in column block gj (local ids)
        piece = d // S
        rows_of = np.repeat(np.arange(n), np.diff(g.row_ptr))
        drow, dcol = d[rows_of], d[g.col]
        in_rows = (drow // S) // pc == gi
        in_cols = (dcol // S) % pc == gj
        sel = in_rows & in_cols
        lrow = drow[sel] - gi * pc * S
        lcol = ((dcol[sel] // S) // pc) * S + dcol[sel] % S
        wv = g.w[sel]
        # owned piece of x (pads 0)
        x = np.random.default_rng(0).standard_normal(n)
        xd = np.zeros(world * S)
        xd[d] = x
        own = torch.from_numpy(xd[rank * S:(rank + 1) * S].copy())
        # column allgather (column communicator rank order = grid row order)
        parts = [torch.zeros(S, dtype=torch.float64) for _ in range(pr)]
        dist.all_gather(parts, own, group=cg)
        xcol = torch.cat(parts).numpy()
        ypart = np.zeros(pc * S)
        np.add.at(ypart, lrow, wv * xcol[lcol])
        # row reduce-scatter (row communicator rank order = grid column order)
        out = torch.zeros(S, dtype=torch.float64)
        segs = [torch.from_numpy(ypart[j * S:(j + 1) * S].copy()) for j in range(pc)]
        dist.reduce_scatter(out, segs, group=rg)
        full = [torch.zeros(S, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(full, out)
        yd = torch.cat(full).numpy()
        yref = _global_spmv(g, x)
        err = np.abs(yd[d] - yref).max()
        q.put((rank, float(err), float(np.abs(yd).max() if np.all(yd[np.setdiff1d(np.arange(world * S), d)] == 0) else -1)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("pr,pc", [(1, 2), (2, 1), (2, 2)])
def test_2d_exchange_reproduces_global_spmv_gloo(pr, pc):
    import torch.multiprocessing as mp
    world = pr * pc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, pr, pc, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, err, padchk in res:
        assert err <= 1e-12, (rank, err)
        assert padchk >= 0, "pads of the reduce-scattered y must be exactly 0"
