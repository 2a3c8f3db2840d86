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
        own_x = own.numpy().copy()
        # column allgather (column communicator rank order = grid row order)
        parts = [torch.zeros(S, dtype=torch.float64) for _ in range(pr)]
        dist.all_gather(parts, own, group=cg)
        xcol = torch.cat(parts).numpy()
        ypart = np.zeros(pc * S)
        np.add.at(ypart, lrow, wv * xcol[lcol])
        # the library's split of A_ij (dist.cu build_part): columns of this rank's
        # OWN piece (local ids into the piece, usable before the column allgather)
        # and the rest of the column block; own + remote = the whole block product
        own = ((dcol[sel] // S) // pc) == gi
        y_own = np.zeros(pc * S)
        np.add.at(y_own, lrow[own], wv[own] * own_x[(dcol[sel] % S)[own]])
        y_rem = np.zeros(pc * S)
        np.add.at(y_rem, lrow[~own], wv[~own] * xcol[lcol[~own]])
        assert np.allclose(y_own + y_rem, ypart, rtol=1e-13, atol=1e-13)
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


# ---------------------------------------------------------------- distributed setup
def _galerkin_row_terms(lv):
    """terms of each coarse row of R L P: fine entries (i, j) with
    agg_i = a != agg_j -- the counts the library's split balances."""
    rows = np.repeat(np.arange(lv.n), np.diff(lv.row_ptr))
    a, b = lv.agg[rows], lv.agg[lv.col]
    return np.bincount(a[a != b], minlength=int(lv.agg.max()) + 1)


@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_setup_split_rule(P):
    """lap_setup_split: a partition of the output rows into P contiguous ranges
    with nearly equal term counts (each range's terms within one row's terms of
    total / P), and bit-equal to the rule written out here."""
    L = _lib()
    import oracle
    for g in [lapgen.rmat(12), lapgen.barabasi_albert(3000, 6), lapgen.grid2d(60, 50)]:
        ho = oracle.Hierarchy(g)
        lv = next(ho.level(l) for l in range(ho.nlev) if ho.level(l).kind == oracle.AGG)
        t = _galerkin_row_terms(lv)
        cum = np.concatenate([[0], np.cumsum(t)])
        b = L.setup_split(cum, P)
        assert b[0] == 0 and b[-1] == len(t) and np.all(np.diff(b) >= 0)
        ref = [0] + [int(np.searchsorted(cum * P, r * cum[-1], side="left")) for r in range(1, P)] + [len(t)]
        assert list(b) == ref
        loads = cum[b[1:]] - cum[b[:-1]]
        assert loads.max() <= cum[-1] / P + t.max()
    with pytest.raises(L.LapError):
        L.setup_split(np.array([0, 5, 3]), 2)


def _split_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        L = _lib()
        g = lapgen.barabasi_albert(4000, 7)
        ho = oracle.Hierarchy(g)
        la = next(l for l in range(ho.nlev) if ho.level(l).kind == oracle.AGG)
        lv, co = ho.level(la), ho.level(la + 1)
        cum = np.concatenate([[0], np.cumsum(_galerkin_row_terms(lv))])
        b = L.setup_split(cum, world)
        lo, hi = int(b[rank]), int(b[rank + 1])
        # this rank's rows of R L P (stand-in for its device build): local row_ptr from 0
        rp = co.row_ptr[lo:hi + 1] - co.row_ptr[lo]
        col = co.col[co.row_ptr[lo]:co.row_ptr[hi]]
        w = co.w[co.row_ptr[lo]:co.row_ptr[hi]]
        # setup_gather: entry counts of every rank, offsets, one broadcast per root
        cnt = torch.zeros(world, dtype=torch.int64)
        dist.all_gather(list(cnt.chunk(world)), torch.tensor([len(col)], dtype=torch.int64))
        off = np.concatenate([[0], np.cumsum(cnt.numpy())])
        n_out, nnz = int(b[-1]), int(off[-1])
        row_ptr = torch.zeros(n_out + 1, dtype=torch.int64)
        col_all = torch.zeros(nnz, dtype=torch.int32)
        w_all = torch.zeros(nnz, dtype=torch.float64)
        for r in range(world):
            a0, a1 = int(b[r]), int(b[r + 1])
            seg = torch.from_numpy(rp[:-1].copy()) if r == rank else torch.zeros(a1 - a0, dtype=torch.int64)
            dist.broadcast(seg, src=r)
            row_ptr[a0:a1] = seg + int(off[r])           # shifted by the root's entry offset
            c = torch.from_numpy(col.copy()) if r == rank else torch.zeros(int(cnt[r]), dtype=torch.int32)
            v = torch.from_numpy(w.copy()) if r == rank else torch.zeros(int(cnt[r]), dtype=torch.float64)
            dist.broadcast(c, src=r)
            dist.broadcast(v, src=r)
            col_all[int(off[r]):int(off[r + 1])] = c
            w_all[int(off[r]):int(off[r + 1])] = v
        row_ptr[n_out] = nnz
        ok = (np.array_equal(row_ptr.numpy(), co.row_ptr) and np.array_equal(col_all.numpy(), co.col)
              and w_all.numpy().tobytes() == co.w.tobytes())
        q.put((rank, bool(ok), hi - lo))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_setup_split_gather_gloo(world):
    """N1 host logic with torch.distributed 'gloo' (world 2 and 4): every rank
    takes its row range from lap_setup_split, contributes those rows of the
    coarse operator with a local row_ptr, and the gather of dist.cu
    setup_gather (entry counts all-gathered, one broadcast per root, row_ptr
    pieces shifted by the root's entry offset) rebuilds the whole operator
    bit for bit on every rank."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    assert sum(nr for _, _, nr in res) > 0


def _vote_worker(rank, world, port, q):
    """One setup rank of the row-split vote rounds (setup.cu aggregate_attempt
    under a setup communicator): its rows of each synchronous round
    (Alg. 3) from the replicated round-start state, the new states
    shared by one broadcast per root (dist.cu setup_share), the votes summed
    over the ranks (K4; dist.cu setup_sum_i32)."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        L = _lib()
        res = []
        for g in [lapgen.barabasi_albert(3000, 6), lapgen.rmat(11), lapgen.grid2d(40, 30)]:
            n, rp, col = g.n, g.row_ptr, g.col
            d = oracle.row_sums(n, rp, g.w)
            X = oracle.test_vectors(n, rp, col, g.w, d, seed=0, level=0)
            S = oracle.normalize_strength(n, rp, col, oracle.affinity(n, rp, col, X))
            agg_ref, m_ref, st_ref, votes_ref = oracle.aggregate(n, rp, col, S)
            b = L.setup_split(rp, world)          # rows in ranges of equal entry counts
            lo, hi = int(b[rank]), int(b[rank + 1])
            DEC, UND, SEED = 0, 1, 2
            st = np.full(n, UND, np.int8)
            idx = np.arange(n, dtype=np.int32)
            votes = torch.zeros(n, dtype=torch.int32)
            vloc = torch.zeros(n, dtype=torch.int32)
            for t in range(1, 11):
                filt = 2.0 ** -t
                nst, nidx = st.copy(), idx.copy()
                for i in range(lo, hi):
                    if st[i] != UND:
                        continue
                    best = None
                    for k in range(rp[i], rp[i + 1]):
                        j, s = int(col[k]), S[k]
                        if s == 0.0 or s < filt or st[j] == DEC:
                            continue
                        key = (int(st[j]), s, -j)
                        if best is None or key > best:
                            best = key
                    if best is None:
                        continue
                    if best[0] == SEED:
                        nst[i], nidx[i] = DEC, -best[2]
                    else:
                        vloc[-best[2]] += 1
                ts, ti = torch.from_numpy(nst), torch.from_numpy(nidx)
                for r in range(world):                # setup_share: one broadcast per root
                    a0, a1 = int(b[r]), int(b[r + 1])
                    for buf in (ts, ti):
                        seg = buf[a0:a1].clone()
                        dist.broadcast(seg, src=r)
                        buf[a0:a1] = seg
                dist.all_reduce(votes.copy_(vloc), op=dist.ReduceOp.SUM)   # setup_sum_i32
                st, idx = ts.numpy().copy(), ti.numpy().copy()
                st[(st == UND) & (votes.numpy() >= 8)] = SEED              # the promotion of k_vote_commit
            root = st != DEC
            rid = np.cumsum(root) - 1
            agg = np.where(root, rid, rid[idx]).astype(np.int32)
            res.append(bool(np.array_equal(agg, agg_ref) and np.array_equal(st, st_ref)
                            and np.array_equal(votes.numpy(), votes_ref) and int(root.sum()) == m_ref))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_split_voting_gloo(world):
    """N1 row-split vote rounds with torch.distributed 'gloo' (world 2 and 3):
    each rank runs Alg. 3's synchronous rounds on its lap_setup_split row range
    (split by entries, cum = row_ptr) against the replicated round-start
    states, the new states are shared by one broadcast per root and the votes
    summed over the ranks; the aggregates, final states and vote counts equal
    the oracle's whole-graph aggregation on every rank."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_vote_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(all(ok) for _, ok in res), res
