"""Hierarchy interchange format: the oracle exports, liblap's
lap_import_hierarchy reads (GPU), and the GPU solve on the oracle-built
hierarchy matches the oracle's solve."""
import json
import os

import numpy as np
import pytest

import lapgen
import oracle


def test_oracle_export_layout(tmp_path):
    g = lapgen.rmat(10)
    ho = oracle.Hierarchy(g)
    ho.export(str(tmp_path))
    meta = json.load(open(tmp_path / "meta.json"))
    assert meta["format"] == "lap-hierarchy-v1" and meta["nlev"] == ho.nlev and meta["n0"] == g.n
    assert np.array_equal(np.fromfile(tmp_path / "perm.i64", "<i8"), ho.perm())
    for l in range(ho.nlev):
        L = ho.level(l)
        d = tmp_path / f"L{l}"
        lm = json.load(open(d / "meta.json"))
        assert (lm["kind"], lm["n"], lm["nnz"]) == (L.kind, L.n, L.nnz)
        assert np.array_equal(np.fromfile(d / "row_ptr.i64", "<i8"), L.row_ptr)
        assert np.fromfile(d / "w.f64", "<f8").tobytes() == L.w.tobytes()
        if L.kind == oracle.AGG:
            assert lm["lambda"] == L.lam and np.array_equal(np.fromfile(d / "agg.i32", "<i4"), L.agg)
        if L.kind == oracle.ELIM:
            assert np.array_equal(np.fromfile(d / "fmap.i32", "<i4"), L.fmap)
        if L.kind == oracle.COARSEST:
            assert np.fromfile(d / "coarse_pinv.f64", "<f8").tobytes() == L.pinv.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("mk", [lambda: lapgen.grid2d(64, 64), lambda: lapgen.rmat(12),
                                lambda: lapgen.barabasi_albert(5000, 8), lambda: lapgen.path(3000)],
                         ids=["cfg1", "rmat12", "ba5000", "path3000"])
def test_import_oracle_hierarchy_solves_like_oracle(tmp_path, mk):
    import paper_1705_06266_b200 as P
    g = mk()
    ho = oracle.Hierarchy(g)
    ho.export(str(tmp_path))
    hi = P.Hierarchy.import_dir(str(tmp_path))
    hb = P.Hierarchy(g)
    assert hi.nlev == ho.nlev
    for l in range(ho.nlev):
        a, o = hi.level(l), ho.level(l)
        assert a["kind"] == o.kind and a["col"].tobytes() == o.col.tobytes() and a["w"].tobytes() == o.w.tobytes()
    b = lapgen.rhs(g.n, seed=2)
    x, it, rr, rc = hi.solve(b)
    xo, ito, rro, rco = ho.solve(b)
    assert rc == 0 and rr <= 1e-8 and abs(it - ito) <= 1, (it, ito, rr)
    assert np.abs(x - xo).max() <= 1e-6 * np.abs(xo).max()
    # the GPU's own setup builds the same operators and maps; only the coarsest
    # L^+ differs in rounding (the oracle grounds + Cholesky, the GPU Gauss-Jordan)
    xb, itb, _, _ = hb.solve(b)
    assert abs(itb - it) <= 1 and np.abs(xb - x).max() <= 1e-9 * np.abs(x).max()


@pytest.mark.gpu
def test_import_rejects_bad_directories(tmp_path):
    import paper_1705_06266_b200 as P
    with pytest.raises(P.LapError) as e:
        P.Hierarchy.import_dir(str(tmp_path / "missing"))
    assert e.value.code == P.LAP_EINVAL
    g = lapgen.rmat(9)
    oracle.Hierarchy(g).export(str(tmp_path / "h"))
    fn = tmp_path / "h" / "L0" / "col.i32"
    data = open(fn, "rb").read()
    open(fn, "wb").write(data[:-4])  # truncated
    with pytest.raises(P.LapError) as e:
        P.Hierarchy.import_dir(str(tmp_path / "h"))
    assert e.value.code == P.LAP_EINVAL
