"""The oracle's OpenMP build gives bitwise the same hierarchy and solution
for any thread count: parallel loops are over independent
rows / entries / aggregates, integer counters are atomic, and every floating
sum has one fixed order (CanonSums are exact; dots are fixed 4096-chunk sums)."""
import numpy as np
import pytest

import lapgen
import oracle

_DEFAULT = oracle.get_threads()


def oracle_default_threads():
    return _DEFAULT


def _run(g, threads, **kw):
    oracle.set_threads(threads)
    try:
        h = oracle.Hierarchy(g, **kw)
        x, it, rr, rc = h.solve(lapgen.rhs(g.n, seed=1))
        return h, x, it, rr
    finally:
        oracle.set_threads(oracle_default_threads())


@pytest.mark.parametrize("mk", [lambda: lapgen.rmat(13), lambda: lapgen.barabasi_albert(20000, 8),
                                lambda: lapgen.grid3d(24), lambda: lapgen.star(9000)],
                         ids=["rmat13", "ba20000", "grid3d24", "star9000"])
def test_thread_count_does_not_change_results(mk):
    g = mk()
    h1, x1, i1, r1 = _run(g, 1)
    h4, x4, i4, r4 = _run(g, 5)
    assert h1.nlev == h4.nlev
    for l in range(h1.nlev):
        a, b = h1.level(l), h4.level(l)
        assert (a.kind, a.n, a.nnz) == (b.kind, b.n, b.nnz)
        for f in ("row_ptr", "col", "w", "d"):
            assert getattr(a, f).tobytes() == getattr(b, f).tobytes(), (l, f)
        if a.kind == oracle.AGG:
            assert a.agg.tobytes() == b.agg.tobytes() and a.S.tobytes() == b.S.tobytes()
            assert np.float64(a.lam).tobytes() == np.float64(b.lam).tobytes()
        if a.kind == oracle.ELIM:
            assert a.fmap.tobytes() == b.fmap.tobytes()
    assert i1 == i4 and x1.tobytes() == x4.tobytes() and r1 == r4
