"""Work / WDA accounting of the benchmark (SPEC examples S:584-586)."""
import math

import pytest

from paper_1705_06266_b200 import metrics as MX


def test_wda_spec_examples():
    assert MX.wda(80.0, 1e-8) == pytest.approx(10.0)
    assert MX.wda(3.0, 0.1) == pytest.approx(3.0)
    with pytest.raises(ValueError):
        MX.wda(5.0, 1.0)
    assert MX.tda(2.0, 1e-4) == pytest.approx(0.5)


def test_vcycle_work_by_hand():
    # aggregation level n=100, nnz_off=400 (nnz(L)=500) -> coarse 10 (nnz_off 30) -> coarsest
    levels = [dict(kind=0, n=100, nnz=400, m=10), dict(kind=2, n=10, nnz=30)]
    # 2K SpMV applications (K=2: 1 pre + resid + 2 post) of nnz(L0)=500 -> 4 units;
    # step 0: n/500 = 0.2; R and P: 2*(100+10)/500 = 0.44; coarsest 10^2/500 = 0.2
    assert MX.vcycle_work(levels) == pytest.approx(4 + 0.2 + 0.44 + 0.2)


def test_elimination_and_solve_work():
    levels = [dict(kind=1, n=50, nnz=100, nnz_fc=20), dict(kind=2, n=30, nnz=80)]
    nnz0 = 150
    vw = 2 * (50 + 20) / nnz0 + 30 ** 2 / nnz0
    assert MX.vcycle_work(levels) == pytest.approx(vw)
    # 3 iterations, 4 V-cycles, 8 vector ops per iteration, + final residual
    assert MX.solve_work(levels, 3, 4) == pytest.approx(3 * (1 + 8 * 50 / nnz0) + 4 * vw + 1)
    assert math.isfinite(MX.wda(MX.solve_work(levels, 3, 4), 1e-9))
