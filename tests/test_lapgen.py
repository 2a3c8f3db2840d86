"""The C/OpenMP R-MAT pipeline used for cfg 5 (scale 26) produces exactly the
graph of the numpy/scipy post-processing of the same edge stream."""
import numpy as np
import pytest

import lapgen


@pytest.mark.parametrize("scale", [8, 11, 14])
def test_rmat_large_matches_reference_pipeline(scale):
    g = lapgen.rmat_large(scale, 16)
    r = lapgen.rmat_large_reference(scale, 16)
    assert g.n == r.n and g.nnz == r.nnz
    assert np.array_equal(g.row_ptr, r.row_ptr)
    assert np.array_equal(g.col, r.col)
    assert g.w is None and np.all(r.w == 1.0)
