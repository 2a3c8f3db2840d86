"""paper_1705_06266_b200 -- B200-native (sm_100a) hot path of the
unsmoothed-aggregation multigrid solver for graph Laplacians (Konolige &
Brown, arXiv 1705.06266): GPU hierarchy setup (elimination, strength, vote
aggregation, Galerkin) and PCG + V-cycle solve, behind the C ABI of
include/lap.h (liblap.so).  This package is only the ctypes binding.
"""
from .lap import (Hierarchy, Comm, dist_index, setup_split, LapError, lap_params_default, lib, load, EXPORTS,  # noqa: F401
                  random_stream, pool_retain, bench_gather,
                  KIND_AGG, KIND_ELIM, KIND_COARSEST, LAP_OK, LAP_ENOCONV, LAP_ESTALL, LAP_EGRAPH,
                  LAP_EDISCONNECTED, LAP_EINVAL)
