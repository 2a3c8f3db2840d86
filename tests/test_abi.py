"""C-ABI checks that need no GPU: liblap.so loads, exports every function
include/lap.h declares (and the binding's EXPORTS list matches the header),
the parameter defaults are the paper's values, and struct layouts agree
between the header and the ctypes binding."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "lap.h")


def header_functions():
    src = open(HDR).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(lap_[a-z0-9_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def P():
    from paper_1705_06266_b200 import build
    build.build()
    import paper_1705_06266_b200 as P
    return P


def test_header_declares_the_boundary():
    names = header_functions()
    for must in ["lap_setup", "lap_solve", "lap_free", "lap_spmv", "lap_vcycle", "lap_params_default",
                 "lap_last_error"]:
        assert must in names, must


def test_library_exports_every_header_symbol(P):
    lib = P.lib()
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # dynamic symbol table agrees (extern "C": unmangled names)
    out = subprocess.run(["nm", "-D", "--defined-only", P.lap.LIB_PATH], capture_output=True, text=True).stdout
    syms = {l.split()[-1] for l in out.splitlines() if l.strip()}
    assert set(header_functions()) <= syms
    assert sorted(P.EXPORTS) == header_functions()


def test_params_default_are_the_papers(P):
    p = P.lap_params_default()
    assert p.tol == 1e-8
    assert p.cheby_degree == 2
    assert (p.cheby_lo, p.cheby_hi) == (0.3, 1.1)
    assert p.lanczos_steps == 10
    assert p.elim_max_degree == 4
    assert p.n_test_vectors == 4 and p.tv_sweeps == 3
    assert p.tv_omega == 2.0 / 3.0            # O-R6
    assert p.vote_rounds == 10 and p.vote_threshold == 8
    assert p.coarse_nnz == 1000
    assert p.max_levels == 40 and p.max_iters == 500
    assert p.random_order == 1 and p.affinity_power == 1


def test_struct_layouts_match_header(P):
    # sizes from the C compiler on the header vs the ctypes mirrors
    code = ('#include "lap.h"\n#include <stdio.h>\n#include <stddef.h>\n'
            'int main(){printf("%zu %zu %zu\\n", sizeof(lap_graph), sizeof(lap_params), sizeof(lap_stats));}\n')
    tmp = os.path.join(ROOT, "paper_1705_06266_b200", "_build")
    os.makedirs(tmp, exist_ok=True)
    c = os.path.join(tmp, "sz.c")
    exe = os.path.join(tmp, f"sz{os.getpid()}")
    open(c, "w").write(code)
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
    g, p, s = map(int, subprocess.check_output([exe]).split())
    os.remove(exe)
    assert g == ctypes.sizeof(P.lap.lap_graph)
    assert p == ctypes.sizeof(P.lap.lap_params)
    assert s == ctypes.sizeof(P.lap.lap_stats)


def test_errors_without_gpu_are_statuses_not_crashes(P):
    """On a machine with no GPU, lap_setup must return an error status (no
    exception across the ABI, no CPU fallback)."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    import numpy as np
    import lapgen
    g = lapgen.path(5)
    with pytest.raises(P.LapError) as e:
        P.Hierarchy(g)
    assert e.value.code in (P.LAP_EINVAL, 5)  # LAP_ECUDA
