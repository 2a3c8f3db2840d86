"""Golden values of the method's counter-based streams (SURVEY.md §8(c) O-S11,
O-P17): the oracle and, through the C ABI, liblap must reproduce them.

Sources (none is the oracle or liblap):
  * tests/golden/canonical.json "survey_o_s11": the values SURVEY O-S11 lists
    (mix64(1), salts, h(0..3), Pi_rand for n = 8, X0 row 0 of level 0);
  * tests/golden/canonical.json "splitmix64_seed0_outputs": the published
    SplitMix64 output sequence (pins the pure-Python mix64 below);
  * tests/golden/streams.json: written by tools/golden_streams.py in pure
    Python integers from the O-S11 / O-S6 definitions (Lanczos start vector,
    reading R-U' of DESIGN.md; more X0 rows; h(0..7)).
A slip in an index (4i+k vs i+4k), a salt (salt_3 vs salt_4) or a counter
composition (2l + attempt) changes every value and fails these tests.
"""
import json
import os
import sys

import numpy as np
import pytest

import lapgen
import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import golden_streams as GS  # noqa: E402  (pure Python; imports neither oracle nor liblap)

CAN = json.load(open(os.path.join(GOLD, "canonical.json")))
SURV = CAN["survey_o_s11"]
STR = json.load(open(os.path.join(GOLD, "streams.json")))


def test_pure_python_mix64_matches_published_splitmix64():
    outs = [int(h, 16) for h in CAN["splitmix64_seed0_outputs"]]
    for k, want in enumerate(outs, start=1):
        assert GS.mix64(k * GS.GAMMA) == want
    assert GS.mix64(0) == 0


def test_pure_python_generator_reproduces_survey_goldens():
    # the generator of streams.json agrees with SURVEY's independently computed values
    assert GS.mix64(1) == int(SURV["mix64_of_1"], 16)
    assert [hex(GS.mix64(j ^ GS.salt(0, 2))) for j in range(4)] == [hex(int(h, 16)) for h in SURV["h_0_to_3_seed0"]]
    assert GS.x0_row(0, 0, 0, 0) == SURV["x0_level0_attempt0_row0"]


def test_oracle_mix64_and_salts_match_survey():
    assert oracle.mix64(0) == 0
    assert oracle.mix64(1) == int(SURV["mix64_of_1"], 16)
    assert oracle.mix64(0x9E3779B97F4A7C15) == int(SURV["mix64_of_gamma"], 16)
    for k, h in enumerate(SURV["salts_seed0"], start=1):
        assert oracle.salt(0, k) == int(h, 16)


def test_oracle_elim_hash_matches_survey_h():
    for j, h in enumerate(SURV["h_0_to_3_seed0"]):
        assert oracle.elim_hash(j, 0) == int(h, 16)
    assert [hex(oracle.elim_hash(j, 0)) for j in range(8)] == STR["elim_hash_seed0"]


def test_oracle_elim_select_uses_h():
    # a path 0-1-2-3-4: all candidates; F = the strict local minima of (h(j), j) over closed neighbourhoods
    g = lapgen.path(5)
    F, nF = oracle.elim_select(g.n, g.row_ptr, g.col, 4, 0)
    h = [int(x, 16) for x in STR["elim_hash_seed0"]]
    want = []
    for i in range(5):
        nb = [j for j in (i - 1, i, i + 1) if 0 <= j < 5]
        want.append(min(nb, key=lambda j: (h[j], j)) == i)
    assert F.tolist() == want


def test_oracle_pi_rand_n8_matches_survey():
    assert oracle.random_perm(8, 0).tolist() == SURV["pi_rand_n8_seed0"]


def test_oracle_x0_rows_match_goldens():
    g = lapgen.path(8)
    X = oracle.test_vectors(g.n, g.row_ptr, g.col, g.w, oracle.row_sums(g.n, g.row_ptr, g.w), seed=0, level=0,
                            attempt=0, sweeps=0)
    assert X[0].tolist() == SURV["x0_level0_attempt0_row0"]
    for key, row in STR["x0_rows"].items():
        l = int(key.split("_level")[1].split("_")[0])
        a = int(key.split("_attempt")[1].split("_")[0])
        i = int(key.split("_row")[1])
        Xl = oracle.test_vectors(g.n, g.row_ptr, g.col, g.w, oracle.row_sums(g.n, g.row_ptr, g.w), seed=0, level=l,
                                 attempt=a, sweeps=0)
        assert Xl[i].tolist() == row, key


def test_oracle_lanczos_start_matches_goldens():
    for key, vals in STR["lanczos_start"].items():
        seed = int(key.split("seed")[1].split("_")[0])
        level = int(key.split("level")[1])
        assert oracle.lanczos_start(8, seed, level).tolist() == vals, key


# ------------------------------------------------------------------ C ABI (GPU)

@pytest.mark.gpu
def test_liblap_streams_match_goldens():
    import paper_1705_06266_b200 as P
    assert P.random_stream(3, 2)[1] == np.uint64(int(SURV["mix64_of_1"], 16))
    h = P.random_stream(0, 8, seed=0)
    assert [hex(int(x)) for x in h] == STR["elim_hash_seed0"]
    X = P.random_stream(1, 8, seed=0, level=0, attempt=0)
    assert X[0].tolist() == SURV["x0_level0_attempt0_row0"]
    for key, row in STR["x0_rows"].items():
        l = int(key.split("_level")[1].split("_")[0])
        a = int(key.split("_attempt")[1].split("_")[0])
        i = int(key.split("_row")[1])
        assert P.random_stream(1, 8, seed=0, level=l, attempt=a)[i].tolist() == row, key
    for key, vals in STR["lanczos_start"].items():
        seed = int(key.split("seed")[1].split("_")[0])
        level = int(key.split("level")[1])
        assert P.random_stream(2, 8, seed=seed, level=level).tolist() == vals, key


@pytest.mark.gpu
def test_liblap_pi_rand_n8_matches_survey():
    import paper_1705_06266_b200 as P
    h = P.Hierarchy(lapgen.path(8))
    assert h.perm().tolist() == SURV["pi_rand_n8_seed0"]
