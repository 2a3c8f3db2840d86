"""Pins for the oracle's canonical arithmetic (SURVEY O-S11, O-P17, O-P3)."""
import json
import os
import random
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_mix64_matches_splitmix64_reference_sequence():
    g = json.load(open(os.path.join(GOLD, "canonical.json")))
    outs = [int(h, 16) for h in g["splitmix64_seed0_outputs"]]
    # SplitMix64 from state 0: k-th output = mix64(k * golden); salt_k is that output
    for k, want in enumerate(outs, start=1):
        assert oracle.mix64((k * 0x9E3779B97F4A7C15) & (2**64 - 1)) == want
        assert oracle.salt(0, k) == want
    assert oracle.mix64(0) == int(g["mix64_of_zero"], 16)


def test_mix64_is_a_bijection_roundtrip():
    rng = random.Random(1)
    for _ in range(20000):
        z = rng.getrandbits(64)
        assert oracle.mix64_inverse(oracle.mix64(z)) == z
        assert oracle.mix64(oracle.mix64_inverse(z)) == z


def test_random_perm_is_bijection_and_sorts_hash():
    for n in [1, 2, 8, 1000]:
        p = oracle.random_perm(n, 0)
        assert sorted(p.tolist()) == list(range(n))
        # rank order follows the (bijective) hash of i ^ salt_1: strictly increasing along the order
        inv = np.argsort(p)
        s1 = oracle.salt(0, 1)
        keys = [oracle.mix64(int(i) ^ s1) for i in inv]
        assert all(keys[k] < keys[k + 1] for k in range(n - 1))
    assert not np.array_equal(oracle.random_perm(1000, 0), oracle.random_perm(1000, 1))


def _exact(ts):
    return sum((Fraction(t) for t in ts), Fraction(0))


def _ulp(x):
    return np.spacing(abs(x)) if x != 0 else np.spacing(0.0)


@pytest.mark.parametrize("seed", range(60))
def test_canon_sum_error_bound_and_order_invariance(seed):
    """|CanonSum - exact| <= 1/2 ulp(result) + cnt * 2^(E_lo - 1)  (O-S11),
    and the result is identical under any permutation of the terms."""
    rng = np.random.default_rng(seed)
    cnt = int(rng.integers(1, 3000))
    mag = 10.0 ** rng.uniform(-9, 0, cnt)
    t = mag * rng.choice([-1.0, 1.0], cnt) * rng.uniform(0.5, 1.0, cnt)
    if seed % 3 == 0:  # heavy cancellation
        t = np.concatenate([t, -t[: cnt // 2] * (1 + 1e-15)])
    e_max = oracle.ilogb(np.abs(t).max()) + 1
    K = int(rng.integers(len(t), 2**31))
    s = oracle.canon_sum(t, e_max, K)
    ex = _exact(t)
    elo = oracle.canon_elo(e_max, K)
    bound = Fraction(_ulp(s)) / 2 + len(t) * Fraction(2) ** (elo - 1)
    assert abs(Fraction(s) - ex) <= bound
    for _ in range(3):
        perm = rng.permutation(len(t))
        assert oracle.canon_sum(t[perm], e_max, K) == s


def test_canon_sum_is_correctly_rounded_when_terms_on_grid():
    """If every term is a multiple of 2^E_lo the integer sum is exact and the
    result must equal the correctly rounded exact sum (Python Fraction->float
    rounds correctly)."""
    rng = np.random.default_rng(7)
    for _ in range(200):
        cnt = int(rng.integers(1, 500))
        t = rng.uniform(-1, 1, cnt) * 2.0 ** rng.integers(-30, 0, cnt)
        e_max = 1
        K = 1000
        s = oracle.canon_sum(t, e_max, K)
        assert s == float(_exact(t))
    # exact cancellation to zero and single terms
    assert oracle.canon_sum([1.0, -1.0], 1, 2) == 0.0
    assert oracle.canon_sum([0.375], 1, 1) == 0.375
    assert oracle.canon_sum([], 1, 1) == 0.0


def test_canon_sum_halfway_rounding_to_even():
    # grid spacing 2^E_lo; terms below half a grid step vanish, exact half rounds to even
    e_max, K = 1, 1
    elo = oracle.canon_elo(e_max, K)  # 1 + 1 - 125 = -123
    assert elo == -123
    h = 2.0 ** (elo - 1)
    assert oracle.canon_sum([h], e_max, K) == 0.0            # 0.5 -> 0 (even)
    assert oracle.canon_sum([3 * h], e_max, K) == 2.0 ** (elo + 1)  # 1.5 -> 2
    assert oracle.canon_sum([h * 0.999], e_max, K) == 0.0
    # int128 -> double: ties at the 53-bit boundary round to even (O-S11)
    e_max, K = 60, 1
    elo = oracle.canon_elo(e_max, K)
    assert elo == -64
    g = 2.0 ** elo
    top = 2.0 ** (53 + elo)
    assert oracle.canon_sum([top, g], e_max, K) == top                # 2^53+1 -> 2^53
    assert oracle.canon_sum([top, 3 * g], e_max, K) == top + 4 * g   # 2^53+3 -> 2^53+4
    assert oracle.canon_sum([-top, -3 * g], e_max, K) == -(top + 4 * g)
    assert oracle.canon_sum([top, 2 * top - g], e_max, K) == float(_exact([top, 2 * top - g]))
