"""Write tests/golden/streams.json: golden values of the method's counter-based
random streams, computed here in pure Python integers straight from the
definitions of SURVEY.md §8(c) O-S11 (SplitMix64 output function, salts,
U(l,i,k)) and O-S6 / DESIGN.md reading R-U' (the Lanczos start vector).
Independent of oracle/ (C) and of liblap (CUDA): neither is imported here.
The SplitMix64 function itself is checked against its published output
sequence (tests/golden/canonical.json) by tests/test_golden_streams.py.

    python tools/golden_streams.py
"""
import json
import os

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


def mix64(z):
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def salt(seed, k):
    return mix64(seed ^ ((k * GAMMA) & M64))


def u01(u):
    return float(u >> 11) * 2.0 ** -53  # exact: a 53-bit integer times a power of two


def lanczos_start(seed, level, n):
    base = mix64(salt(seed, 4) ^ (2 * level))
    return [2.0 * u01(mix64(base ^ i)) - 1.0 for i in range(n)]  # 2u - 1 is exact for u in [0,1) on 2^-53 grid


def x0_row(seed, level, attempt, i):
    base = mix64(salt(seed, 3) ^ (2 * level + attempt))
    return [2.0 * u01(mix64(base ^ (4 * i + k))) - 1.0 for k in range(4)]


def main():
    out = {
        "_source": "Pure-Python evaluation of SURVEY.md O-S11 / O-S6 definitions by tools/golden_streams.py "
                   "(no oracle, no liblap). lanczos_start: v_i = 2 u01(mix64(mix64(salt_4 ^ 2l) ^ i)) - 1 "
                   "(DESIGN.md reading R-U'); x0_rows: X0[i,k] = 2 u01(mix64(mix64(salt_3 ^ (2l+attempt)) ^ (4i+k))) - 1.",
        "lanczos_start": {f"seed{s}_level{l}": lanczos_start(s, l, 8) for s in (0, 7) for l in (0, 1, 3)},
        "x0_rows": {f"seed0_level{l}_attempt{a}_row{i}": x0_row(0, l, a, i)
                    for (l, a, i) in [(0, 0, 0), (0, 0, 5), (1, 0, 0), (2, 1, 3)]},
        "elim_hash_seed0": [hex(mix64(j ^ salt(0, 2))) for j in range(8)],
    }
    fn = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "streams.json")
    with open(fn, "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")
    print("wrote", fn)


if __name__ == "__main__":
    main()
