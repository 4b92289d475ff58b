"""CPU: the exact integer digit split that feeds the tensor-core Gram
(rsm_dev.cuh digits_i8 / k_gram_i8.cu), restated in Python integers: every
value |w| <= 1 is reproduced to 2^-(7+8(S-1)) by balanced base-256 digits that
fit int8, and products of split values carry only the stated truncation."""
import random

import pytest


def digits(x, S=6):
    """rsm_dev.cuh digits_i8<S>: Y = rint(x 2^(6+8(S-1))) + sum 128*256^s; bytes^0x80, top = Y >> 8(S-1)."""
    LB = 8 * (S - 1)
    C = int("80" * (S - 1), 16)
    Y = round(x * 2 ** (6 + LB)) + C
    z = ((Y ^ C) & ((1 << LB) - 1)) | (((Y >> LB) & 0xFF) << LB)
    a = []
    for s in range(S):
        byte = (z >> (8 * (S - 1 - s))) & 0xFF
        a.append(byte - 256 if byte >= 128 else byte)
    return a


@pytest.mark.parametrize("S", [5, 6, 7])
def test_digits_reconstruct_and_fit_int8(S):
    rng = random.Random(S)
    xs = [rng.uniform(-1, 1) for _ in range(20000)] + [1.0, -1.0, 0.0, 0.5, -0.5, 2 ** -40, -(2 ** -47), 0.99999999]
    for x in xs:
        a = digits(x, S)
        assert -64 <= a[0] <= 64 and all(-128 <= d <= 127 for d in a[1:])
        rec = sum(d * 2.0 ** (-6 - 8 * s) for s, d in enumerate(a))
        assert abs(rec - x) <= 2.0 ** (-7 - 8 * (S - 1)) * (1 + 1e-12)


def test_class_sums_reproduce_products():
    # k_gram_i8: w_i w_j ~= sum_{d<S} 2^(-12-8d) sum_{s+t=d} a_s(i) a_t(j); the
    # dropped classes bound the error by ~S 2^(2-8S)
    S = 6
    rng = random.Random(1)
    for _ in range(5000):
        x, y = rng.uniform(-1, 1), rng.uniform(-1, 1)
        a, b = digits(x, S), digits(y, S)
        approx = sum(2.0 ** (-12 - 8 * d) * sum(a[s] * b[d - s] for s in range(d + 1)) for d in range(S))
        assert abs(approx - x * y) <= S * 2.0 ** (2 - 8 * S)
