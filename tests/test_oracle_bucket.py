"""Oracle bucket function F(x) = clamp(floor(a x + b), 0, k-1), pinned by
exact rationals: mul rounded once, then add rounded once (R7), never one fused FMA."""
from fractions import Fraction
import math
import struct

import numpy as np
import pytest

import oracle


def rn(q: Fraction) -> float:
    """Correctly rounded binary64 of an exact rational (Fraction -> float is RN-even)."""
    return float(q)


def bucket_exact(a, b, x, k, fused=False):
    if fused:
        y = rn(Fraction(a) * Fraction(x) + Fraction(b))
    else:
        y = rn(Fraction(rn(Fraction(a) * Fraction(x))) + Fraction(b))
    if not (y >= 0):
        return 0
    if y >= k:
        return k - 1
    return math.floor(y)


def test_fma_vectors(golden):
    rows = golden("fma_vectors.txt")
    vecs = [[k_] + r for k_, rs in rows.items() for r in rs]
    assert len(vecs) == 3
    for a, b, x, k in vecs:
        a, b, x, k = float(a), float(b), float(x), int(k)
        two = bucket_exact(a, b, x, k)
        fused = bucket_exact(a, b, x, k, fused=True)
        assert two != fused, "vector must separate mul+add from FMA"
        assert oracle.bucket(x, a, b, k) == two


@pytest.mark.parametrize("trial", range(30))
def test_random_exact_rational(trial):
    rng = np.random.default_rng(trial)
    k = int(rng.choice([4, 256, 1024]))
    a = float(rng.uniform(0.1, 2000.0))
    b = float(rng.uniform(-500, 500))
    for x in rng.normal(0, 1, 200):
        assert oracle.bucket(float(x), a, b, k) == bucket_exact(a, b, float(x), k)


def test_floor_toward_minus_infinity_and_clamps():
    # y in (-1, 0) must clamp to 0 (floor(-0.5) = -1 < 0), never truncate to 0 by accident
    assert oracle.bucket(-0.5, 1.0, 0.0, 8) == 0
    assert oracle.bucket(7.999, 1.0, 0.0, 8) == 7
    assert oracle.bucket(8.0, 1.0, 0.0, 8) == 7
    assert oracle.bucket(1e308, 1.0, 0.0, 8) == 7
    assert oracle.bucket(float("inf"), 1.0, 0.0, 8) == 7
    assert oracle.bucket(float("-inf"), 1.0, 0.0, 8) == 0
    assert oracle.bucket(2.0, 1.0, 0.5, 8) == 2  # floor(2.5)


def test_u64_model_domain_is_rn_conversion():
    # 2^53 + 1 converts (RN-even) to 2^53: same bucket as 2^53
    x = (1 << 53) + 1
    a = 2.0 ** -50
    assert oracle.bucket(np.uint64(x), a, 0.0, 16) == oracle.bucket(np.uint64(1 << 53), a, 0.0, 16)
    assert float(np.uint64(x)) == 2.0 ** 53


def test_eq3():
    piv = oracle.ordering_key(struct.unpack("<Q", struct.pack("<d", 1.5))[0], oracle.KEY_F64)
    for x, want in [(1.0, 0), (1.5, 1), (2.0, 2), (-0.0, 0)]:
        assert oracle.bucket(x, 0, 0, 3, kind=oracle.MODEL_EQ3, pivot_ok=piv) == want


def test_ordering_key_order():
    rng = np.random.default_rng(1)
    v = np.concatenate([rng.normal(0, 1e3, 5000), [-0.0, 0.0, np.inf, -np.inf, 5e-324, -5e-324]])
    ok = oracle.ordering_keys(v)
    order = np.argsort(ok, kind="stable")
    s = v[order]
    assert np.all(s[:-1] <= s[1:])
    # -0.0 sorts before +0.0
    z = np.where(s == 0)[0]
    assert np.signbit(s[z[0]]) and not np.signbit(s[z[-1]])
    assert oracle.ordering_key(0, oracle.KEY_F64) == 0x8000000000000000  # +0.0
