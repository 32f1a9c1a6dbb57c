"""Sampling: sample size rule and stratified positions (R1, R2, R18, R19).
The sampled positions themselves are parity-unpinned against the paper (it shows no
sample); the generator is pinned to SplitMix64's published outputs and to structure."""
import numpy as np
import pytest

import oracle


def test_splitmix64_published_vector():
    # SplitMix64 (Steele, Lea, Flood 2014; Vigna's reference code), state seeded 1234567:
    # first outputs 6457827717110365317, 3203168211198807973, 9817491932198370423.
    g = 0x9E3779B97F4A7C15
    assert oracle.splitmix64(1234567) == 6457827717110365317
    assert oracle.splitmix64(1234567 + g) == 3203168211198807973
    assert oracle.splitmix64(1234567 + 2 * g) == 9817491932198370423
    assert oracle.splitmix64(0) == 0xE220A8397B1DCDAF


@pytest.mark.parametrize("m,k,S", [
    (2 ** 20, 256, 1023),           # SPEC.md S:237-240 example: alpha = ceil(20/5) = 4
    (1_000_000, 256, 1023),         # C1 level 0
    (100_000_000, 1024, 6143),      # C2-C4 level 0 (ceil(log2 1e8) = 27)
    (200_000_000, 1024, 6143),      # C5 level 0 (28)
    (5000, 1024, 2500),             # capped at floor(m/2)
    (2 ** 15, 1024, 3071),
    (2 ** 15 + 1, 1024, 4095),
    (20, 4, 4),                     # worked example: alpha k - 1 = 3 -> at least 4
    (7, 4, 3),                      # floor(7/2) = 3 < 4 -> the equality split (R19)
])
def test_sample_size(m, k, S):
    assert oracle.sample_size(m, k) == S


@pytest.mark.parametrize("trial", range(200))
def test_positions_one_per_stratum(trial):
    rng = np.random.default_rng(trial)
    m = int(rng.integers(8, 10 ** 7))
    k = int(rng.choice([4, 256, 1024]))
    S = oracle.sample_size(m, k)
    begin = int(rng.integers(0, 10 ** 9))
    level = int(rng.integers(0, 5))
    idx = oracle.sample_positions(0x49504C53, level, begin, m, S).astype(np.int64) - begin
    j = np.arange(S, dtype=np.int64)
    lo = (j * m) // S
    hi = ((j + 1) * m) // S
    assert np.all(idx >= lo) and np.all(idx < hi)
    assert np.all(np.diff(idx) > 0)
    # inverse map used to recognise a sample position from its offset r: j = ceil((r+1)S/m)-1
    assert np.all(-(-(idx + 1) * S // m) - 1 == j)


def test_positions_depend_on_seed_level_begin():
    a = oracle.sample_positions(1, 0, 0, 10 ** 6, 1023)
    assert not np.array_equal(a, oracle.sample_positions(2, 0, 0, 10 ** 6, 1023))
    assert not np.array_equal(a, oracle.sample_positions(1, 1, 0, 10 ** 6, 1023))
    b = oracle.sample_positions(1, 0, 5, 10 ** 6, 1023) - 5
    assert not np.array_equal(a, b)


def test_positions_roughly_uniform_within_strata():
    m, S = 10 ** 8, 6143
    idx = oracle.sample_positions(0x49504C53, 0, 0, m, S).astype(np.float64)
    j = np.arange(S)
    frac = (idx - (j * m) // S) / (m / S)
    assert 0.45 < frac.mean() < 0.55
    assert frac.min() >= 0 and frac.max() < 1
