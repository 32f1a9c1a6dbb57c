"""Oracle whole sort and partition level, pinned by numpy's sort (the plain definition of
the final array: the input permuted into nondecreasing ordering-key order) and by
brute force on tiny inputs (all bucket assignments enumerated)."""
import itertools

import numpy as np
import pytest

import oracle
from paper_2208_06902_b200 import datagen


def ref_sorted(a):
    ok = oracle.ordering_keys(a)
    return a[np.argsort(ok, kind="stable")]


@pytest.mark.parametrize("kind", datagen.FUZZ_KINDS)
@pytest.mark.parametrize("n,k,B", [(0, 256, 4096), (1, 256, 4096), (2, 4, 1), (37, 4, 3),
                                   (1000, 16, 10), (20000, 256, 64), (70000, 1024, 4096)])
def test_sort_matches_numpy(kind, n, k, B):
    rng = np.random.default_rng(hash((kind, n, k)) & 0xFFFF)
    a = datagen.fuzz_array(rng, n, kind)
    want = ref_sorted(a)
    r = oracle.sort(a, k=k, base_case=B)
    assert r.status == 0
    assert a.tobytes() == want.tobytes()


def test_nan_rejected_unmodified():
    a = np.array([3.0, 1.0, np.nan, 2.0])
    before = a.copy()
    r = oracle.sort(a, k=4, base_case=1)
    assert r.status == 2
    assert a.tobytes() == before.tobytes()


def test_invalid_k():
    assert oracle.sort(np.zeros(10), k=2, base_case=1).status == 1


def test_all_permutations_n8():
    base = np.array([5.0, -1.0, 3.0, 3.0, 0.5, -0.0, 0.0, 9.0])
    want = ref_sorted(base).tobytes()
    for p in itertools.permutations(range(8)):
        a = base[list(p)].copy()
        assert oracle.sort(a, k=3, base_case=1).status == 0
        assert a.tobytes() == want


def test_all_binary_arrays_n12():
    """Every 0/1 array of length <= 12: exercises the equality split and homogeneity."""
    for n in range(13):
        for bits in range(1 << n):
            a = np.array([(bits >> i) & 1 for i in range(n)], dtype=np.float64)
            want = np.sort(a)
            assert oracle.sort(a, k=4, base_case=1).status == 0
            assert np.array_equal(a, want)


@pytest.mark.parametrize("trial", range(200))
def test_partition_brute_force(trial):
    """n <= 64: out is the unique stable order: bucket_i < bucket_j => pos_i < pos_j, and
    equal buckets keep input order; offsets are the bucket histogram's prefix sums."""
    rng = np.random.default_rng(trial)
    n = int(rng.integers(0, 65))
    k = int(rng.choice([3, 4, 16, 64]))
    a = rng.normal(0, 1, n)
    A, B = float(rng.uniform(0.5, 20)), float(rng.uniform(-10, 10))
    out, off, ids = oracle.partition(a, A, B, k)
    pos = sorted(range(n), key=lambda i: (ids[i], i))
    assert out.tolist() == [a[i] for i in pos]
    assert np.array_equal(np.diff(off), np.bincount(ids, minlength=k)) if n else True
    for i in range(n):
        assert ids[i] == oracle.bucket(float(a[i]), A, B, k)


def test_level_structure_on_c1_sized_uniform():
    a = datagen.generate("C1", 200_000)
    r = oracle.sort(a, k=256, base_case=4096, trace=True, snapshots=True)
    assert r.status == 0
    # every partitioned segment's children cover it exactly and are range-ordered
    for rec in r.records:
        assert int(rec.counts.sum()) == rec.m
        assert rec.S == oracle.sample_size(rec.m, 256)
    # snapshot after each level is a permutation of the input
    for snap in r.snapshots:
        assert np.array_equal(np.sort(snap.view(np.float64)), a)


def test_c1_full_size_equals_numpy():
    a = datagen.generate("C1")
    want = np.sort(a)
    assert oracle.sort(a, k=256, base_case=4096).status == 0
    assert a.tobytes() == want.tobytes()


@pytest.mark.parametrize("name", list(datagen.PAPER_WORKLOADS))
def test_paper_workloads_match_numpy(name):
    """The paper's nine synthetic workloads through the oracle, k = 1024 and 256."""
    for n, k in [(60_000, 1024), (30_000, 256)]:
        a = datagen.paper_workload(name, n)
        want = ref_sorted(a)
        assert oracle.sort(a, k=k, base_case=4096).status == 0
        assert a.tobytes() == want.tobytes()


@pytest.mark.parametrize("kind", datagen.STRESS_KINDS)
def test_stress_arrays_match_numpy(kind):
    a = datagen.stress_array(np.random.default_rng(3), 50_000, kind)
    want = ref_sorted(a)
    assert oracle.sort(a, k=256, base_case=4096).status == 0
    assert a.tobytes() == want.tobytes()
