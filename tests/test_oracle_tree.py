"""Oracle splitter-tree model (IPS4o's decision tree; SURVEY §8(f) NEXT #2;
DESIGN.md R22-R24), pinned against the paper's own description of the classifier:

* the implicit binary tree built by taking the middle splitter at every node (P:373-375,
  SPEC tree_build: candidates 1..7, depth 3 -> heap [4,2,6,1,3,5,7]) and descended with
  j <- 2j + (x > a_j) reaches the leaf the oracle returns (a count of the
  splitters strictly below the key) — written out here as the paper's loop;
* the splitters are equidistant order statistics of the sorted sample;
* the whole sort with the tree model equals numpy's sort, every level's layout is the stable
  counting partition by the tree bucket, and duplicates hit the no-progress guard.
"""
import numpy as np
import pytest

import oracle
from paper_2208_06902_b200 import datagen


def build_heap(spl):
    """middle element at each node, recursively; heap[1..] (1-based)."""
    heap = [None] * (len(spl) + 1)

    def rec(j, lo, hi):
        if lo > hi:
            return
        mid = (lo + hi) // 2
        heap[j] = spl[mid]
        rec(2 * j, lo, mid - 1)
        rec(2 * j + 1, mid + 1, hi)
    rec(1, 0, len(spl) - 1)
    return heap


def descend(heap, k, o):
    """j = 2j + (x > a_j), log2(k) steps from the root; leaf j - k."""
    j = 1
    for _ in range(k.bit_length() - 1):
        j = 2 * j + (1 if o > heap[j] else 0)
    return j - k


def test_heap_construction_spec_example():
    assert build_heap([1, 2, 3, 4, 5, 6, 7])[1:] == [4, 2, 6, 1, 3, 5, 7]


@pytest.mark.parametrize("k", [4, 8, 64, 256, 1024])
def test_descent_equals_oracle_bucket(k):
    rng = np.random.default_rng(k)
    for trial in range(20):
        S = int(rng.integers(k, 4 * k))
        smp = np.sort(rng.normal(0, 1, S) if trial % 2 else rng.integers(0, 50, S).astype(np.float64))
        spl = oracle.tree_splitters(smp, k)
        heap = build_heap([int(v) for v in spl])
        keys = np.concatenate([smp, rng.normal(0, 1.5, 200), [-0.0, 0.0, np.inf, -np.inf]])
        for x in keys:
            o = int(oracle.ordering_keys(np.array([x]))[0])
            assert oracle.tree_bucket(x, spl, k) == descend(heap, k, o)


def test_splitters_are_equidistant_order_statistics():
    for S, k in [(16, 4), (1023, 256), (4095, 1024), (6143, 1024), (100, 8)]:
        s = np.arange(S, dtype=np.float64)
        spl = oracle.tree_splitters(s, k)
        want = oracle.ordering_keys(np.array([float((i * S) // k) for i in range(1, k)]))
        assert np.array_equal(spl, want)


def test_ties_go_left_and_signed_zeros():
    spl = oracle.ordering_keys(np.array([-1.0, -0.0, 0.0, 2.0, 2.0, 2.0, 5.0]))
    assert oracle.tree_bucket(-1.0, spl, 8) == 0
    assert oracle.tree_bucket(-0.0, spl, 8) == 1
    assert oracle.tree_bucket(0.0, spl, 8) == 2
    assert oracle.tree_bucket(2.0, spl, 8) == 3
    assert oracle.tree_bucket(2.5, spl, 8) == 6
    assert oracle.tree_bucket(9.0, spl, 8) == 7


@pytest.mark.parametrize("kind", ["uniform", "normal", "lognormal", "few_distinct",
                                  "u64_above_2_53", "signed_zeros", "infs", "mixture"])
@pytest.mark.parametrize("n,k,B", [(5000, 16, 64), (70001, 256, 4096), (120000, 1024, 4096)])
def test_tree_sort_matches_numpy_and_stable_levels(kind, n, k, B):
    rng = np.random.default_rng(n + k + len(kind))
    a = datagen.fuzz_array(rng, n, kind)
    want = a[np.argsort(oracle.ordering_keys(a), kind="stable")]
    src = a.copy()
    r = oracle.sort(a, k=k, base_case=B, trace=True, snapshots=True, model=oracle.MODEL_TREE)
    assert r.status == 0
    assert a.tobytes() == want.tobytes()
    # level 0: the recorded sample's splitters, a stable partition by the descent
    r0 = r.records[0]
    if r0.kind == oracle.MODEL_TREE:
        spl = oracle.tree_splitters(r0.sample.view(src.dtype), k)
        heap = build_heap([int(v) for v in spl])
        ok = oracle.ordering_keys(src)
        b = np.array([descend(heap, k, int(o)) for o in ok])
        assert np.array_equal(np.bincount(b, minlength=k), r0.counts)
        assert np.array_equal(r.snapshots[0].view(src.dtype), src[np.argsort(b, kind="stable")])


def test_all_equal_requeues_to_eq3():
    a = np.full(50000, 3.0)
    r = oracle.sort(a, k=256, base_case=4096, trace=True, model=oracle.MODEL_TREE)
    assert r.status == 0
    assert r.records[0].kind == oracle.MODEL_TREE and r.records[0].requeued == 1
    assert r.records[1].kind == oracle.MODEL_EQ3


def test_tree_needs_power_of_two_k():
    a = np.random.default_rng(0).random(10000)
    assert oracle.sort(a.copy(), k=1000, model=oracle.MODEL_TREE).status == 1
    assert oracle.sort(a.copy(), k=1024, model=oracle.MODEL_TREE).status == 0


# ---- equality buckets (R24): MODEL_TREE_EQ ----

def eq_bucket_paper(heap, sorted_spl, leaves, o):
    """the descent over the tree of `leaves` leaves, then "a bucket B_i just for the
    elements x = s_i": bucket 2i+1 for a key equal to its leaf's splitter, else 2i."""
    i = descend(heap, leaves, o)
    return 2 * i + (1 if i < leaves - 1 and o == sorted_spl[i] else 0)


def test_equality_bucket_hand_example():
    # splitters of a tree of 8 leaves; 2.0 is a duplicated splitter
    vals = [-1.0, 0.0, 2.0, 2.0, 2.0, 5.0, 7.0]
    spl = oracle.ordering_keys(np.array(vals))
    want = {-2.0: 0, -1.0: 1, -0.5: 2, 0.0: 3, 1.0: 4, 2.0: 5, 3.0: 10, 5.0: 11, 6.0: 12,
            7.0: 13, 9.0: 14}
    for x, b in want.items():
        assert oracle.tree_eq_bucket(x, spl, 8) == b, x
    # -0.0 is below the splitter 0.0 in ordering-key order, so it is not "equal" to it
    assert oracle.tree_eq_bucket(-0.0, spl, 8) == 2


@pytest.mark.parametrize("leaves", [4, 8, 128, 512])
def test_equality_buckets_definition(leaves):
    rng = np.random.default_rng(leaves)
    for trial in range(10):
        S = int(rng.integers(leaves, 4 * leaves))
        smp = np.sort(rng.normal(0, 1, S) if trial % 2 else rng.integers(0, 40, S).astype(np.float64))
        spl = oracle.tree_splitters(smp, leaves)
        sl = [int(v) for v in spl]
        heap = build_heap(sl)
        sset = set(sl)
        keys = np.concatenate([smp, rng.normal(0, 1.5, 200), [-0.0, 0.0, np.inf, -np.inf]])
        for x in keys:
            o = int(oracle.ordering_keys(np.array([x]))[0])
            b = oracle.tree_eq_bucket(x, spl, leaves)
            assert b == eq_bucket_paper(heap, sl, leaves, o)
            i = b // 2
            if b & 1:   # an equality bucket holds exactly the keys equal to its splitter
                assert o == sl[i]
            else:       # the others lie strictly between the neighbouring splitters
                assert o not in sset
                assert (i == 0 or sl[i - 1] < o) and (i == leaves - 1 or o < sl[i])


@pytest.mark.parametrize("kind", ["uniform", "normal", "few_distinct", "u64_above_2_53",
                                  "signed_zeros", "infs", "mixture"])
@pytest.mark.parametrize("n,k,B", [(5000, 16, 64), (70001, 256, 4096), (120000, 1024, 4096)])
def test_tree_eq_sort_matches_numpy_and_stable_levels(kind, n, k, B):
    rng = np.random.default_rng(n + k + len(kind) + 1)
    a = datagen.fuzz_array(rng, n, kind)
    want = a[np.argsort(oracle.ordering_keys(a), kind="stable")]
    src = a.copy()
    r = oracle.sort(a, k=k, base_case=B, trace=True, snapshots=True, model=oracle.MODEL_TREE_EQ)
    assert r.status == 0
    assert a.tobytes() == want.tobytes()
    r0 = r.records[0]
    if r0.kind == oracle.MODEL_TREE:
        spl = oracle.tree_splitters(r0.sample.view(src.dtype), k // 2)
        sl = [int(v) for v in spl]
        heap = build_heap(sl)
        ok = oracle.ordering_keys(src)
        b = np.array([eq_bucket_paper(heap, sl, k // 2, int(o)) for o in ok])
        assert np.array_equal(np.bincount(b, minlength=k), r0.counts)
        snap = r.snapshots[0].view(src.dtype)
        assert np.array_equal(snap, src[np.argsort(b, kind="stable")])
        # "the equality bucket B_i will already be sorted as all the elements on it
        # are identical"
        off = np.concatenate([[0], np.cumsum(r0.counts)]).astype(np.int64)
        sok = oracle.ordering_keys(snap)
        for j in range(1, k, 2):
            if off[j + 1] > off[j]:
                assert sok[off[j]:off[j + 1]].min() == sok[off[j]:off[j + 1]].max()


def test_equality_buckets_retire_heavy_duplicates_at_once():
    """decision trees with equality buckets are robust against many duplicates: half
    of the keys share one value, which the sample sees, so it becomes a splitter and all its
    copies are final after level 0; without equality buckets they are partitioned again."""
    rng = np.random.default_rng(7)
    n = 200000
    a = rng.random(n)
    a[rng.random(n) < 0.5] = 0.5
    want = np.sort(a)
    work = {}
    for model in (oracle.MODEL_TREE, oracle.MODEL_TREE_EQ):
        b = a.copy()
        r = oracle.sort(b, k=256, base_case=4096, trace=True, model=model)
        assert r.status == 0 and np.array_equal(b, want)
        work[model] = sum(rec.m for rec in r.records if rec.level >= 1)
        if model == oracle.MODEL_TREE_EQ:
            assert all(rec.requeued == 0 for rec in r.records)
    dup = int((a == 0.5).sum())
    assert work[oracle.MODEL_TREE] >= dup          # the duplicates go down at least once more
    assert work[oracle.MODEL_TREE_EQ] <= n - dup   # never again


def test_tree_eq_needs_power_of_two_k_at_least_8():
    a = np.random.default_rng(0).random(10000)
    assert oracle.sort(a.copy(), k=4, model=oracle.MODEL_TREE_EQ).status == 1
    assert oracle.sort(a.copy(), k=1000, model=oracle.MODEL_TREE_EQ).status == 1
    assert oracle.sort(a.copy(), k=8, base_case=64, model=oracle.MODEL_TREE_EQ).status == 0
