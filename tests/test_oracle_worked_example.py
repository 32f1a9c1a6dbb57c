"""Oracle vs the paper's worked example (PAPER.md Chapter 4)."""
import numpy as np

import oracle


def _we(golden):
    g = golden("worked_example.txt")
    f = lambda key: [float(t) for t in g[key][0]]
    i = lambda key: [int(t) for t in g[key][0]]
    return g, f, i


def test_key28_bucket(golden):
    g, f, i = _we(golden)
    a, b, k = f("a")[0], f("b")[0], i("k")[0]
    # floor(0.15 * 28 - 1.55) = floor(2.65) = 2
    assert oracle.bucket(28.0, a, b, k) == i("key28")[0]
    # SPEC.md examples restating the same figure: key 2 -> 0 (clamp), key 50 -> 3 (clamp)
    assert oracle.bucket(2.0, a, b, k) == 0
    assert oracle.bucket(50.0, a, b, k) == 3


def test_contiguous_layout_is_stable_partition(golden):
    """P:527 is exactly the stable counting partition of P:486 by the model of P:491."""
    g, f, i = _we(golden)
    x = np.array(f("input"))
    out, off, ids = oracle.partition(x, f("a")[0], f("b")[0], i("k")[0])
    assert out.tolist() == f("contiguous")
    sizes = np.diff(off).tolist()
    assert sizes == i("bucket_sizes")
    assert off.tolist() == [0, 7, 9, 13, 20]


def test_buffered_classification_table(golden):
    """IPS4o-style classification with buffer size 2 reproduces the colored
    table from the oracle's per-key buckets (checks every bucket id, incl. colours)."""
    g, f, i = _we(golden)
    x = np.array(f("input"))
    _, _, ids = oracle.partition(x, f("a")[0], f("b")[0], i("k")[0])
    buf = {b: [] for b in range(4)}
    written, written_b = [], []
    for key, b in zip(x.tolist(), ids.tolist()):
        buf[b].append(key)
        if len(buf[b]) == 2:  # flush a full block of b = 2 keys
            written += buf[b]; written_b += [b, b]; buf[b] = []
    for b in range(4):  # cleanup: partially filled buffers are flushed in bucket order
        written += buf[b]; written_b += [b] * len(buf[b])
    # The table lists the flushed blocks first, then the leftovers.
    assert written_b == i("buffered_buckets")
    assert written == f("buffered")


def test_sorted_output(golden):
    """the final array."""
    g, f, i = _we(golden)
    x = np.array(f("input"))
    r = oracle.sort(x, k=4, base_case=9)
    assert r.status == 0
    assert x.tolist() == f("sorted")
