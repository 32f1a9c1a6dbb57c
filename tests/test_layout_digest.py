"""Pins of tests/golden/make_oracle_layouts.py's layout_digest (test infrastructure): it must
be blind exactly to the order inside the free ranges (children of terminal segments, R11)
and see everything else."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from make_oracle_layouts import layout_digest  # noqa: E402


def _case():
    rng = np.random.default_rng(7)
    img = rng.integers(0, 2 ** 64 - 1, 5000, dtype=np.uint64, endpoint=True)
    lo = np.array([10, 100, 2000, 4990], dtype=np.int64)
    hi = np.array([20, 400, 2001 + 50, 5000], dtype=np.int64)
    return rng, img, lo, hi


def test_blind_to_order_inside_free_ranges():
    rng, img, lo, hi = _case()
    d0 = layout_digest(img, lo, hi)
    b = img.copy()
    for l, h in zip(lo, hi):
        rng.shuffle(b[l:h])
    assert layout_digest(b, lo, hi) == d0


def test_sees_fixed_positions_and_multisets():
    rng, img, lo, hi = _case()
    d0 = layout_digest(img, lo, hi)
    b = img.copy(); b[5] ^= np.uint64(1)                    # a fixed position
    assert layout_digest(b, lo, hi) != d0
    b = img.copy(); b[[6, 7]] = b[[7, 6]]                   # order of fixed positions
    assert layout_digest(b, lo, hi) != d0
    b = img.copy(); b[15] ^= np.uint64(1 << 40)             # a key inside a free range
    assert layout_digest(b, lo, hi) != d0
    b = img.copy(); b[[15, 150]] = b[[150, 15]]             # a key moved between free ranges
    assert layout_digest(b, lo, hi) != d0
    b = img.copy(); b[[19, 20]] = b[[20, 19]]               # across a free range's edge
    assert layout_digest(b, lo, hi) != d0
    assert layout_digest(img, lo[:3], hi[:3]) != d0         # other free ranges
