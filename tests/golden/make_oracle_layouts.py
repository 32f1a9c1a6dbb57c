"""Write tests/golden/oracle_layouts.txt by running ONLY the CPU oracle (oracle/) on the
BASELINE configs at full size: a digest of the array image after every level.

The image after level L is fixed except inside the children of terminal segments (every
child <= base case) of levels <= L, whose interior order is unspecified (R11: the
base case sorts them).  layout_digest() hashes the fixed positions in order and every such
child by an order-independent multiset summary (sum and xor of a 64-bit mix of its keys), so
the GPU image after each level can be compared with the oracle's at full size without
storing either.  Pure numpy test infrastructure: it computes nothing of the method.
"""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def _mix64(x):
    x = x.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        x += np.uint64(0x9E3779B97F4A7C15)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def free_ranges(records, level, base_case):
    """(lo, hi) of the children (> 1 key) of terminal segments at levels <= level."""
    los, his = [], []
    for r in records:
        if r.level > level:
            continue
        cnt = np.asarray(r.counts, dtype=np.int64)
        if cnt.size and cnt.max() <= base_case:
            edges = r.begin + np.concatenate([[0], np.cumsum(cnt)])
            lo, hi = edges[:-1], edges[1:]
            keep = hi - lo > 1
            los.append(lo[keep])
            his.append(hi[keep])
    if not los:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    lo, hi = np.concatenate(los), np.concatenate(his)
    o = np.argsort(lo, kind="stable")
    return lo[o], hi[o]


def layout_digest(image_u64, lo, hi):
    n = image_u64.size
    d = np.zeros(n + 1, dtype=np.int32)
    np.add.at(d, lo, 1)
    np.add.at(d, hi, -1)
    free = np.cumsum(d[:-1]) > 0
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(image_u64[~free]).astype("<u8").tobytes())
    if lo.size:
        mixed = _mix64(image_u64[free])
        starts = np.concatenate([[0], np.cumsum(hi - lo)[:-1]])
        sums = np.add.reduceat(mixed, starts)
        xors = np.bitwise_xor.reduceat(mixed, starts)
        h.update(np.stack([lo.astype(np.uint64), hi.astype(np.uint64), sums, xors], axis=1)
                 .astype("<u8").tobytes())
    return h.hexdigest()[:16]


def main():
    import oracle
    from paper_2208_06902_b200 import datagen
    names = sys.argv[1:] or list(datagen.CONFIGS)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "oracle_layouts.txt")
    lines = ["# Written by tests/golden/make_oracle_layouts.py (oracle/ only; seed 0x49504C53).",
             "# LAYOUT cfg level digest  (layout_digest of the image after the level)"]
    for name in names:
        cfg = datagen.CONFIGS[name]
        a = datagen.generate(name)
        r = oracle.sort(a, k=cfg.k, base_case=cfg.base_case, trace=True, snapshots=True)
        assert r.status == 0
        for lv, snap in enumerate(r.snapshots):
            lo, hi = free_ranges(r.records, lv, cfg.base_case)
            lines.append(f"LAYOUT {name} {lv} {layout_digest(snap.view(np.uint64), lo, hi)}")
            print(lines[-1], flush=True)
        del r, a
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
