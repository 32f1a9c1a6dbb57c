"""Write tests/golden/oracle_digests.txt by running ONLY the CPU oracle (oracle/) on the
BASELINE configs at full size.  The GPU parity tests compare the CUDA path's trace and
final array against these oracle-produced values.

Per level: digest of the 48-byte segment records (SURVEY §8(c) format), of the child
counts (k_eff x u64 per record, in begin order) and of the sorted samples (raw key bits).
"""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2208_06902_b200 import datagen  # noqa: E402


def digests(records):
    by = {}
    for r in records:
        by.setdefault(r.level, []).append(r)
    out = []
    for lv in sorted(by):
        rs = sorted(by[lv], key=lambda r: r.begin)
        h1, h2, h3 = hashlib.sha256(), hashlib.sha256(), hashlib.sha256()
        for r in rs:
            h1.update(r.packed())
            h2.update(r.counts.astype("<u8").tobytes())
            h3.update(r.sample.astype("<u8").tobytes())
        out.append((lv, len(rs), h1.hexdigest()[:16], h2.hexdigest()[:16], h3.hexdigest()[:16]))
    return out


def main():
    # usage: make_oracle_digests.py [--tree | --tree-eq] [cfg ...]; --tree: the splitter-tree
    # model (IPLS_FLAG_TREE_MODEL, R22-R23) into oracle_digests_tree.txt; --tree-eq: the tree
    # with equality buckets (R24) into oracle_digests_tree_eq.txt
    args = sys.argv[1:]
    tree = "--tree" in args
    tree_eq = "--tree-eq" in args
    args = [x for x in args if x not in ("--tree", "--tree-eq")]
    names = args or list(datagen.CONFIGS)
    fname = ("oracle_digests_tree_eq.txt" if tree_eq else
             "oracle_digests_tree.txt" if tree else "oracle_digests.txt")
    flag = " --tree-eq" if tree_eq else " --tree" if tree else ""
    model = (oracle.MODEL_TREE_EQ if tree_eq else oracle.MODEL_TREE if tree
             else oracle.MODEL_LINEAR)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), fname)
    lines = [f"# Written by tests/golden/make_oracle_digests.py{flag} "
             "(oracle/ only; seed 0x49504C53).",
             "# LEVEL cfg level n_records records_sha counts_sha samples_sha",
             "# FINAL cfg levels final_sha256"]
    for name in names:
        cfg = datagen.CONFIGS[name]
        a = datagen.generate(name)
        r = oracle.sort(a, k=cfg.k, base_case=cfg.base_case, trace=True, model=model)
        assert r.status == 0
        for lv, nrec, d1, d2, d3 in digests(r.records):
            lines.append(f"LEVEL {name} {lv} {nrec} {d1} {d2} {d3}")
        lines.append(f"FINAL {name} {r.levels} {hashlib.sha256(a.tobytes()).hexdigest()}")
        print(lines[-1], flush=True)
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
