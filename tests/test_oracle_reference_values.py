"""Oracle vs SURVEY.md §8(c) cross-implementation reference values and the BASELINE input
hashes.  Level-0 values at full size are cheap; full-size digests run the whole oracle."""
import hashlib
import struct

import numpy as np
import pytest

import oracle
from paper_2208_06902_b200 import datagen


def bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def h16(b):
    return hashlib.sha256(b).hexdigest()[:16]


@pytest.fixture(scope="module")
def ref(golden):
    return golden("survey_reference.txt")


def level0(a, cfg):
    """Level 0 exactly as oracle.sort does it, exposed step by step."""
    kt = oracle.KEY_U64 if a.dtype == np.uint64 else oracle.KEY_F64
    n = a.size
    S = oracle.sample_size(n, cfg.k)
    idx = oracle.sample_positions(oracle.DEFAULT_SEED, 0, 0, n, S)
    smp = a[idx.astype(np.int64)]
    smp = smp[np.argsort(oracle.ordering_keys(smp), kind="stable")]
    fit = oracle.fit_fmcd(smp.astype(np.float64), cfg.k)
    out, off, ids = oracle.partition(a, fit.A, fit.B, cfg.k)
    return S, smp, fit, np.diff(off), ids


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_level0_reference(name, ref, golden):
    cfg = datagen.CONFIGS[name]
    a = datagen.generate(name)
    want_sha = dict((r[0], r[1]) for r in golden("inputs.txt").get(name, []) and
                    [[name, golden("inputs.txt")[name][0][0]]])
    assert datagen.sha256(a) == want_sha[name]
    row = [r for r in ref["L0"] if r[0] == name][0]
    S, smp, fit, counts, ids = level0(a, cfg)
    assert S == int(row[1]) and fit.D == int(row[2])
    assert bits(fit.A) == int(row[3], 16) and bits(fit.B) == int(row[4], 16)
    c = counts.astype("<u8")
    assert int(c.max()) == int(row[5]) and int(c.argmax()) == int(row[6])
    assert int(c[0]) == int(row[7]) and int(c[-1]) == int(row[8])
    assert h16(c.tobytes()) == row[9]
    assert h16(ids.astype("<u2").tobytes()) == row[10]
    assert h16(smp.tobytes()) == row[11]


def test_worked_example_digests(ref):
    a = np.array([18, 39, 33, 28, 25, 34, 11, 27, 47, 2, 48, 50, 10, 6, 36, 13, 9, 12, 22, 29],
                 dtype=np.float64)
    r = oracle.sort(a, k=4, base_case=9, trace=True)
    row = [x for x in ref["DIG"] if x[0] == "WE"][0]
    assert oracle.level_digests(r.records) == row[1:row.index("final")]
    assert h16(a.tobytes()) == row[row.index("final") + 1]


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_full_digests(name, ref):
    cfg = datagen.CONFIGS[name]
    a = datagen.generate(name)
    r = oracle.sort(a, k=cfg.k, base_case=cfg.base_case, trace=True)
    assert r.status == 0
    row = [x for x in ref["DIG"] if x[0] == name][0]
    assert oracle.level_digests(r.records) == row[1:row.index("final")]
    assert h16(a.tobytes()) == row[row.index("final") + 1]
    ok = oracle.ordering_keys(a)
    assert np.all(ok[:-1] <= ok[1:])
