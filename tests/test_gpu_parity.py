"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, element by element.

Bit-exact everywhere: FMCD coefficients (A, B bits), D, kind, pivot, per-key bucket ids,
bucket counts, per-level layouts and the final array.
"""
import hashlib
import os

import numpy as np
import pytest

import oracle
from paper_2208_06902_b200 import datagen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def ipls():
    import paper_2208_06902_b200 as m
    assert torch.cuda.is_available()
    m.lib()
    return m


def dev(a: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64).copy()).cuda()


def host(t, dtype):
    return t.cpu().numpy().view(dtype)


def kt_of(a):
    return 0 if a.dtype == np.float64 else 1


def ok_sorted_sample(a, idx):
    s = a[idx.astype(np.int64)]
    return s[np.argsort(oracle.ordering_keys(s), kind="stable")]


# ---------------------------------------------------------------- FMCD (K2) ----------
def fit_cases():
    rng = np.random.default_rng(11)
    cases = []
    for t in range(60):
        S = int(rng.choice([4, 5, 17, 100, 1023, 3071, 4095, 6143, 7167, 8192]))
        k = int(rng.choice([3, 4, 10, 256, 1024]))
        dist = ["normal", "lognormal", "uniform", "ints", "dups", "const", "sorted_i",
                "u64"][t % 8]
        if dist == "normal":
            a = rng.normal(0, 1, S)
        elif dist == "lognormal":
            a = rng.lognormal(0, 2, S)
        elif dist == "uniform":
            a = rng.random(S)
        elif dist == "ints":
            a = rng.integers(0, 50, S).astype(np.float64)
        elif dist == "dups":
            a = np.where(rng.random(S) < 0.9, 1.0, rng.normal(0, 1, S))
        elif dist == "const":
            a = np.full(S, -2.5)
        elif dist == "sorted_i":
            a = np.arange(S, dtype=np.float64)
        else:
            a = rng.integers(0, 2 ** 64 - 1, S, dtype=np.uint64, endpoint=True)
        cases.append((a, k))
    return cases


@pytest.mark.parametrize("case", range(60))
def test_fit_fmcd_parity(ipls, case):
    a, k = fit_cases()[case]
    s = a[np.argsort(oracle.ordering_keys(a), kind="stable")]
    m = ipls.fit_fmcd(dev(s), k, key_type=kt_of(s))
    if s.size < 4:
        return
    o = oracle.fit_fmcd(s.astype(np.float64), k)
    assert m.degenerate == o.degenerate
    if o.degenerate:
        assert m.kind == ipls.MODEL_EQ3
        assert m.pivot_ok == int(oracle.ordering_keys(s[s.size // 2:s.size // 2 + 1])[0])
    else:
        assert (m.D, bool(m.capped)) == (o.D, o.capped)
        assert m.a == o.A and m.b == o.B  # bit-exact binary64


# ---------------------------------------------------------- partition (K3..K4) -------
def test_partition_worked_example(ipls, golden):
    g = golden("worked_example.txt")
    x = np.array([float(v) for v in g["input"][0]])
    mdl = ipls.Model(0.15, -1.55, 4, 0, ipls.MODEL_LINEAR, 0, 0)
    out = torch.empty(x.size, dtype=torch.int64, device="cuda")
    off, ids = ipls.partition_level(dev(x), out, mdl, key_type=0, want_ids=True)
    assert host(out, np.float64).tolist() == [float(v) for v in g["contiguous"][0]]
    assert off.cpu().tolist() == [0, 7, 9, 13, 20]
    assert ids.cpu().numpy().tolist() == [1, 3, 3, 2, 2, 3, 0, 2, 3, 0, 3, 3, 0, 0, 3, 0, 0, 0,
                                          1, 2]


@pytest.mark.parametrize("n", [0, 1, 2, 31, 4095, 4096, 4097, 65536 * 3 + 17, 1_000_003])
@pytest.mark.parametrize("dist", ["normal", "lognormal", "dups", "u64"])
@pytest.mark.parametrize("k", [3, 256, 1024])
def test_partition_level_parity(ipls, n, dist, k):
    rng = np.random.default_rng(n * 7 + k)
    if dist == "normal":
        a = rng.normal(0, 1, n)
    elif dist == "lognormal":
        a = rng.lognormal(0, 2, n)
    elif dist == "dups":
        a = rng.integers(0, 7, n).astype(np.float64)
    else:
        a = rng.integers(0, 2 ** 64 - 1, n, dtype=np.uint64, endpoint=True)
    if n >= 8:
        S = min(oracle.sample_size(n, k), 8192)
        idx = oracle.sample_positions(oracle.DEFAULT_SEED, 0, 0, n, S)
        fit = oracle.fit_fmcd(ok_sorted_sample(a, idx).astype(np.float64), k)
    else:
        fit = oracle.Fit(1.0, 0.0, 1, False, False)
    if fit.degenerate or k == 3:
        piv = int(oracle.ordering_keys(a[n // 2:n // 2 + 1])[0]) if n else 0
        kind, A, B, kk = oracle.MODEL_EQ3, 0.0, 0.0, 3
    else:
        kind, A, B, kk = oracle.MODEL_LINEAR, fit.A, fit.B, k
        piv = 0
    want, woff, wids = oracle.partition(a, A, B, kk, kind=kind, pivot_ok=piv)
    mdl = ipls.Model(A, B, kk, 0, kind, 0, piv)
    out = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")[:n]
    off, ids = ipls.partition_level(dev(a), out, mdl, key_type=kt_of(a), want_ids=True)
    assert np.array_equal(off.cpu().numpy().astype(np.uint64), woff)
    assert host(out, a.dtype).tobytes() == want.tobytes()
    assert np.array_equal(ids.cpu().numpy().view(np.uint16), wids)


# ------------------------------------------------------------- whole sort ------------
def compare_traces(gtr, ores):
    assert gtr.levels == ores.levels
    assert len(gtr.records) == len(ores.records)
    for g, o in zip(gtr.records, ores.records):
        assert (g.level, g.begin, g.m, g.S) == (o.level, o.begin, o.m, o.S)
        assert (g.kind, g.D, g.capped, g.pivot_ok, g.k_eff, g.requeued) == \
            (o.kind, o.D, o.capped, o.pivot_ok, o.k_eff, o.requeued)
        assert g.A == o.A and g.B == o.B
        assert np.array_equal(g.counts, o.counts)
        assert np.array_equal(g.sample, o.sample)


FUZZ_SIZES = [(2, 4, 1), (9, 4, 2), (100, 4, 9), (5000, 16, 64), (70_001, 256, 4096),
              (300_000, 1024, 4096), (200_000, 64, 100)]


@pytest.mark.parametrize("kind", datagen.FUZZ_KINDS)
@pytest.mark.parametrize("size", range(len(FUZZ_SIZES)))
def test_sort_parity_fuzz(ipls, kind, size):
    n, k, B = FUZZ_SIZES[size]
    rng = np.random.default_rng(size * 131 + len(kind))
    a = datagen.fuzz_array(rng, n, kind)
    sort_parity_with_layouts(ipls, a, k, B)


@pytest.mark.parametrize("order", ["sorted", "reverse", "runs8", "bucket_blocks"])
@pytest.mark.parametrize("n,k", [(3_000_000, 256), (3_000_000, 1024), (1_500_007, 64)])
def test_presorted_parity(ipls, order, n, k):
    """Presorted inputs put whole warps of keys into one bucket: the scatters' dense-tile path
    (one aggregated atomic per warp, K3) must keep the stable layouts bit-exact."""
    rng = np.random.default_rng(n + k)
    a = rng.normal(0, 1, n)
    if order == "sorted":
        a = np.sort(a)
    elif order == "reverse":
        a = np.sort(a)[::-1].copy()
    elif order == "runs8":
        a = np.concatenate([np.sort(x) for x in np.array_split(a, 8)])
    else:  # what dist_sort's local sorts receive: coarse ranges in order, random inside
        q = np.floor(a * 8).astype(np.int64)
        a = a[np.argsort(q, kind="stable")]
    sort_parity_with_layouts(ipls, a, k, 4096)


def sort_parity_with_layouts(ipls, a, k, B):
    want = a.copy()
    ores = oracle.sort(want, k=k, base_case=B, trace=True, snapshots=True)
    t = dev(a)
    gtr = ipls.sort_trace(t, k=k, base_case=B, key_type=kt_of(a),
                          snapshot_levels=max(1, ores.levels))
    assert host(t, a.dtype).tobytes() == want.tobytes()
    compare_traces(gtr, ores)
    # Layout after every level: bit-exact, except inside the children of terminal segments
    # (every child <= base case).  Those are handed to the base case, an exact sort, right
    # after the level, so their interior order is unspecified (R11); the GPU places
    # them unstably and only their multisets must agree.
    free = []  # (level, begin, end) of children whose interior order is unspecified
    for o in ores.records:
        cnt = np.asarray(o.counts, dtype=np.int64)
        if cnt.max() <= B:
            edges = o.begin + np.concatenate([[0], np.cumsum(cnt)])
            free += [(o.level, int(lo), int(hi)) for lo, hi in zip(edges[:-1], edges[1:]) if hi - lo > 1]
    for lv in range(ores.levels):
        g = gtr.snapshots[lv].cpu().numpy().view(np.uint64).copy()
        w = ores.snapshots[lv].copy()
        for flv, lo, hi in free:
            if flv <= lv:
                g[lo:hi] = np.sort(g[lo:hi])
                w[lo:hi] = np.sort(w[lo:hi])
        assert np.array_equal(g, w), f"layout after level {lv} differs"


@pytest.mark.parametrize("kind", datagen.STRESS_KINDS)
@pytest.mark.parametrize("n,k", [(300_000, 1024), (1_000_003, 256), (2_000_000, 1024)])
def test_base_case_stress_parity(ipls, kind, n, k):
    """Clustered keys put several keys (in every order, up to > kFineOverflow) into one
    interpolation bin of the base case: warp windows (k=1024: children ~100-300 keys) and
    CTA windows (k=256 at 1e6: children ~4k keys); negative, zero-straddling and u64 windows."""
    rng = np.random.default_rng(n + k + len(kind))
    a = datagen.stress_array(rng, n, kind)
    want = a.copy()
    oracle.sort(want, k=k, base_case=4096)
    t = dev(a)
    ipls.sort(t, k=k, base_case=4096, key_type=kt_of(a))
    assert host(t, a.dtype).tobytes() == want.tobytes()


@pytest.mark.parametrize("name", list(datagen.PAPER_WORKLOADS))
@pytest.mark.parametrize("n,k", [(300_000, 1024), (1_000_003, 256)])
def test_paper_workloads_parity(ipls, name, n, k):
    """The paper's nine synthetic workloads: models, counts,
    samples at every level and the final array, bit-exact against the oracle."""
    a = datagen.paper_workload(name, n)
    want = a.copy()
    ores = oracle.sort(want, k=k, base_case=4096, trace=True)
    t = dev(a)
    gtr = ipls.sort_trace(t, k=k, base_case=4096, key_type=kt_of(a))
    assert host(t, a.dtype).tobytes() == want.tobytes()
    compare_traces(gtr, ores)


TREE_KINDS = ["uniform", "normal", "lognormal", "few_distinct", "two_values", "signed_zeros",
              "infs", "u64_above_2_53", "root_dups_u64", "mixture"]


@pytest.mark.parametrize("kind", TREE_KINDS)
@pytest.mark.parametrize("n,k,B", [(5000, 16, 64), (70_001, 256, 4096), (300_000, 1024, 4096)])
def test_tree_model_parity(ipls, kind, n, k, B):
    """Splitter-tree model (R22-R24): samples, tree kind, per-segment counts,
    every level's layout and the final array, bit-exact against the oracle's tree model."""
    rng = np.random.default_rng(n + k + len(kind))
    a = datagen.fuzz_array(rng, n, kind)
    want = a.copy()
    ores = oracle.sort(want, k=k, base_case=B, trace=True, snapshots=True,
                       model=oracle.MODEL_TREE)
    t = dev(a)
    gtr = ipls.sort_trace(t, k=k, base_case=B, key_type=kt_of(a),
                          snapshot_levels=max(1, ores.levels), model=ipls.MODEL_TREE)
    assert host(t, a.dtype).tobytes() == want.tobytes()
    compare_traces(gtr, ores)
    assert any(r.kind == ipls.MODEL_TREE for r in gtr.records) or kind in ("few_distinct",
                                                                           "two_values")


@pytest.mark.parametrize("name", ["C2", "C3", "C5"])
def test_tree_model_configs_scaled(ipls, name):
    a = datagen.generate(name, 2_000_000)
    cfg = datagen.CONFIGS[name]
    want = a.copy()
    ores = oracle.sort(want, k=cfg.k, base_case=cfg.base_case, trace=True,
                       model=oracle.MODEL_TREE)
    t = dev(a)
    gtr = ipls.sort_trace(t, k=cfg.k, base_case=cfg.base_case, key_type=kt_of(a),
                          model=ipls.MODEL_TREE)
    assert host(t, a.dtype).tobytes() == want.tobytes()
    compare_traces(gtr, ores)


@pytest.mark.parametrize("kind", TREE_KINDS)
@pytest.mark.parametrize("n,k,B", [(5000, 16, 64), (70_001, 256, 4096), (300_000, 1024, 4096)])
def test_tree_equal_buckets_parity(ipls, kind, n, k, B):
    """The tree with IPS4o's equality buckets (R24): samples, per-segment counts, every
    level's layout and the final array, bit-exact against the oracle's MODEL_TREE_EQ."""
    rng = np.random.default_rng(n + k + len(kind) + 1)
    a = datagen.fuzz_array(rng, n, kind)
    want = a.copy()
    ores = oracle.sort(want, k=k, base_case=B, trace=True, snapshots=True,
                       model=oracle.MODEL_TREE_EQ)
    t = dev(a)
    gtr = ipls.sort_trace(t, k=k, base_case=B, key_type=kt_of(a),
                          snapshot_levels=max(1, ores.levels), model=ipls.MODEL_TREE_EQ)
    assert host(t, a.dtype).tobytes() == want.tobytes()
    compare_traces(gtr, ores)
    # the untraced entry point gives the same bytes
    t2 = dev(a)
    ipls.sort(t2, k=k, base_case=B, key_type=kt_of(a), model=ipls.MODEL_TREE_EQ)
    assert torch.equal(t, t2)


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_tree_equal_buckets_configs_scaled(ipls, name):
    a = datagen.generate(name, 2_000_000)
    cfg = datagen.CONFIGS[name]
    want = a.copy()
    ores = oracle.sort(want, k=cfg.k, base_case=cfg.base_case, trace=True,
                       model=oracle.MODEL_TREE_EQ)
    t = dev(a)
    gtr = ipls.sort_trace(t, k=cfg.k, base_case=cfg.base_case, key_type=kt_of(a),
                          model=ipls.MODEL_TREE_EQ)
    assert host(t, a.dtype).tobytes() == want.tobytes()
    compare_traces(gtr, ores)


def test_tree_equal_buckets_heavy_duplicates(ipls):
    """Half of the keys share one value (P:382's case): all of them are final after level 0,
    exactly as in the oracle."""
    rng = np.random.default_rng(7)
    n = 1_000_000
    a = rng.random(n)
    a[rng.random(n) < 0.5] = 0.5
    want = a.copy()
    ores = oracle.sort(want, k=1024, base_case=4096, trace=True, snapshots=True,
                       model=oracle.MODEL_TREE_EQ)
    t = dev(a)
    gtr = ipls.sort_trace(t, k=1024, base_case=4096, key_type=kt_of(a),
                          snapshot_levels=max(1, ores.levels), model=ipls.MODEL_TREE_EQ)
    assert host(t, a.dtype).tobytes() == want.tobytes()
    compare_traces(gtr, ores)
    assert sum(r.m for r in gtr.records if r.level >= 1) <= n - int((a == 0.5).sum())


def test_tree_equal_buckets_flag_validation(ipls):
    t = dev(np.random.default_rng(0).random(10000))
    with pytest.raises(ipls.IPLSError):
        ipls.sort(t, k=4, model=ipls.MODEL_TREE_EQ)       # k >= 8
    with pytest.raises(ipls.IPLSError):
        ipls.sort(t, k=1000, model=ipls.MODEL_TREE_EQ)    # k a power of two
    assert ipls.workspace_bytes(10000, ipls.KEY_F64, k=4, model=ipls.MODEL_TREE_EQ) == 0


def test_tree_model_nan_rejected_unmodified(ipls):
    a = np.random.default_rng(3).normal(0, 1, 300_000)
    a[123_456] = np.nan
    t = dev(a)
    with pytest.raises(ipls.IPLSError) as e:
        ipls.sort(t, k=1024, key_type=ipls.KEY_F64, model=ipls.MODEL_TREE)
    assert e.value.status == 2
    assert host(t, np.float64).tobytes() == a.tobytes()


def test_tree_model_rejects_k_not_power_of_two(ipls):
    t = dev(np.random.default_rng(0).random(10000))
    with pytest.raises(ipls.IPLSError):
        ipls.sort(t, k=1000, model=ipls.MODEL_TREE)


@pytest.mark.parametrize("k,B,n", [(3, 1, 3000), (5, 17, 20_000), (7, 255, 100_000),
                                   (100, 4096, 250_000), (1000, 1000, 400_001),
                                   (513, 257, 150_000), (1023, 4096, 1_500_000)])
@pytest.mark.parametrize("kind", ["normal", "lognormal", "few_distinct", "u64_big"])
def test_sort_parity_odd_k_and_base(ipls, k, B, n, kind):
    """Fan-outs and base-case thresholds other than the configs' (k odd or not a power of two,
    B from 1 to 4096): full trace and final array against the oracle."""
    rng = np.random.default_rng(k * 7 + B + len(kind))
    a = datagen.fuzz_array(rng, n, kind)
    want = a.copy()
    ores = oracle.sort(want, k=k, base_case=B, trace=True)
    t = dev(a)
    gtr = ipls.sort_trace(t, k=k, base_case=B, key_type=kt_of(a))
    assert host(t, a.dtype).tobytes() == want.tobytes()
    compare_traces(gtr, ores)


def test_worked_example_sort(ipls, golden):
    x = np.array([float(v) for v in golden("worked_example.txt")["input"][0]])
    t = dev(x)
    want = x.copy()
    ores = oracle.sort(want, k=4, base_case=9, trace=True)
    gtr = ipls.sort_trace(t, k=4, base_case=9, key_type=0)
    assert host(t, np.float64).tolist() == [float(v) for v in golden("worked_example.txt")["sorted"][0]]
    compare_traces(gtr, ores)


@pytest.mark.parametrize("name,n", [("C1", None), ("C2", 2_000_000), ("C3", 2_000_000),
                                    ("C4", 2_000_000), ("C5", 3_000_000)])
def test_configs_scaled_full_trace(ipls, name, n):
    cfg = datagen.CONFIGS[name]
    a = datagen.generate(name, n)
    want = a.copy()
    ores = oracle.sort(want, k=cfg.k, base_case=cfg.base_case, trace=True)
    t = dev(a)
    gtr = ipls.sort_trace(t, k=cfg.k, base_case=cfg.base_case, key_type=kt_of(a))
    assert host(t, a.dtype).tobytes() == want.tobytes()
    compare_traces(gtr, ores)


def load_oracle_digests(fname="oracle_digests.txt"):
    lv, fin = {}, {}
    with open(os.path.join(GOLD, fname)) as f:
        for line in f:
            tok = line.split()
            if not tok or tok[0].startswith("#"):
                continue
            if tok[0] == "LEVEL":
                lv.setdefault(tok[1], []).append((int(tok[2]), int(tok[3]), tok[4], tok[5], tok[6]))
            elif tok[0] == "FINAL":
                fin[tok[1]] = (int(tok[2]), tok[3])
    return lv, fin


def gpu_digests(records):
    by = {}
    for r in records:
        by.setdefault(r.level, []).append(r)
    out = []
    for lv in sorted(by):
        rs = sorted(by[lv], key=lambda r: r.begin)
        h1, h2, h3 = hashlib.sha256(), hashlib.sha256(), hashlib.sha256()
        for r in rs:
            orec = oracle.Record(r.level, r.kind, r.begin, r.m, r.S, r.A, r.B, r.D, r.capped,
                                 r.pivot_ok, r.k_eff, r.requeued, r.sample, r.counts)
            h1.update(orec.packed())
            h2.update(r.counts.astype("<u8").tobytes())
            h3.update(r.sample.astype("<u8").tobytes())
        out.append((lv, len(rs), h1.hexdigest()[:16], h2.hexdigest()[:16], h3.hexdigest()[:16]))
    return out


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_configs_full_size_vs_oracle_digests(ipls, name):
    """Full BASELINE sizes, launched exactly as bench.py times them: every level's records,
    counts and samples, and the final array, against digests written by the oracle."""
    lvd, fin = load_oracle_digests()
    cfg = datagen.CONFIGS[name]
    a = datagen.generate(name)
    t = dev(a)
    del a
    gtr = ipls.sort_trace(t, k=cfg.k, base_case=cfg.base_case, key_type=kt_of(datagen.generate(name, 1)))
    assert gpu_digests(gtr.records) == lvd[name]
    assert gtr.levels == fin[name][0]
    h = hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()
    assert h == fin[name][1]
    # and the untraced entry point (the one bench.py times) gives the same bytes
    b = datagen.generate(name)
    t2 = dev(b)
    ipls.sort(t2, k=cfg.k, base_case=cfg.base_case, key_type=kt_of(b))
    assert torch.equal(t, t2)


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_tree_configs_full_size_vs_oracle_digests(ipls, name):
    """Splitter-tree model (NEXT #2) at full BASELINE sizes against oracle-written digests
    (tests/golden/oracle_digests_tree.txt)."""
    lvd, fin = load_oracle_digests("oracle_digests_tree.txt")
    cfg = datagen.CONFIGS[name]
    a = datagen.generate(name)
    t = dev(a)
    del a
    gtr = ipls.sort_trace(t, k=cfg.k, base_case=cfg.base_case,
                          key_type=kt_of(datagen.generate(name, 1)), model=ipls.MODEL_TREE)
    assert gpu_digests(gtr.records) == lvd[name]
    assert gtr.levels == fin[name][0]
    assert hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest() == fin[name][1]


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_tree_eq_configs_full_size_vs_oracle_digests(ipls, name):
    """The tree with equality buckets (R24) at full BASELINE sizes against oracle-written
    digests (tests/golden/oracle_digests_tree_eq.txt)."""
    lvd, fin = load_oracle_digests("oracle_digests_tree_eq.txt")
    cfg = datagen.CONFIGS[name]
    a = datagen.generate(name)
    t = dev(a)
    del a
    gtr = ipls.sort_trace(t, k=cfg.k, base_case=cfg.base_case,
                          key_type=kt_of(datagen.generate(name, 1)), model=ipls.MODEL_TREE_EQ)
    assert gpu_digests(gtr.records) == lvd[name]
    assert gtr.levels == fin[name][0]
    assert hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest() == fin[name][1]


def _mix_sum(t, step=1 << 28):
    """Order-independent multiset digest: wrapping sum of a SplitMix64-style mix of every key
    (int64 arithmetic on the GPU, in slices to bound the temporaries)."""
    acc = 0
    for i in range(0, t.numel(), step):
        z = t[i:i + step] * -7046029254386353131  # 0x9E3779B97F4A7C15
        z = (z ^ (z >> 30)) * -4658895280553007687  # 0xBF58476D1CE4E5B9
        z = (z ^ (z >> 27)) * -7723592293110705685  # 0x94D049BB133111EB
        acc = (acc + int((z ^ (z >> 31)).sum())) & 0xFFFFFFFFFFFFFFFF
    return acc


def test_api_maximum_size(ipls):
    """n = 2^32 - 1 keys (34 GB, the ABI's limit, odd): sorted, same multiset (the oracle
    cannot run at this size; the final array is defined by sortedness + multiset)."""
    n = 2**32 - 1
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=g).view(torch.int64)
    before = _mix_sum(x)
    ipls.sort(x, k=1024, base_case=4096, key_type=ipls.KEY_F64)
    f = x.view(torch.float64)
    step = 1 << 28
    for i in range(0, n - 1, step):  # sorted, checked in overlapping slices
        s = f[i:min(i + step + 1, n)]
        assert bool((s[1:] >= s[:-1]).all())
    assert _mix_sum(x) == before
    del x, f
    torch.cuda.empty_cache()


def test_nan_rejected_unmodified(ipls):
    rng = np.random.default_rng(0)
    for n in (10, 5000, 300_000):
        a = rng.normal(0, 1, n)
        a[n // 3] = np.nan
        t = dev(a)
        with pytest.raises(ipls.IPLSError) as e:
            ipls.sort(t, k=256, base_case=4096, key_type=0)
        assert e.value.status == 2
        assert host(t, np.float64).tobytes() == a.tobytes()


def test_trivial_sizes_and_args(ipls):
    t = torch.empty(0, dtype=torch.int64, device="cuda")
    ipls.sort(t, key_type=0)
    t = dev(np.array([3.5]))
    ipls.sort(t, key_type=0)
    assert host(t, np.float64).tolist() == [3.5]
    with pytest.raises(ipls.IPLSError):
        ipls.sort(dev(np.zeros(100)), k=2, key_type=0)
    with pytest.raises(ipls.IPLSError):
        ipls.sort(dev(np.zeros(100)), k=2048, key_type=0)


def test_sort_host_e2e(ipls):
    a = datagen.generate("C2", 3_000_000)
    want = np.sort(a)
    h = torch.from_numpy(a.copy()).pin_memory()
    ipls.sort_host_ptr(h.data_ptr(), h.numel(), ipls.KEY_F64, k=1024, base_case=4096)
    torch.cuda.synchronize()
    assert h.numpy().tobytes() == want.tobytes()


def test_sort_host_batch(ipls):
    """ipls_sort_host_batch: pipelined host arrays of mixed sizes (empty, one key, sizes
    that reallocate the internal buffers, u64 above 2^53), some in place; outputs bit-exact."""
    rng = np.random.default_rng(11)
    arrs = [datagen.generate("C2", 2_000_000), np.zeros(0), np.array([2.5]),
            datagen.generate("C3", 3_000_001), rng.normal(size=100_000),
            np.repeat(rng.normal(size=1000), 1000)]
    ins = [torch.from_numpy(x.copy()).pin_memory() for x in arrs]
    outs = [torch.empty(x.size, dtype=torch.float64).pin_memory() for x in arrs]
    outs[2] = ins[2]  # in place
    outs[4] = ins[4]
    ipls.sort_host_batch([t.data_ptr() for t in ins], [t.data_ptr() for t in outs],
                         [x.size for x in arrs], ipls.KEY_F64, k=1024, base_case=4096)
    for x, o in zip(arrs, outs):
        assert o.numpy().tobytes() == np.sort(x).tobytes()
    u = rng.integers(0, 2**64 - 1, 500_000, dtype=np.uint64, endpoint=True)
    hu = [torch.from_numpy(u.view(np.int64).copy()).pin_memory() for _ in range(3)]
    ipls.sort_host_batch([t.data_ptr() for t in hu], [t.data_ptr() for t in hu], [u.size] * 3,
                         ipls.KEY_U64, k=1024, base_case=4096)
    for t in hu:
        assert t.numpy().view(np.uint64).tobytes() == np.sort(u).tobytes()
    bad = datagen.generate("C2", 100_000)
    bad[777] = np.nan
    hb = torch.from_numpy(bad).pin_memory()
    with pytest.raises(ipls.IPLSError) as e:
        ipls.sort_host_batch([hb.data_ptr()], [hb.data_ptr()], [bad.size], ipls.KEY_F64,
                             k=1024, base_case=4096)
    assert e.value.status == 2
    with pytest.raises(ipls.IPLSError):
        ipls.sort_host_batch([0], [0], [5], ipls.KEY_F64)


def test_caller_workspace(ipls):
    a = datagen.generate("C3", 1_000_000)
    want = np.sort(a)
    t = dev(a)
    wb = ipls.workspace_bytes(a.size, ipls.KEY_F64, k=1024, base_case=4096)
    ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
    ipls.sort(t, k=1024, base_case=4096, key_type=0, workspace=ws)
    assert host(t, np.float64).tobytes() == want.tobytes()
    small = torch.empty(1024, dtype=torch.uint8, device="cuda")
    t2 = dev(a)
    with pytest.raises(ipls.IPLSError) as e:
        ipls.sort(t2, k=1024, base_case=4096, key_type=0, workspace=small)
    assert e.value.status == 4


def test_deterministic_repeat(ipls):
    a = datagen.generate("C5", 2_000_000)
    t1, t2 = dev(a), dev(a)
    r1 = ipls.sort_trace(t1, k=1024, base_case=4096, key_type=0)
    r2 = ipls.sort_trace(t2, k=1024, base_case=4096, key_type=0)
    assert torch.equal(t1, t2)
    assert gpu_digests(r1.records) == gpu_digests(r2.records)


def test_concurrent_streams_threads(ipls):
    """ipls.h: concurrent calls on different streams are safe (one workspace per stream)."""
    import threading
    arrays = [datagen.generate(name, 1_500_000) for name in ("C2", "C3", "C4", "C5")]
    wants = []
    for a in arrays:
        w = a.copy()
        cfg = datagen.CONFIGS["C2"]
        assert oracle.sort(w, k=cfg.k, base_case=cfg.base_case).status == 0
        wants.append(w)
    ts = [dev(a) for a in arrays]
    streams = [torch.cuda.Stream() for _ in arrays]
    errs = []

    def run(i):
        try:
            with torch.cuda.stream(streams[i]):
                for _ in range(3):
                    x = dev(arrays[i])
                    ipls.sort(x, k=1024, base_case=4096, key_type=kt_of(arrays[i]),
                              stream=streams[i])
                    ts[i] = x
            streams[i].synchronize()
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(arrays))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for t, w, a in zip(ts, wants, arrays):
        assert host(t, a.dtype).tobytes() == w.tobytes()


@pytest.mark.parametrize("tag", [0x3FF0, 0xBFF0])
def test_stale_status_words_cannot_pass_the_epoch_check(ipls, tag):
    """Regression: a level's lookback status words overlap what earlier levels stored in the
    same metadata (first keys of homogeneous buckets, prefixes).  A stale key whose top 16 bits
    equal the level's epoch tag (and whose bits 46-47 are set) looked like a valid status word,
    giving wrong prefixes (wrong output, illegal addresses; tools/epoch_collision.py).  The
    status region is now cleared every level; epochs are forced onto the keys' tag here."""
    rng = np.random.default_rng(tag)
    base = np.uint64(tag) << np.uint64(48)
    vals = (base | (np.uint64(3) << np.uint64(46)) |
            rng.integers(0, 1 << 20, 40).astype(np.uint64)).view(np.float64)
    a = np.concatenate([vals[rng.integers(0, vals.size, 3_000_000)], rng.normal(0, 1, 1_000_000)])
    rng.shuffle(a)
    want = np.sort(a)
    for e0 in range(tag - 3, tag + 1):
        ipls.lib().ipls_debug_set_epoch(e0)
        t = dev(a)
        ipls.sort(t, k=1024, base_case=4096, key_type=0)
        assert host(t, np.float64).tobytes() == want.tobytes(), f"epoch {e0:#x}"


@pytest.mark.parametrize("kind", ["normal", "dups", "presorted"])
def test_match_rank_path_keeps_stable_layouts(ipls, kind):
    """The stable scatter ranks keys by shared-memory atomics, whose same-address lanes B200
    serves in lane order; every CTA probes that and otherwise ranks with match.any peer masks
    (K3).  The probe has never failed on B200, so the fallback is forced here
    (ipls_debug_force_match_rank): layouts after every level, models and the final array must
    stay bit-exact with the oracle."""
    rng = np.random.default_rng(len(kind))
    n = 700_001
    if kind == "normal":
        a = rng.normal(0, 1, n)
    elif kind == "dups":
        a = rng.integers(0, 300, n).astype(np.float64)
    else:
        a = np.sort(rng.lognormal(0, 2, n))
    ipls.lib().ipls_debug_force_match_rank(1)
    try:
        sort_parity_with_layouts(ipls, a, 256, 4096)
        sort_parity_with_layouts(ipls, a, 1024, 1000)
    finally:
        ipls.lib().ipls_debug_force_match_rank(0)


@pytest.mark.parametrize("n,k", [(100_000, 256), (1_000_000, 1024)])
def test_no_progress_guard_fires_and_matches_oracle(ipls, n, k):
    """The no-progress guard (R10): a model that keeps all m keys of a segment in one bucket
    re-queues the segment with a forced equality split.  With FMCD it cannot fire on a
    segment's own sample (the anchors s[D] and s[N-1-D] land k-2 buckets apart, DESIGN.md
    R10), but IPS4o's splitter tree can: on a one-valued root every splitter equals the key,
    every key descends to leaf 0.  The GPU must re-queue exactly as the oracle does."""
    a = np.full(n, 3.25)
    want = a.copy()
    ores = oracle.sort(want, k=k, base_case=4096, trace=True, model=oracle.MODEL_TREE)
    t = dev(a)
    gtr = ipls.sort_trace(t, k=k, base_case=4096, key_type=0, model=ipls.MODEL_TREE)
    assert host(t, np.float64).tobytes() == want.tobytes()
    compare_traces(gtr, ores)
    assert any(r.requeued for r in gtr.records)
    assert any(r.level == 1 and r.kind == ipls.MODEL_EQ3 for r in gtr.records)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_configs_full_size_layout_after_every_level(ipls, name):
    """Full BASELINE sizes: the array image after every level against the oracle's
    (tests/golden/oracle_layouts.txt, written by make_oracle_layouts.py from the oracle only),
    element by element outside the children of terminal segments and as a multiset inside
    each of them (their interior order is unspecified, R11)."""
    import sys
    sys.path.insert(0, GOLD)
    from make_oracle_layouts import free_ranges, layout_digest
    want = {}
    with open(os.path.join(GOLD, "oracle_layouts.txt")) as f:
        for line in f:
            tok = line.split()
            if tok and tok[0] == "LAYOUT":
                want.setdefault(tok[1], {})[int(tok[2])] = tok[3]
    cfg = datagen.CONFIGS[name]
    a = datagen.generate(name)
    t = dev(a)
    del a
    levels = len(want[name])
    gtr = ipls.sort_trace(t, k=cfg.k, base_case=cfg.base_case,
                          key_type=kt_of(datagen.generate(name, 1)), snapshot_levels=levels)
    assert gtr.levels == levels
    for lv in range(levels):
        img = gtr.snapshots[lv].cpu().numpy().view(np.uint64)
        lo, hi = free_ranges(gtr.records, lv, cfg.base_case)
        assert layout_digest(img, lo, hi) == want[name][lv], f"{name}: layout after level {lv}"
    del gtr
    torch.cuda.empty_cache()


@pytest.fixture(params=[1, 2, 3], ids=["fused", "separate", "windows"])
def term_mode(ipls, request):
    ipls.lib().ipls_debug_term_mode(request.param)
    yield request.param
    ipls.lib().ipls_debug_term_mode(0)


@pytest.mark.parametrize("kind", ["normal", "lognormal", "few_distinct", "mixture", "u64_above_2_53"])
@pytest.mark.parametrize("n,k,B", [(70_001, 256, 4096), (300_000, 1024, 4096), (200_000, 64, 100)])
def test_terminal_paths_parity(ipls, term_mode, kind, n, k, B):
    """Both ways of processing a level's terminal segments -- the last level fused with the
    base case (k_term_fused) and the separate terminal scatter + base-case
    kernels -- give the oracle's records and layouts after every level and its final array
    (the size rule that picks one in production is overridden here)."""
    rng = np.random.default_rng(n + k + len(kind))
    a = datagen.fuzz_array(rng, n, kind)
    sort_parity_with_layouts(ipls, a, k, B)


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_terminal_paths_configs_scaled(ipls, term_mode, name):
    a = datagen.generate(name, 3_000_000)
    cfg = datagen.CONFIGS[name]
    want = a.copy()
    ores = oracle.sort(want, k=cfg.k, base_case=cfg.base_case, trace=True)
    t = dev(a)
    gtr = ipls.sort_trace(t, k=cfg.k, base_case=cfg.base_case, key_type=kt_of(a))
    assert host(t, a.dtype).tobytes() == want.tobytes()
    compare_traces(gtr, ores)
