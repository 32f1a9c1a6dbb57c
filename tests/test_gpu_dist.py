"""GPU parity of the distributed top level's kernels.

* `ipls_sample_strata` on simulated shards (one GPU, shards of one array; each call is an
  independent kernel, no rank waits on another): the shards' slots summed are the oracle's
  level-0 sample of the whole array (`oracle.sample_positions`, R2/R18) bit for bit, and the
  sample the one-GPU sort records at level 0.
* `dist_sort` in a real one-rank NCCL group: output = the sorted input; the shared model and
  the global counts equal the oracle's level-0 record.  (The N-rank orchestration is covered
  over gloo by tests/test_dist_sort.py; this box has one GPU.)
"""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2208_06902_b200 import datagen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ipls():
    import paper_2208_06902_b200 as m
    assert torch.cuda.is_available()
    m.lib()
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64).copy()).cuda()


@pytest.mark.parametrize("G", [1, 2, 3, 8])
@pytest.mark.parametrize("n,k", [(100, 4), (70001, 256), (3_000_000, 1024)])
def test_sample_strata_shards_sum_to_oracle_sample(ipls, G, n, k):
    rng = np.random.default_rng(n + G)
    a = datagen.fuzz_array(rng, n, "lognormal")
    cuts = np.sort(rng.integers(0, n + 1, G - 1))
    if G > 2:
        cuts[1] = cuts[0]  # an empty shard
    S = ipls.sample_size(n, k)
    tot = torch.zeros(S, dtype=torch.int64, device="cuda")
    begin = 0
    for sh in np.split(a, cuts):
        part = torch.zeros(S, dtype=torch.int64, device="cuda")
        ipls.sample_strata(dev(sh), begin, n, S, part)
        tot += part
        begin += sh.size
    pos = oracle.sample_positions(ipls.DEFAULT_SEED, 0, 0, n, S).astype(np.int64)
    assert np.array_equal(tot.cpu().numpy().view(np.uint64), a.view(np.uint64)[pos])
    if n > 4096:  # the one-GPU sort partitions the root and records its sorted sample
        tr = ipls.sort_trace(dev(a), k=k, base_case=4096, key_type=0)
        smp = a[pos]
        smp = smp[np.argsort(oracle.ordering_keys(smp), kind="stable")]
        assert np.array_equal(tr.records[0].sample, smp.view(np.uint64))


def test_sample_strata_rejects_bad_ranges(ipls):
    t = torch.zeros(10, dtype=torch.int64, device="cuda")
    out = torch.zeros(16, dtype=torch.int64, device="cuda")
    with pytest.raises(ipls.IPLSError):
        ipls.sample_strata(t, 5, 12, 4, out)    # [5, 15) outside [0, 12)
    with pytest.raises(ipls.IPLSError):
        ipls.sample_strata(t, 0, 10, 11, out)   # S > m


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl1():
    import torch.distributed as dist
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(_free_port())})
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,n", [("normal", 2_000_000), ("lognormal", 300_000),
                                    ("few_distinct", 500_000), ("u64_above_2_53", 400_000),
                                    ("all_equal", 100_000), ("uniform", 5)])
def test_dist_sort_one_rank_nccl(ipls, nccl1, kind, n):
    from paper_2208_06902_b200.distributed import dist_sort
    a = datagen.fuzz_array(np.random.default_rng(n), n, kind)
    src = dev(a)
    if a.dtype == np.float64:
        src = src.view(torch.float64)
    before = src.clone()
    res = dist_sort(src, k=1024, base_case=4096)
    assert torch.equal(src, before)  # the shard is left unmodified
    want = a[np.argsort(oracle.ordering_keys(a), kind="stable")]
    assert res.keys.cpu().numpy().tobytes() == want.tobytes()
    assert res.bounds == [0, len(res.counts)] and res.global_begin == 0 and res.global_n == n
    if n >= 8:
        ref = oracle.sort(a.copy(), k=1024, base_case=4096, trace=True)
        r0 = ref.records[0]
        assert np.array_equal(res.counts.astype(np.uint64), r0.counts)
        m = res.model
        if r0.kind == oracle.MODEL_LINEAR:
            assert (m.kind, m.a, m.b, m.D) == (ipls.MODEL_LINEAR, r0.A, r0.B, r0.D)
        else:
            assert m.kind == ipls.MODEL_EQ3 and m.pivot_ok == r0.pivot_ok


@pytest.mark.parametrize("kind,n", [("normal", 2_000_000), ("lognormal", 300_000),
                                    ("few_distinct", 500_000), ("u64_above_2_53", 400_000),
                                    ("all_equal", 100_000), ("uniform", 5)])
def test_dist_sort_fused_one_rank_nccl(ipls, nccl1, kind, n):
    """The fused exchange in a real one-rank NCCL group: the receive buffer is torch symmetric
    memory and the scatter stores into it through the address the rendezvous returns."""
    from paper_2208_06902_b200.distributed import dist_sort
    a = datagen.fuzz_array(np.random.default_rng(n), n, kind)
    src = dev(a)
    if a.dtype == np.float64:
        src = src.view(torch.float64)
    before = src.clone()
    res = dist_sort(src, k=1024, base_case=4096, fused=True)
    assert torch.equal(src, before)
    want = a[np.argsort(oracle.ordering_keys(a), kind="stable")]
    assert res.keys.cpu().numpy().tobytes() == want.tobytes()
    ref = dist_sort(src, k=1024, base_case=4096, fused=False)
    assert torch.equal(ref.keys.view(torch.int64), res.keys.view(torch.int64))
    assert ref.bounds == res.bounds and ref.cuts == res.cuts


def test_dist_sort_fused_reused_buffers(ipls, nccl1):
    """SymmPeers(reuse=True): the receive buffer is kept while it is large enough and replaced
    when it is not; every call's result is right while it is the latest."""
    from paper_2208_06902_b200.distributed import SymmPeers, dist_sort
    peers = SymmPeers(reuse=True)
    rng = np.random.default_rng(5)
    ptrs = []
    for n in (200_000, 150_000, 900_000, 899_999):
        a = rng.normal(0, 1, n)
        res = dist_sort(dev(a).view(torch.float64), k=1024, base_case=4096, peers=peers)
        assert res.keys.cpu().numpy().tobytes() == np.sort(a).tobytes()
        ptrs.append(peers.buf.data_ptr())
        assert res.keys.data_ptr() == peers.buf.data_ptr()
    assert ptrs[0] == ptrs[1] and ptrs[2] == ptrs[3] and ptrs[1] != ptrs[2]


def _model_of(ipls, r0, k):
    if r0.kind == oracle.MODEL_LINEAR:
        return ipls.Model(r0.A, r0.B, k, r0.D, ipls.MODEL_LINEAR, int(r0.capped), 0, False)
    return ipls.Model(0.0, 0.0, 3, 0, ipls.MODEL_EQ3, 0, int(r0.pivot_ok), True)


@pytest.mark.parametrize("G", [1, 2, 3, 8])
@pytest.mark.parametrize("kind,n,k", [("normal", 3_000_000, 1024), ("lognormal", 70_001, 256),
                                      ("u64_above_2_53", 400_000, 1024),
                                      ("few_distinct", 200_000, 64), ("all_equal", 50_000, 256),
                                      ("normal", 5000, 16)])
def test_partition_count_and_scatter_to_simulated_ranks(ipls, G, kind, n, k):
    """ipls_partition_count + ipls_partition_scatter_to on the shards of one array (one GPU,
    one independent call per simulated rank, the G receive buffers being local tensors): every
    shard's offsets are the oracle's stable partition's, and the receive buffers, concatenated
    in rank order, are the oracle's stable partition of the WHOLE array by the top-level
    model (the bytes partition + all-to-all + regroup deliver), bit for bit."""
    from paper_2208_06902_b200.distributed import fused_plan
    rng = np.random.default_rng(n + G + k)
    a = datagen.fuzz_array(rng, n, kind)
    r0 = oracle.sort(a.copy(), k=k, base_case=64, trace=True).records[0]
    m = _model_of(ipls, r0, k)
    kt = 0 if a.dtype == np.float64 else 1
    cuts = np.sort(rng.integers(0, n + 1, G - 1))
    if G > 2:
        cuts[1] = cuts[0]  # an empty shard
    shards = np.split(a, cuts)
    tsh = [dev(sh) for sh in shards]
    cnt = []
    for sh, t in zip(shards, tsh):
        off = ipls.partition_count(t, m, key_type=kt).cpu().numpy()
        _, want_off, _ = oracle.partition(sh, m.a, m.b, m.k, m.kind, m.pivot_ok)
        assert np.array_equal(off.astype(np.uint64), np.asarray(want_off, dtype=np.uint64))
        cnt.append(np.diff(off))
    cnt = np.array(cnt)
    _, bounds, owner, offset, recv = fused_plan(cnt, G)
    bufs = [torch.full((max(1, recv[d]),), -1, dtype=torch.int64, device="cuda") for d in range(G)]
    for s, t in enumerate(tsh):
        before = t.clone()
        addr = torch.tensor([bufs[int(owner[b])].data_ptr() + 8 * int(offset[s, b])
                             for b in range(cnt.shape[1])], dtype=torch.int64, device="cuda")
        ipls.partition_scatter_to(t, m, addr, key_type=kt)
        assert torch.equal(t, before)  # the source shard is left unmodified
    got = np.concatenate([bufs[d][:recv[d]].cpu().numpy() for d in range(G)])
    want, _, _ = oracle.partition(a, m.a, m.b, m.k, m.kind, m.pivot_ok)
    assert got.tobytes() == want.tobytes()
    assert np.array_equal(cnt.sum(axis=0).astype(np.uint64), r0.counts)


def test_fused_exchange_full_size_c2(ipls):
    """C2 at full size (1e8 keys) cut into 8 even shards, as bench.py --gpus 8 shards it: the
    eight receive buffers filled by ipls_partition_scatter_to are, concatenated, the oracle's
    stable partition of the whole array by the oracle's level-0 model (SHA-256 of the bytes),
    and the plan's ranges are the buckets' global prefix sums."""
    import hashlib
    from paper_2208_06902_b200.distributed import fused_plan
    G = 8
    cfg = datagen.CONFIGS["C2"]
    a = datagen.generate("C2")
    n = a.size
    S = oracle.sample_size(n, cfg.k)
    pos = oracle.sample_positions(ipls.DEFAULT_SEED, 0, 0, n, S).astype(np.int64)
    smp = np.sort(a[pos])
    f = oracle.fit_fmcd(smp, cfg.k)
    assert not f.degenerate
    m = ipls.Model(f.A, f.B, cfg.k, f.D, ipls.MODEL_LINEAR, int(f.capped), 0, False)
    want, want_off, _ = oracle.partition(a, m.a, m.b, m.k, m.kind, 0)
    want_sha = hashlib.sha256(want.tobytes()).hexdigest()
    del want
    tsh = [dev(a[n * r // G: n * (r + 1) // G]) for r in range(G)]
    del a
    cnt = np.array([np.diff(ipls.partition_count(t, m, key_type=0).cpu().numpy()) for t in tsh])
    assert np.array_equal(np.concatenate([[0], np.cumsum(cnt.sum(axis=0))]).astype(np.uint64),
                          np.asarray(want_off, dtype=np.uint64))
    cuts, bounds, owner, offset, recv = fused_plan(cnt, G)
    assert sum(recv) == n and max(recv) < 1.2 * n / G   # C2's buckets balance the ranks
    bufs = [torch.empty(recv[d], dtype=torch.int64, device="cuda") for d in range(G)]
    base = np.array([bufs[int(owner[b])].data_ptr() for b in range(cfg.k)], dtype=np.int64)
    for s, t in enumerate(tsh):
        addr = torch.from_numpy(base + 8 * offset[s]).cuda()
        ipls.partition_scatter_to(t, m, addr, key_type=0)
    h = hashlib.sha256()
    for d in range(G):
        h.update(bufs[d].cpu().numpy().tobytes())
    assert h.hexdigest() == want_sha


def test_partition_scatter_to_rejects_bad_arguments(ipls):
    t = dev(np.random.default_rng(0).random(1000))
    m = ipls.Model(1.0, 0.0, 8, 1, ipls.MODEL_LINEAR, 0, 0, False)
    with pytest.raises(ValueError):
        ipls.partition_scatter_to(t, m, torch.zeros(4, dtype=torch.int64, device="cuda"))
    assert ipls.lib().ipls_partition_scatter_to(t.data_ptr(), 1000, 0, None, None, None) == 1
    assert ipls.lib().ipls_partition_count(t.data_ptr(), 1000, 0, None, None, None) == 1


def test_dist_sort_nan_raises(ipls, nccl1):
    from paper_2208_06902_b200.distributed import dist_sort
    a = np.random.default_rng(0).normal(size=50000)
    a[31337] = np.nan
    with pytest.raises(ipls.IPLSError) as e:
        dist_sort(dev(a).view(torch.float64))
    assert e.value.status == 2


@pytest.mark.parametrize("S,k,kind", [(6143, 1024, "normal"), (4095, 256, "lognormal"),
                                      (100, 10, "few_distinct"), (5119, 1024, "all_equal"),
                                      (8192, 1024, "u64_above_2_53")])
def test_fit_sample_unsorted_equals_oracle_fit(ipls, S, k, kind):
    """ipls_fit_sample sorts the given sample in the fit kernel: same model as the oracle's
    Listing 1 on the sorted sample (degenerate -> EQ3 with the sorted sample's median)."""
    a = datagen.fuzz_array(np.random.default_rng(S + k), S, kind)
    m = ipls.fit_fmcd(dev(a), k, key_type=0 if a.dtype == np.float64 else 1, presorted=False)
    s = a[np.argsort(oracle.ordering_keys(a), kind="stable")]
    f = oracle.fit_fmcd(s.astype(np.float64), k)
    if f.degenerate:
        assert m.degenerate and m.kind == ipls.MODEL_EQ3
        assert m.pivot_ok == int(oracle.ordering_keys(s[S // 2:S // 2 + 1])[0])
    else:
        assert (m.a, m.b, m.D, bool(m.capped)) == (f.A, f.B, f.D, f.capped)


# ---------------------------------------------------------------- local sort after exchange --
def _ok_sorted(a):
    return a[np.argsort(oracle.ordering_keys(a), kind="stable")]


@pytest.mark.parametrize("G,nb", [(1, 5), (2, 1), (3, 7), (5, 64)])
def test_regroup_runs_is_bucket_major(ipls, G, nb):
    rng = np.random.default_rng(G * 100 + nb)
    counts = rng.integers(0, 50, (G, nb)).astype(np.uint64)
    counts[0, 0] = 0
    tot = int(counts.sum())
    src = rng.integers(0, 2 ** 63, tot).astype(np.int64)
    want, pieces, o = [], [[] for _ in range(nb)], 0
    for g in range(G):
        for b in range(nb):
            c = int(counts[g, b])
            pieces[b].append(src[o:o + c])
            o += c
    want = np.concatenate([x for p in pieces for x in p]) if tot else src
    s = torch.from_numpy(src).cuda()
    d = torch.empty_like(s)
    ipls.regroup_runs(s, d, counts)
    assert np.array_equal(d.cpu().numpy(), want)


@pytest.mark.parametrize("name,n", [("C2", 3_000_000), ("C3", 2_000_000), ("C4", 1_000_000)])
def test_sort_segments_resumes_the_one_gpu_sort(ipls, name, n):
    """ipls_sort_segments on the stable level-0 partition of an array, with the level-0 buckets
    as segments, performs exactly the levels >= 1 of the one-GPU sort: every record of the
    resumed sort equals the oracle's record of the same (level, begin), and the output is the
    sorted input (the multi-GPU local sort)."""
    cfg = datagen.CONFIGS[name]
    a = datagen.generate(name, n)
    ores = oracle.sort(a.copy(), k=cfg.k, base_case=cfg.base_case, trace=True)
    r0 = ores.records[0]
    assert r0.level == 0
    kt = 0 if a.dtype == np.float64 else 1
    mdl = ipls.Model(r0.A, r0.B, r0.k_eff, r0.D, r0.kind, r0.capped, r0.pivot_ok)
    part = torch.empty(n, dtype=torch.int64, device="cuda")
    off, _ = ipls.partition_level(dev(a), part, mdl, key_type=kt)
    sizes = np.diff(off.cpu().numpy().astype(np.int64))
    tr = ipls.sort_trace(part, k=cfg.k, base_case=cfg.base_case, key_type=kt,
                         segments=sizes, level=1)
    assert part.cpu().numpy().view(a.dtype).tobytes() == _ok_sorted(a).tobytes()
    # the oracle's records below level 0, except children it classed homogeneous-final (the
    # resumed sort cannot know they are one-valued and partitions them once more, EQ3)
    want = {(o.level, o.begin): o for o in ores.records if o.level >= 1}
    got = {(g.level, g.begin): g for g in tr.records}
    for key, o in want.items():
        g = got[key]
        assert (g.m, g.S, g.kind, g.D, g.capped, g.pivot_ok) == (o.m, o.S, o.kind, o.D, o.capped, o.pivot_ok)
        assert g.A == o.A and g.B == o.B
        assert np.array_equal(g.counts, o.counts)
    for key, g in got.items():
        if key not in want:  # only one-valued segments may be extra
            assert g.kind == ipls.MODEL_EQ3 and g.counts[1] == g.m


@pytest.mark.parametrize("kind", ["normal", "dups", "small_segments", "u64"])
def test_sort_segments_edge_cases(ipls, kind):
    rng = np.random.default_rng(len(kind))
    n = 400_000
    if kind == "u64":
        a = np.sort(rng.integers(0, 2 ** 64 - 1, n, dtype=np.uint64, endpoint=True))
    elif kind == "dups":
        a = np.sort(rng.integers(0, 20, n).astype(np.float64))
    else:
        a = np.sort(rng.normal(0, 1, n))
    if kind == "small_segments":
        cuts = np.sort(rng.integers(0, n, 3000))  # mostly base-case segments, zeros included
    else:
        cuts = np.sort(rng.integers(0, n, 40))
    cuts = np.concatenate([[0], cuts, cuts[:3], [n]])
    cuts.sort()
    sizes = np.diff(cuts)
    b = a.copy()
    for lo, hi in zip(cuts[:-1], cuts[1:]):  # shuffle inside each range-ordered segment
        rng.shuffle(b[lo:hi])
    t = dev(b)
    ipls.sort_segments(t, sizes, level=1, k=256, base_case=4096,
                       key_type=1 if kind == "u64" else 0)
    assert t.cpu().numpy().view(a.dtype).tobytes() == a.tobytes()


def test_sort_segments_nan_leaves_array_unmodified(ipls):
    a = np.sort(np.random.default_rng(5).normal(0, 1, 100_000))
    a[77_777] = np.nan
    t = dev(a)
    with pytest.raises(ipls.IPLSError) as e:
        ipls.sort_segments(t, [50_000, 50_000], level=1, k=1024, base_case=4096, key_type=0)
    assert e.value.status == 2
    assert t.cpu().numpy().tobytes() == a.tobytes()


@pytest.mark.parametrize("G", [2, 3, 8])
def test_simulated_ranks_data_path(ipls, G):
    """The N-rank data path of dist_sort on one GPU (no rank waits on another): the global
    level-0 model, every shard's stable partition, the exchange as slicing, regroup and the
    resumed local sorts with the rank's global position as hash base; the concatenation is the
    sorted input, and every record below level 0 on every rank is the one-GPU sort's record of
    the same (level, global begin)."""
    a = datagen.generate("C5", 2_000_000)
    n = a.size
    cfg = datagen.CONFIGS["C5"]
    ores = oracle.sort(a.copy(), k=cfg.k, base_case=cfg.base_case, trace=True)
    r0 = ores.records[0]
    mdl = ipls.Model(r0.A, r0.B, r0.k_eff, r0.D, r0.kind, r0.capped, r0.pivot_ok)
    shards = np.array_split(a, G)
    parts, offs = [], []
    for sh in shards:
        p = torch.empty(sh.size, dtype=torch.int64, device="cuda")
        off, _ = ipls.partition_level(dev(sh), p, mdl, key_type=0)
        parts.append(p)
        offs.append(off.cpu().numpy().astype(np.int64))
    cnt = np.stack([np.diff(o) for o in offs])
    bounds = ipls.assign_ranges(cnt.sum(axis=0), G)
    pre = np.concatenate([[0], np.cumsum(cnt.sum(axis=0))])
    want = {(o.level, o.begin): o for o in ores.records if o.level >= 1}
    out, seen = [], 0
    for r in range(G):
        b0, b1 = bounds[r], bounds[r + 1]
        runs = torch.cat([parts[s][int(offs[s][b0]):int(offs[s][b1])] for s in range(G)])
        mine = cnt[:, b0:b1].astype(np.uint64)
        reg = torch.empty_like(runs)
        if runs.numel():
            ipls.regroup_runs(runs, reg, mine)
            tr = ipls.sort_trace(reg, k=cfg.k, base_case=cfg.base_case, key_type=0,
                                 segments=mine.sum(axis=0), level=1, global_begin=int(pre[b0]))
            for g in tr.records:
                o = want.get((g.level, g.begin + int(pre[b0])))
                if o is None:  # only one-valued segments may be extra (see above)
                    assert g.kind == ipls.MODEL_EQ3 and g.counts[1] == g.m
                    continue
                seen += 1
                assert (g.m, g.S, g.kind, g.D, g.capped, g.pivot_ok) == \
                    (o.m, o.S, o.kind, o.D, o.capped, o.pivot_ok)
                assert g.A == o.A and g.B == o.B
                assert np.array_equal(g.counts, o.counts)
                assert np.array_equal(g.sample, o.sample)
        out.append(reg.cpu().numpy())
    got = np.concatenate(out).view(np.float64)
    assert got.tobytes() == _ok_sorted(a).tobytes()
    assert seen == len(want)  # every one-GPU record below level 0 was reproduced
