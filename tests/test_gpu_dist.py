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
