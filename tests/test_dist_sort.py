"""Distributed top level (paper_2208_06902_b200/distributed.py) over
gloo with 2 and 3 CPU processes.

The orchestration (sizes, sample all-reduce, count all-gather, `ipls_assign_ranges`, the
all-to-all and the status agreement) is the product code; the per-rank compute steps are
the oracle's (tests may use it; on GPUs `CudaOps` calls libipls.so).  Pins:

* the concatenation of the ranks' outputs is the input sorted by ordering key;
* the shared top-level model and the global bucket counts equal the oracle's level-0 record
  of a one-process sort of the concatenated array (same strata, R2/R18), so the exchange
  partitions the global array exactly as level 0 of the single-GPU method would;
* every rank's range is the contiguous bucket range `assign_ranges` gave it;
* a NaN anywhere raises on every rank.
Also the host function `ipls_assign_ranges` against brute force.
"""
import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2208_06902_b200 as ipls  # noqa: E402
from paper_2208_06902_b200 import datagen  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleOps:
    """The per-rank compute steps done by the CPU oracle on CPU tensors (test stand-in)."""

    @staticmethod
    def _np(t, kt):
        a = t.numpy().view(np.uint64)
        return a.view(np.float64) if kt == ipls.KEY_F64 else a

    def sample(self, keys, gbegin, gm, S, seed):
        pos = oracle.sample_positions(seed, 0, 0, gm, S).astype(np.int64)
        out = torch.zeros(S, dtype=torch.int64)
        own = (pos >= gbegin) & (pos < gbegin + keys.numel())
        bits = keys.view(torch.int64)
        out[torch.from_numpy(np.nonzero(own)[0])] = bits[torch.from_numpy(pos[own] - gbegin)]
        return out

    def sort(self, t, kt, k, base_case, seed):
        a = self._np(t, kt).copy()
        r = oracle.sort(a, k=k, base_case=base_case, seed=seed)
        if r.status == 0:
            t.view(torch.int64).copy_(torch.from_numpy(a.view(np.int64)))
        return r.status

    def fit(self, s, kt, k):
        a = self._np(s, kt)
        a = a[np.argsort(oracle.ordering_keys(a), kind="stable")]  # the sample arrives unsorted
        f = oracle.fit_fmcd(a.astype(np.float64), k)
        if f.degenerate:
            piv = int(oracle.ordering_keys(a[a.size // 2: a.size // 2 + 1])[0])
            return ipls.Model(0.0, 0.0, 3, 0, ipls.MODEL_EQ3, 0, piv, True)
        return ipls.Model(f.A, f.B, k, f.D, ipls.MODEL_LINEAR, int(f.capped), 0, False)

    def partition(self, keys, m, kt):
        a = self._np(keys, kt)
        out, off, _ = oracle.partition(a, m.a, m.b, m.k, m.kind, m.pivot_ok)
        return torch.from_numpy(out.view(np.int64).copy()), [int(x) for x in off]

    peers = None  # fused exchange: the ShmPeers whose views stand for peer memory

    def partition_count(self, keys, m, kt):
        a = self._np(keys, kt)
        _, off, _ = oracle.partition(a, m.a, m.b, m.k, m.kind, m.pivot_ok)
        return [int(x) for x in off]

    def scatter_to(self, keys, m, kt, addresses):
        """Stable partition by the oracle, every bucket copied to its "address" (ShmPeers:
        rank << 44 | byte offset in that rank's shared-memory buffer)."""
        a = self._np(keys, kt)
        out, off, _ = oracle.partition(a, m.a, m.b, m.k, m.kind, m.pivot_ok)
        bits = out.view(np.int64)
        for b, ad in enumerate(addresses):
            c = int(off[b + 1] - off[b])
            if c:
                d, o = ad >> 44, (ad & ((1 << 44) - 1)) // 8
                self.peers.views[d][o:o + c] = bits[int(off[b]):int(off[b + 1])]
        return 0

    def regroup(self, runs, counts):
        """Bucket-major order of the G received runs (the reference for ipls_regroup_runs)."""
        bits = runs.view(torch.int64).numpy()
        pieces, o = [[] for _ in range(counts.shape[1])], 0
        for g in range(counts.shape[0]):
            for b in range(counts.shape[1]):
                c = int(counts[g, b])
                pieces[b].append(bits[o:o + c])
                o += c
        flat = [x for p in pieces for x in p]
        out = np.concatenate(flat) if flat else bits[:0]
        return torch.from_numpy(out.copy()).view(runs.dtype)

    def sort_segments(self, t, kt, k, base_case, seed, sizes, level, global_begin=0):
        # the segments are range-ordered: sorting the whole range sorts each of them
        assert int(np.sum(sizes)) == t.numel()
        return self.sort(t, kt, k, base_case, seed)


class ShmPeers:
    """Test stand-in for SymmPeers: every rank's receive buffer is a named POSIX shared-memory
    block the other processes attach to; an "address" is rank << 44 | byte offset."""

    def __init__(self, tag, rank, world):
        self.tag, self.rank, self.world = tag, rank, world
        self.shms, self.views = [], []

    def alloc(self, nelems, device):
        import torch.distributed as dist
        from multiprocessing import shared_memory
        n = max(1, nelems)
        own = shared_memory.SharedMemory(create=True, size=8 * n, name=f"{self.tag}_{self.rank}")
        dist.barrier()
        for d in range(self.world):
            shm = own if d == self.rank else shared_memory.SharedMemory(name=f"{self.tag}_{d}")
            self.shms.append(shm)
            self.views.append(np.ndarray((n,), np.int64, buffer=shm.buf))
        self.views[self.rank][:] = -1
        return torch.from_numpy(self.views[self.rank]), [d << 44 for d in range(self.world)]

    def barrier(self):
        import torch.distributed as dist
        dist.barrier()

    def close(self):
        import torch.distributed as dist
        self.views = []
        dist.barrier()
        for d, shm in enumerate(self.shms):
            try:
                shm.close()
            except BufferError:
                pass
            if d == self.rank:
                shm.unlink()


def _shards(kind, n, G, seed):
    rng = np.random.default_rng(seed)
    a = datagen.fuzz_array(rng, n, "normal" if kind == "nan_one" else kind)
    if kind == "nan_one":
        a[(2 * n) // 3] = np.nan  # not a sampled position's concern: any NaN must raise
    cuts = np.sort(rng.integers(0, n + 1, G - 1))
    if G > 2:
        cuts[0] = cuts[1]  # one empty shard
    return a, np.split(a, cuts)


def _worker(rank, world, port, q, kind, n, k, B, seed, fused=False):
    os.environ.update({"MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    import torch.distributed as dist
    from paper_2208_06902_b200.distributed import dist_sort
    dist.init_process_group("gloo", rank=rank, world_size=world)
    peers = ShmPeers(f"ipls{port}", rank, world) if fused else None
    try:
        _, shards = _shards(kind, n, world, seed)
        mine = torch.from_numpy(shards[rank].view(np.int64).copy())
        kt = ipls.KEY_F64 if shards[rank].dtype == np.float64 else ipls.KEY_U64
        ops = OracleOps()
        ops.peers = peers
        try:
            res = dist_sort(mine, k=k, base_case=B, key_type=kt, ops=ops, fused=fused,
                            peers=peers)
            m = res.model
            q.put((rank, "ok", res.keys.numpy().copy(), res.bounds, res.counts,
                   None if m is None else (m.a, m.b, m.D, m.kind, m.pivot_ok),
                   res.global_begin, res.global_n))
        except ipls.IPLSError as e:
            q.put((rank, "err", e.status))
        if peers is not None and peers.shms:
            del res
            peers.close()
    finally:
        dist.destroy_process_group()


def _run(world, kind, n, k=64, B=64, seed=3, fused=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q, kind, n, k, B, seed, fused))
          for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        v = q.get(timeout=300)
        res[v[0]] = v
    for p in ps:
        p.join(120)
        assert p.exitcode == 0
    return [res[r] for r in range(world)]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", ["normal", "lognormal", "few_distinct", "u64_above_2_53",
                                  "signed_zeros", "all_equal"])
def test_dist_sort_matches_oracle_level0(world, kind):
    n, k, B, seed = 30000, 64, 64, 3
    a, _ = _shards(kind, n, world, seed)
    res = _run(world, kind, n, k, B, seed)
    assert all(r[1] == "ok" for r in res)
    got = np.concatenate([r[2] for r in res]).view(a.dtype)
    want = a[np.argsort(oracle.ordering_keys(a), kind="stable")]
    assert got.tobytes() == want.tobytes()
    ref = oracle.sort(a.copy(), k=k, base_case=B, trace=True)
    r0 = ref.records[0]
    bounds, counts, model = res[0][3], res[0][4], res[0][5]
    assert all(r[3] == bounds and np.array_equal(r[4], counts) and r[5] == model for r in res)
    assert np.array_equal(counts.astype(np.uint64), r0.counts)
    if r0.kind == oracle.MODEL_LINEAR:
        assert model[3] == ipls.MODEL_LINEAR
        assert (model[0], model[1], model[2]) == (r0.A, r0.B, r0.D)
    else:
        assert model[3] == ipls.MODEL_EQ3 and model[4] == r0.pivot_ok
    # rank r holds global positions [cuts[r], cuts[r+1]): bucket boundaries unless EQ3's
    # ==pivot bucket is cut (bounds are then ipls_assign_ranges')
    pre = np.concatenate([[0], np.cumsum(counts)])
    split = [0, 1, 0] if model[3] == ipls.MODEL_EQ3 else None
    cuts = ipls.assign_cuts(counts, world, split)
    if split is None:
        assert bounds == ipls.assign_ranges(counts, world)
        assert cuts == [int(pre[b]) for b in bounds]
    for r in res:
        rk = r[0]
        assert r[6] == cuts[rk] and len(r[2]) == cuts[rk + 1] - cuts[rk]
        assert r[7] == n


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", ["normal", "few_distinct", "u64_above_2_53", "all_equal"])
def test_dist_sort_fused_exchange_equals_all_to_all_path(world, kind):
    """The fused exchange (count, plan, scatter into the owners' buffers: here shared memory
    standing for peer memory) gives every rank exactly what partition + all-to-all + regroup
    gives it (an EQ3 top level, all_equal, takes that path itself)."""
    n, k, B, seed = 30000, 64, 64, 3
    a, _ = _shards(kind, n, world, seed)
    ref = _run(world, kind, n, k, B, seed)
    res = _run(world, kind, n, k, B, seed, fused=True)
    assert all(r[1] == "ok" for r in res)
    for x, y in zip(ref, res):
        assert x[2].tobytes() == y[2].tobytes()
        assert x[3] == y[3] and np.array_equal(x[4], y[4]) and x[5:] == y[5:]
    got = np.concatenate([r[2] for r in res]).view(a.dtype)
    assert got.tobytes() == a[np.argsort(oracle.ordering_keys(a), kind="stable")].tobytes()


def test_fused_plan_places_the_global_stable_partition():
    """fused_plan against the definition: rank d's buffer, filled source by source at
    offset[s, b], is the stable partition of the concatenated array restricted to d's
    buckets."""
    from paper_2208_06902_b200.distributed import exchange_plan, fused_plan
    rng = np.random.default_rng(11)
    for trial in range(60):
        G, k = int(rng.integers(1, 6)), int(rng.integers(3, 12))
        shards = [rng.integers(0, k, int(rng.integers(0, 40))) for _ in range(G)]  # bucket ids
        tags = [np.arange(len(sh)) + 1000 * s for s, sh in enumerate(shards)]     # key identity
        cnt = np.array([np.bincount(sh, minlength=k) for sh in shards])
        cuts, bounds, owner, offset, recv = fused_plan(cnt, G)
        c2, b2, M = exchange_plan(cnt, G, None)
        assert cuts == c2 and bounds == b2 and recv == [int(m.sum()) for m in M]
        bufs = [np.full(recv[d], -1, np.int64) for d in range(G)]
        for s in range(G):
            order = np.argsort(shards[s], kind="stable")
            off = np.concatenate([[0], np.cumsum(cnt[s])])
            for b in range(k):
                run = tags[s][order][off[b]:off[b + 1]]
                o = int(offset[s, b])
                bufs[int(owner[b])][o:o + len(run)] = run
        allb, allt = np.concatenate(shards), np.concatenate(tags)
        glob = allt[np.argsort(allb, kind="stable")]
        assert np.array_equal(np.concatenate(bufs), glob)
        for d in range(G):
            assert len(bufs[d]) == cuts[d + 1] - cuts[d]


def test_dist_sort_tiny_and_nan():
    res = _run(2, "normal", 5)  # global n < 8: no sample, everything to one rank
    assert all(r[1] == "ok" and r[5] is None for r in res)
    a, _ = _shards("normal", 5, 2, 3)
    got = np.concatenate([r[2] for r in res]).view(np.float64)
    assert got.tobytes() == np.sort(a).tobytes()
    res = _run(2, "nan_one", 20000)
    assert all(r[1] == "err" and r[2] == 2 for r in res)


@pytest.mark.parametrize("G", [1, 2, 3, 5, 8])
def test_assign_ranges_is_argmin_per_boundary(G):
    rng = np.random.default_rng(G)
    for trial in range(200):
        k = int(rng.integers(1, 40))
        c = rng.integers(0, 5, k) * (rng.random(k) < 0.7)
        if trial % 7 == 0:
            c[:] = 0
            c[rng.integers(0, k)] = 100
        b = ipls.assign_ranges(c, G)
        assert b[0] == 0 and b[G] == k and all(b[i] <= b[i + 1] for i in range(G))
        pre = np.concatenate([[0], np.cumsum(c)])
        tot = int(pre[-1])
        for r in range(1, G):
            cand = range(b[r - 1], k + 1)
            d = [abs(G * int(pre[x]) - r * tot) for x in cand]
            assert b[r] == b[r - 1] + int(np.argmin(d))  # argmin, ties to the lower boundary


@pytest.mark.parametrize("G", [1, 2, 3, 5, 8])
def test_assign_cuts_is_argmin_per_cut(G):
    """ipls_assign_cuts against brute force over its candidates; without splittable buckets
    it is ipls_assign_ranges in positions."""
    rng = np.random.default_rng(100 + G)
    for trial in range(200):
        k = int(rng.integers(1, 12))
        c = rng.integers(0, 9, k) * (rng.random(k) < 0.7)
        if trial % 5 == 0:
            c[:] = 0
            c[rng.integers(0, k)] = int(rng.integers(1, 50))
        pre = np.concatenate([[0], np.cumsum(c)])
        tot = int(pre[-1])
        cuts = ipls.assign_cuts(c, G)
        assert cuts == [int(pre[b]) for b in ipls.assign_ranges(c, G)]
        sp = rng.random(k) < 0.5
        cuts = ipls.assign_cuts(c, G, sp)
        cand = sorted(set(int(x) for x in pre) |
                      {x for b in range(k) if sp[b] for x in range(pre[b] + 1, pre[b + 1])})
        assert cuts[0] == 0 and cuts[G] == tot
        for r in range(1, G):
            ok = [x for x in cand if x >= cuts[r - 1]]
            d = [abs(G * x - r * tot) for x in ok]
            assert cuts[r] == ok[int(np.argmin(d))]  # argmin, ties to the lower candidate


def test_exchange_plan_moves_every_key_once():
    from paper_2208_06902_b200.distributed import exchange_plan
    rng = np.random.default_rng(7)
    for trial in range(100):
        G, k = int(rng.integers(1, 6)), int(rng.integers(1, 10))
        cnt = rng.integers(0, 7, (G, k)) * (rng.random((G, k)) < 0.8)
        sp = rng.random(k) < 0.4
        cuts, bounds, M = exchange_plan(cnt, G, sp)
        assert np.array_equal(sum(M), cnt)                    # every key goes to one rank
        for d in range(G):
            assert int(M[d].sum()) == cuts[d + 1] - cuts[d]
            pre = np.concatenate([[0], np.cumsum(cnt.sum(axis=0))])
            assert pre[bounds[d]] >= cuts[d] and (bounds[d] == 0 or pre[bounds[d] - 1] < cuts[d]
                                                  or cnt.sum(axis=0)[bounds[d] - 1] == 0)
            for b in range(k):                                # only splittable buckets shared
                if not sp[b] and 0 < M[d][:, b].sum() < cnt[:, b].sum():
                    raise AssertionError((trial, d, b))
        if not sp.any():
            assert bounds == ipls.assign_ranges(cnt.sum(axis=0), G)


def test_dist_sort_splits_a_degenerate_input_evenly():
    """All keys equal: EQ3 puts them in the ==pivot bucket, which is cut between the ranks."""
    world, n = 3, 30000
    res = _run(world, "all_equal", n)
    assert all(r[1] == "ok" for r in res)
    assert [len(r[2]) for r in res] == [10000, 10000, 10000]
    assert [r[6] for r in res] == [0, 10000, 20000]


def test_sample_size_matches_oracle():
    for m in [2, 7, 8, 100, 4097, 10**6, 10**8, 2 * 10**8, 3 * 10**9]:
        for k in [3, 64, 256, 1024]:
            assert ipls.sample_size(m, k) == oracle.sample_size(m, k)
