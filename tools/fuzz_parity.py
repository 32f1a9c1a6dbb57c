"""Randomised GPU-vs-oracle parity campaign (dev tool, run on the GPU box): for SECONDS seconds
draw a random input kind, size, k, base case and model (FMCD, splitter tree, tree with
equality buckets), sort it with the traced GPU entry point and with the oracle, and compare
every record (level, begin, m, S, model, counts, sample) and the final bytes; every few cases
also the fused exchange's two calls (ipls_partition_count / ipls_partition_scatter_to) on
random shards against the oracle's stable partition of the whole array.  Prints the first
mismatch (with the seed that reproduces it) and exits 1, or a summary.

usage: python tools/fuzz_parity.py [SECONDS] [SEED]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle
import paper_2208_06902_b200 as ipls
from paper_2208_06902_b200 import datagen
from paper_2208_06902_b200.distributed import fused_plan

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
seed0 = int(sys.argv[2]) if len(sys.argv) > 2 else 1
MODELS = [(ipls.MODEL_LINEAR, oracle.MODEL_LINEAR), (ipls.MODEL_TREE, oracle.MODEL_TREE),
          (ipls.MODEL_TREE_EQ, oracle.MODEL_TREE_EQ)]


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int64).copy()).cuda()


def check_sort(rng, case):
    kind = datagen.FUZZ_KINDS[int(rng.integers(len(datagen.FUZZ_KINDS)))]
    n = int(10 ** rng.uniform(0.3, 6.3))
    gm, om = MODELS[int(rng.integers(3))]
    if gm == ipls.MODEL_LINEAR:
        k = int(rng.choice([3, 5, 16, 100, 256, 1000, 1024]))
    else:
        k = int(rng.choice([8, 16, 64, 256, 1024]))
    B = int(rng.choice([1, 17, 64, 1000, 4096]))
    if n > 200_000 and (B < 64 or k < 16):   # keep the oracle's recursion short
        B, k = 4096, max(k, 64) if gm == ipls.MODEL_LINEAR else 256
    a = datagen.fuzz_array(rng, n, kind)
    kt = 0 if a.dtype == np.float64 else 1
    want = a.copy()
    ores = oracle.sort(want, k=k, base_case=B, trace=True, model=om)
    t = dev(a)
    desc = f"case {case}: kind={kind} n={n} k={k} B={B} model={gm}"
    gtr = ipls.sort_trace(t, k=k, base_case=B, key_type=kt, model=gm)
    got = t.cpu().numpy()
    assert got.tobytes() == want.tobytes(), desc + ": final bytes differ"
    assert gtr.levels == ores.levels and len(gtr.records) == len(ores.records), desc + ": levels"
    for g, o in zip(gtr.records, ores.records):
        assert (g.level, g.begin, g.m, g.S, g.kind, g.D, g.capped, g.pivot_ok, g.k_eff, g.requeued) \
            == (o.level, o.begin, o.m, o.S, o.kind, o.D, o.capped, o.pivot_ok, o.k_eff, o.requeued), desc
        assert g.A == o.A and g.B == o.B, desc + ": model"
        assert np.array_equal(g.counts, o.counts) and np.array_equal(g.sample, o.sample), desc
    return n


def check_exchange(rng, case):
    kind = ["normal", "lognormal", "few_distinct", "u64_above_2_53", "uniform"][int(rng.integers(5))]
    n = int(10 ** rng.uniform(2, 6.3))
    k = int(rng.choice([3, 16, 100, 256, 1024]))
    G = int(rng.integers(1, 9))
    a = datagen.fuzz_array(rng, n, kind)
    kt = 0 if a.dtype == np.float64 else 1
    desc = f"case {case}: exchange kind={kind} n={n} k={k} G={G}"
    if n < 8:
        return 0
    S = oracle.sample_size(n, k)
    if S < 4:
        return 0
    pos = oracle.sample_positions(ipls.DEFAULT_SEED, 0, 0, n, S).astype(np.int64)
    smp = a[pos]
    smp = smp[np.argsort(oracle.ordering_keys(smp), kind="stable")]
    f = oracle.fit_fmcd(smp.astype(np.float64), k)
    if f.degenerate:
        piv = int(oracle.ordering_keys(smp[S // 2:S // 2 + 1])[0])
        m = ipls.Model(0.0, 0.0, 3, 0, ipls.MODEL_EQ3, 0, piv, True)
    else:
        m = ipls.Model(f.A, f.B, k, f.D, ipls.MODEL_LINEAR, int(f.capped), 0, False)
    want, _, _ = oracle.partition(a, m.a, m.b, m.k, m.kind, m.pivot_ok)
    shards = np.split(a, np.sort(rng.integers(0, n + 1, G - 1)))
    tsh = [dev(s) for s in shards]
    cnt = np.array([np.diff(ipls.partition_count(t, m, key_type=kt).cpu().numpy()) for t in tsh])
    _, _, owner, offset, recv = fused_plan(cnt, G)
    bufs = [torch.full((max(1, recv[d]),), -1, dtype=torch.int64, device="cuda") for d in range(G)]
    base = np.array([bufs[int(owner[b])].data_ptr() for b in range(cnt.shape[1])], dtype=np.int64)
    for s, t in enumerate(tsh):
        ipls.partition_scatter_to(t, m, torch.from_numpy(base + 8 * offset[s]).cuda(), key_type=kt)
    got = np.concatenate([bufs[d][:recv[d]].cpu().numpy() for d in range(G)])
    assert got.tobytes() == want.tobytes(), desc
    return n


t0 = time.time()
case, keys = 0, 0
while time.time() - t0 < secs:
    rng = np.random.default_rng(seed0 * 1_000_003 + case)
    try:
        keys += check_exchange(rng, case) if case % 4 == 3 else check_sort(rng, case)
    except AssertionError as e:
        print(f"MISMATCH (seed {seed0}, {e})", flush=True)
        sys.exit(1)
    case += 1
print(f"fuzz_parity: {case} cases, {keys} keys, seed {seed0}, {time.time() - t0:.0f} s: all bit-exact",
      flush=True)
