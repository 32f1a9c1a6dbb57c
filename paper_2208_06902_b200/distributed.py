"""Multi-GPU top level of IPLS: one exchange step, then local sorts.

The paper parallelises one distribution step across threads and recurses into buckets
independently; across GPUs the same structure is the classic distributed sample
sort.  A global array is the concatenation, in rank order, of every rank's shard:

1. sample — each rank writes the strata of the global level-0 sample it holds
   (`ipls_sample_strata`); a SUM all-reduce of the zero-filled slots assembles the whole
   sample on every rank.  It is exactly the sample a one-GPU sort of the concatenation
   draws at level 0 (R2, R18);
2. fit — every rank sorts the sample and fits FMCD in one kernel (`ipls_fit_sample`,
   Listing 1), so every rank holds the identical model (degenerate → EQ3, R5);
3. partition — every rank partitions its shard by the model (`ipls_partition_level`,
   P:505-530, stable);
4. plan — the per-rank bucket counts are all-gathered; `ipls_assign_cuts` gives rank r the
   global positions [cuts[r], cuts[r+1]) of the bucket-major order balanced by count, cut
   only at bucket boundaries (buckets are range-ordered, so contiguous bucket ranges are key
   ranges) or inside EQ3's ==pivot bucket, which holds one key value (R5) and so can be
   shared between ranks (a degenerate input still spreads evenly);
5. exchange + finish — one all-to-all moves every bucket range to its rank; the rank puts
   the G runs it received (one per source, each bucket-major) into bucket-major order
   (`ipls_regroup_runs`) and resumes the recursion at level 1 with its buckets as the
   segments (`ipls_sort_segments`): the top level is not repeated, and every model below it
   is the one a one-GPU sort of the concatenation fits (the regrouped bucket is exactly the
   stable level-0 child of the global array).

Fused exchange (`dist_sort(..., peers=SymmPeers(reuse=True))` or `fused=True`, for a linear
top-level model; bench.py's multi-GPU path): steps 3 and 5's partition + all-to-all + regroup (three passes over the keys) become
one.  Every rank counts its buckets (`ipls_partition_count`), the counts are all-gathered,
`fused_plan` gives every (source, bucket) its place in the owner's receive buffer
(bucket-major, then source rank: exactly `ipls_regroup_runs`' layout), and the stable scatter
(`ipls_partition_scatter_to`) stores every run straight into that buffer -- the owner's
memory mapped into the source's address space (torch symmetric memory: CUDA VMM allocations
shared over NVLink / NVSwitch).  One barrier, then the local sort.  EQ3 top levels (degenerate
global samples: a bucket shared between ranks) keep the all-to-all path.

Failures agree: every rank all-reduces (MAX) its status before each collective that follows
a step that can fail (fit, partition, the receive allocation) and after the local sort, and
all ranks raise together.

Rank r then holds the r-th key range sorted; the concatenation over ranks is the sorted
global array.  Every step that touches keys runs in libipls.so's kernels; this module only
moves tensors between the C-ABI calls and the collectives (NCCL over NVLink on GPUs).  The
compute steps are the `ops` object's methods so that the CPU `gloo` tests can run the same
orchestration with the oracle standing in for the kernels (tests only; the product `ops`
is `CudaOps`).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from . import (DEFAULT_SEED, MODEL_EQ3, IPLSError, Model, assign_cuts, fit_fmcd, partition_count,
               partition_level, partition_scatter_to, regroup_runs, sample_size, sample_strata,
               sort, sort_segments, _key_type_of)


class CudaOps:
    """The product compute steps: libipls.so calls on CUDA tensors."""

    def __init__(self, stream=None):
        self.stream = stream

    def sample(self, keys, global_begin: int, global_m: int, S: int, seed: int):
        import torch
        out = torch.zeros(S, dtype=torch.int64, device=keys.device)
        sample_strata(keys, global_begin, global_m, S, out, seed=seed, stream=self.stream)
        return out

    def sort(self, keys, key_type: int, k: int, base_case: int, seed: int) -> int:
        """Sort in place; returns the library status (0 = ok) instead of raising, so that
        every rank can agree on the outcome before raising."""
        try:
            sort(keys, k=k, base_case=base_case, seed=seed, key_type=key_type,
                 stream=self.stream)
            return 0
        except IPLSError as e:
            return e.status

    def fit(self, sample, key_type: int, k: int) -> Model:
        """Sort the (unsorted) sample and fit FMCD in one launch (ipls_fit_sample)."""
        return fit_fmcd(sample, k, key_type=key_type, stream=self.stream, presorted=False)

    def partition(self, keys, model: Model, key_type: int):
        """Returns (partitioned keys, offsets as a host list of k_eff + 1 ints)."""
        import torch
        out = torch.empty_like(keys)
        off, _ = partition_level(keys, out, model, key_type=key_type, stream=self.stream)
        return out, [int(x) for x in off.cpu().tolist()]

    def partition_count(self, keys, model: Model, key_type: int):
        """Bucket boundaries of the shard's stable partition (host list of k_eff + 1 ints)."""
        off = partition_count(keys, model, key_type=key_type, stream=self.stream)
        return [int(x) for x in off.cpu().tolist()]

    def scatter_to(self, keys, model: Model, key_type: int, addresses) -> int:
        """Stable scatter with one destination address per bucket (host list of ints; own or
        peer memory); returns the status."""
        import torch
        try:
            dst = torch.tensor(addresses, dtype=torch.int64, device=keys.device)
            partition_scatter_to(keys, model, dst, key_type=key_type, stream=self.stream)
            return 0
        except IPLSError as e:
            return e.status

    def regroup(self, runs, counts: np.ndarray):
        """The G received runs (counts: G x nb) into bucket-major order (ipls_regroup_runs)."""
        import torch
        if counts.shape[0] <= 1:
            return runs  # one run is bucket-major already
        out = torch.empty_like(runs)
        regroup_runs(runs, out, counts, stream=self.stream)
        return out

    def sort_segments(self, keys, key_type: int, k: int, base_case: int, seed: int, sizes,
                      level: int, global_begin: int = 0) -> int:
        """Sort range-ordered segments from `level` on (ipls_sort_segments; global_begin =
        the position of keys[0] in the global order); returns the status instead of raising
        (see sort)."""
        try:
            sort_segments(keys, sizes, level=level, k=k, base_case=base_case, seed=seed,
                          key_type=key_type, stream=self.stream, global_begin=global_begin)
            return 0
        except IPLSError as e:
            return e.status


@dataclass
class DistResult:
    keys: object            # this rank's sorted key range (same dtype/device as the input)
    bounds: List[int]       # bounds[r]: first bucket boundary at or after cuts[r]
    model: Optional[Model]  # the shared top-level model (None when the global n < 8)
    counts: np.ndarray      # global bucket counts of the top level
    global_begin: int       # position of this rank's output in the sorted global array
    global_n: int
    cuts: List[int]         # rank r holds global positions [cuts[r], cuts[r+1])


def exchange_plan(cnt: np.ndarray, G: int, splittable=None):
    """The exchange of step 4 from the G x k per-rank bucket counts (host).

    cuts = ipls_assign_cuts of the global counts (positions in the bucket-major global order;
    only `splittable` buckets may be cut inside); bounds[r] = the first bucket boundary at or
    after cuts[r] (= ipls_assign_ranges' bounds when nothing is split); M[d][s, b] = how many
    of source s's bucket-b keys land on rank d.  Source s's bucket-b keys occupy the global
    positions pre[b] + sum(cnt[:s, b]) + [0, cnt[s, b]) (bucket-major, then rank order, then
    the stable partition order), so each rank's share of a source's run is one contiguous
    piece and the pieces for ranks 0..G-1 follow each other in the source's partitioned array.
    """
    cnt = np.asarray(cnt, dtype=np.int64)
    total = cnt.sum(axis=0)
    cuts = assign_cuts(total, G, splittable)
    pre = np.concatenate([[0], np.cumsum(total)])
    bounds = [int(np.searchsorted(pre, c, side="left")) for c in cuts[:G]] + [len(total)]
    start = pre[:-1][None, :] + np.cumsum(cnt, axis=0) - cnt       # G x k first positions
    end = start + cnt
    M = [np.clip(np.minimum(end, cuts[d + 1]) - np.maximum(start, cuts[d]), 0, None)
         for d in range(G)]
    return cuts, bounds, M


def fused_plan(cnt: np.ndarray, G: int):
    """The fused exchange's plan from the G x k per-rank bucket counts (host; no bucket is
    split between ranks).  Returns (cuts, bounds, owner, offset, recv):
    cuts, bounds as exchange_plan's; owner[b] = the rank that receives bucket b; offset[s, b] =
    the position, in owner[b]'s receive buffer, of source s's first key of bucket b -- the
    buffer holds the owner's buckets in order, each as source 0's keys, then source 1's, ...
    (the stable partition of the global array restricted to those buckets); recv[d] = keys
    rank d receives."""
    cnt = np.asarray(cnt, dtype=np.int64)
    total = cnt.sum(axis=0)
    cuts = assign_cuts(total, G, None)
    pre = np.concatenate([[0], np.cumsum(total)])
    bounds = [int(np.searchsorted(pre, c, side="left")) for c in cuts[:G]] + [len(total)]
    owner = np.zeros(len(total), dtype=np.int64)
    for d in range(G):
        owner[bounds[d]:bounds[d + 1]] = d
    base = pre[:-1] - pre[np.asarray(bounds)[owner]]          # bucket b's region in its owner
    offset = base[None, :] + np.cumsum(cnt, axis=0) - cnt      # + the lower sources' keys of b
    recv = [int(pre[bounds[d + 1]] - pre[bounds[d]]) for d in range(G)]
    return cuts, bounds, owner, offset, recv


class SymmPeers:
    """Receive buffers every rank of the group can store into: torch symmetric memory (CUDA
    VMM allocations exchanged between the processes and mapped over NVLink / NVSwitch)."""

    def __init__(self, group=None, reuse: bool = False):
        """reuse: keep the buffer between calls and hand it out again while it is large enough
        (the allocation and its rendezvous cost milliseconds).  The caller then owns the
        consequence: a dist_sort result is a view of the buffer and is overwritten by the next
        dist_sort that uses this object."""
        import torch.distributed as dist
        self.group = group if group is not None else dist.group.WORLD
        self.handle = None
        self.reuse = reuse
        self.buf = None

    def alloc(self, nelems: int, device):
        """A buffer of nelems int64 on every rank (same size everywhere) -> (this rank's
        tensor, the list of every rank's base address as seen from this rank)."""
        import torch
        import torch.distributed._symmetric_memory as symm
        if self.reuse and self.buf is not None and self.buf.numel() >= nelems:
            return self.buf, [int(p) for p in self.handle.buffer_ptrs]
        t = symm.empty(max(1, nelems), dtype=torch.int64, device=device)
        self.handle = symm.rendezvous(t, self.group)
        self.buf = t if self.reuse else None
        return t, [int(p) for p in self.handle.buffer_ptrs]

    def barrier(self):
        self.handle.barrier()


def _all_gather_int64(vals, group, device):
    """All-gather a 1-D list of ints (same length on every rank) -> [G, len] numpy."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.int64, device=device)
    G = dist.get_world_size(group)
    parts = [torch.empty_like(t) for _ in range(G)]
    dist.all_gather(parts, t, group=group)
    return np.stack([p.cpu().numpy() for p in parts])


def dist_sort(keys, k: int = 1024, base_case: int = 4096, seed: int = DEFAULT_SEED,
              key_type: Optional[int] = None, group=None, ops=None,
              marks: Optional[list] = None, fused: Optional[bool] = None,
              peers=None) -> DistResult:
    """Sort the global array whose rank-ordered shards the ranks of `group` hold.

    keys: this rank's shard (CUDA tensor, float64 or (u)int64 holding uint64 bits; left
    unmodified).  Returns this rank's key range, sorted.  Raises IPLSError on every rank if
    any rank's step fails (e.g. a NaN key anywhere: IPLS_ERR_NAN_KEY).
    marks: optional list; (phase name, CUDA event) pairs are appended at the phase
    boundaries (tools/time_dist.py).
    fused: scatter straight into the owners' receive buffers over peer memory instead of
    partition + all-to-all + regroup (module docstring).  Default: on when `peers` is given.
    peers: the object that provides those buffers; pass SymmPeers(group, reuse=True) and keep
    it between calls (fused=True alone allocates and exchanges fresh buffers in every call,
    ~7 ms: safe, since the result owns its buffer, but slower than the all-to-all path).
    """
    import torch
    import torch.distributed as dist
    ops = ops if ops is not None else CudaOps()

    def mark(name):
        if marks is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append((name, e))
    mark("start")
    kt = _key_type_of(keys, key_type)
    G = dist.get_world_size(group)
    r = dist.get_rank(group)
    dev = keys.device
    # collectives need the backend's device: NCCL takes CUDA tensors, gloo CPU ones
    cdev = dev if dist.get_backend(group) == "nccl" else torch.device("cpu")

    sizes = _all_gather_int64([keys.numel()], group, cdev)[:, 0]
    gbegin, gm = int(sizes[:r].sum()), int(sizes.sum())
    S = sample_size(gm, k) if gm >= 2 else 0

    def agree(st: int) -> int:
        t = torch.tensor([st], dtype=torch.int64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        return int(t.item())

    def attempt(fn):
        """Run fn; (result, 0) or (None, status) on an IPLSError or a device allocation
        failure, so that the ranks can agree before the next collective."""
        try:
            return fn(), 0
        except IPLSError as e:
            return None, e.status
        except torch.cuda.OutOfMemoryError:
            return None, 4  # IPLS_ERR_OUT_OF_MEMORY

    model: Optional[Model] = None
    status = 0
    if S >= 4:
        smp, status = attempt(lambda: ops.sample(keys, gbegin, gm, S, seed))  # step 1
        st = agree(status)
        if st:
            raise IPLSError(st, "in the distributed sample")
        smp_c = smp.to(cdev)
        dist.all_reduce(smp_c, op=dist.ReduceOp.SUM, group=group)
        smp = smp_c.to(dev)
        model, status = attempt(lambda: ops.fit(smp, kt, k))          # step 2 (same on all ranks)
    mark("sample+fit")
    if fused is None:
        fused = peers is not None
    if fused and model is not None and status == 0 and model.kind != MODEL_EQ3:
        return _fused_tail(keys, model, kt, k, base_case, seed, group, ops, peers, agree,
                           attempt, mark, cdev, G, r, gm)
    if model is not None and status == 0:
        po, status = attempt(lambda: ops.partition(keys, model, kt))  # step 3
        part, off = po if po is not None else (keys, [0, keys.numel()])
    else:                                                         # global n < 8 (or failed)
        part, off = keys, [0, keys.numel()]
    st = agree(status)
    if st:
        raise IPLSError(st, "in the distributed partition")
    part_w = part.view(torch.int64)
    ke = len(off) - 1
    cnt = _all_gather_int64([off[b + 1] - off[b] for b in range(ke)], group, cdev)
    total = cnt.sum(axis=0)
    mark("partition")
    # step 4: EQ3's ==pivot bucket holds one key value, so it may be split between ranks
    split = [0, 1, 0] if model is not None and model.kind == MODEL_EQ3 and ke == 3 else None
    cuts, bounds, M = exchange_plan(cnt, G, split)
    send = [int(M[d][r].sum()) for d in range(G)]
    recv = [int(M[r][s].sum()) for s in range(G)]
    out_w, status = attempt(lambda: torch.empty(sum(recv), dtype=torch.int64, device=cdev))
    if status == 0 and sum(recv) > 0xFFFFFFFF:
        status = 1  # IPLS_ERR_INVALID_ARGUMENT: beyond the ABI's 2^32 - 1 keys per call
    st = agree(status)
    if st:
        raise IPLSError(st, "before the exchange")
    dist.all_to_all_single(out_w, part_w.to(cdev), output_split_sizes=recv,   # step 5
                           input_split_sizes=send, group=group)
    runs = out_w.to(dev).view(keys.dtype)
    mark("plan+exchange")
    lo = bounds[r] - (1 if bounds[r] > 0 and total[:bounds[r]].sum() > cuts[r] else 0)
    mine = M[r][:, lo:bounds[r + 1]]                              # G x (my buckets)
    out, status = attempt(lambda: ops.regroup(runs, mine))
    if status == 0:
        sizes = mine.sum(axis=0)
        status = ops.sort_segments(out, kt, k, base_case, seed, sizes, 1, cuts[r])
    else:
        out = runs
    mark("local sort")
    st = agree(status)
    if st:
        raise IPLSError(st, "in the distributed sort")
    return DistResult(out, bounds, model, total, cuts[r], gm, cuts)


def _fused_tail(keys, model, kt, k, base_case, seed, group, ops, peers, agree, attempt, mark,
                cdev, G, r, gm) -> DistResult:
    """Steps 3'-5' of the fused exchange (module docstring)."""
    import torch
    dev = keys.device
    off, status = attempt(lambda: ops.partition_count(keys, model, kt))           # step 3'
    st = agree(status)
    if st:
        raise IPLSError(st, "in the distributed partition")
    ke = len(off) - 1
    cnt = _all_gather_int64([off[b + 1] - off[b] for b in range(ke)], group, cdev)
    total = cnt.sum(axis=0)
    mark("partition")
    cuts, bounds, owner, offset, recv = fused_plan(cnt, G)                        # step 4
    peers = peers if peers is not None else SymmPeers(group)
    status = 1 if max(recv) > 0xFFFFFFFF else 0  # beyond the ABI's 2^32 - 1 keys per call
    bp = None
    def alloc():
        try:
            return peers.alloc(max(recv), dev)
        except (IPLSError, torch.cuda.OutOfMemoryError):
            raise
        except Exception as e:  # no peer access, symmetric memory unavailable, ...
            raise IPLSError(6, f"peer receive buffers: {e}")
    if status == 0:
        bp, status = attempt(alloc)
    st = agree(status)
    if st:
        raise IPLSError(st, "before the exchange")
    buf, ptrs = bp
    addr = (np.asarray(ptrs, dtype=np.int64)[owner] + 8 * offset[r]).tolist()
    peers.barrier()   # every receive buffer exists (and nobody still reads an earlier one)
    status = ops.scatter_to(keys, model, kt, addr)                                # step 5'
    st = agree(status)
    if st:
        raise IPLSError(st, "in the exchange")
    peers.barrier()   # every source's stores have landed (scatter_to synchronises its stream)
    mark("plan+exchange")
    out = buf[:recv[r]].view(keys.dtype)
    sizes = total[bounds[r]:bounds[r + 1]]
    status = ops.sort_segments(out, kt, k, base_case, seed, sizes, 1, cuts[r])
    mark("local sort")
    st = agree(status)
    if st:
        raise IPLSError(st, "in the distributed sort")
    return DistResult(out, bounds, model, total, cuts[r], gm, cuts)


__all__ = ["dist_sort", "DistResult", "CudaOps", "SymmPeers", "fused_plan"]
