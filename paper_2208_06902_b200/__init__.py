"""IPLS distribution step on B200 (sm_100a): thin Python binding of libipls.so.

Argument marshalling only — every step of the sort runs in the library's CUDA kernels
(include/ipls.h).  PyTorch is used for device memory and streams.  If the native library
is missing or fails to load, every call raises: there is no CPU fallback.

Paper: In-Place Parallel Learned Sort (arXiv 2208.06902), PAPER.md cited as P:<line>.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

__all__ = [
    "IPLSError", "lib", "sort", "sort_host", "sort_host_batch", "fit_fmcd", "partition_level", "sort_trace",
    "workspace_bytes", "Model", "Record", "KEY_F64", "KEY_U64", "MODEL_LINEAR", "MODEL_EQ3", "MODEL_TREE",
    "MODEL_TREE_EQ", "DEFAULT_SEED", "launch_count", "sample_size", "sample_strata", "assign_ranges",
    "assign_cuts", "partition_count", "partition_scatter_to", "regroup_runs", "sort_segments",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libipls.so")

KEY_F64 = 0
KEY_U64 = 1
MODEL_LINEAR = 0
MODEL_EQ3 = 1
MODEL_TREE = 2        # splitter tree (IPS4o's classifier; config flag FLAG_TREE_MODEL)
MODEL_TREE_EQ = 3     # sort option: the tree with IPS4o's equality buckets (R24);
                      # trace records carry kind MODEL_TREE
FLAG_TREE_MODEL = 1
FLAG_TREE_EQUAL_BUCKETS = 2
DEFAULT_SEED = 0x49504C53

STATUS = {0: "ok", 1: "invalid argument", 2: "NaN key", 3: "degenerate sample",
          4: "out of memory", 5: "CUDA error", 6: "not implemented"}


class IPLSError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        super().__init__(f"ipls: {STATUS.get(status, status)}{(': ' + what) if what else ''}")


class _Config(ctypes.Structure):
    _fields_ = [("k", ctypes.c_uint32), ("base_case", ctypes.c_uint32),
                ("seed", ctypes.c_uint64), ("flags", ctypes.c_uint32)]


class _Model(ctypes.Structure):
    _fields_ = [("a", ctypes.c_double), ("b", ctypes.c_double), ("k", ctypes.c_uint32),
                ("D", ctypes.c_uint32), ("kind", ctypes.c_uint32), ("capped", ctypes.c_uint32),
                ("pivot_ok", ctypes.c_uint64)]


class _Rec(ctypes.Structure):
    _fields_ = [("level", ctypes.c_uint32), ("kind", ctypes.c_uint32),
                ("begin", ctypes.c_uint64), ("m", ctypes.c_uint64), ("S", ctypes.c_uint64),
                ("a", ctypes.c_double), ("b", ctypes.c_double),
                ("D", ctypes.c_uint32), ("capped", ctypes.c_uint32),
                ("pivot_ok", ctypes.c_uint64),
                ("k_eff", ctypes.c_uint32), ("requeued", ctypes.c_uint32)]


class _Trace(ctypes.Structure):
    _fields_ = [("records", ctypes.POINTER(_Rec)), ("records_cap", ctypes.c_size_t),
                ("records_len", ctypes.c_size_t),
                ("counts", ctypes.POINTER(ctypes.c_uint64)), ("counts_cap", ctypes.c_size_t),
                ("counts_len", ctypes.c_size_t),
                ("samples", ctypes.POINTER(ctypes.c_uint64)), ("samples_cap", ctypes.c_size_t),
                ("samples_len", ctypes.c_size_t),
                ("d_snapshots", ctypes.c_void_p), ("snapshot_levels", ctypes.c_uint32),
                ("levels", ctypes.c_uint32)]


class _ProfEntry(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 32), ("launches", ctypes.c_uint64),
                ("total_ms", ctypes.c_double), ("bytes", ctypes.c_double)]


# C-ABI symbols declared in include/ipls.h (tests check the .so exports all of them)
SYMBOLS = ["ipls_default_config", "ipls_sort_f64", "ipls_sort_u64", "ipls_sort_ex",
           "ipls_workspace_bytes", "ipls_sort_host", "ipls_sort_host_batch", "ipls_fit_fmcd", "ipls_partition_level",
           "ipls_sort_trace", "ipls_status_string", "ipls_last_cuda_error",
           "ipls_kernel_launch_count", "ipls_profile_enable", "ipls_profile_reset",
           "ipls_profile_read", "ipls_sample_size", "ipls_sample_strata", "ipls_assign_ranges", "ipls_assign_cuts", "ipls_fit_sample", "ipls_debug_set_epoch",
           "ipls_debug_force_match_rank", "ipls_sort_segments",
           "ipls_regroup_runs", "ipls_sort_segments_trace", "ipls_debug_term_mode",
           "ipls_partition_count", "ipls_partition_scatter_to"]

_lib = None


def lib():
    """Load libipls.so (fails loudly if it is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise IPLSError(6, f"native library {_LIB_PATH} not built (run __graft_entry__.build())")
        L = ctypes.CDLL(_LIB_PATH)
        vp, sz, u32, u64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_uint64
        i32 = ctypes.c_int
        L.ipls_default_config.restype = _Config
        L.ipls_sort_f64.argtypes = [vp, sz, vp]; L.ipls_sort_f64.restype = i32
        L.ipls_sort_u64.argtypes = [vp, sz, vp]; L.ipls_sort_u64.restype = i32
        L.ipls_sort_ex.argtypes = [vp, sz, i32, ctypes.POINTER(_Config), vp, sz, vp]
        L.ipls_sort_ex.restype = i32
        L.ipls_workspace_bytes.argtypes = [sz, i32, ctypes.POINTER(_Config)]
        L.ipls_workspace_bytes.restype = sz
        L.ipls_sort_host.argtypes = [vp, sz, i32, ctypes.POINTER(_Config), vp]
        L.ipls_sort_host.restype = i32
        L.ipls_sort_host_batch.argtypes = [vp, vp, vp, u32, i32, ctypes.POINTER(_Config), vp]
        L.ipls_sort_host_batch.restype = i32
        L.ipls_fit_fmcd.argtypes = [vp, sz, i32, u32, ctypes.POINTER(_Model), vp]
        L.ipls_fit_fmcd.restype = i32
        L.ipls_partition_level.argtypes = [vp, vp, sz, i32, ctypes.POINTER(_Model), vp, vp, vp]
        L.ipls_partition_level.restype = i32
        L.ipls_partition_count.argtypes = [vp, sz, i32, ctypes.POINTER(_Model), vp, vp]
        L.ipls_partition_count.restype = i32
        L.ipls_partition_scatter_to.argtypes = [vp, sz, i32, ctypes.POINTER(_Model), vp, vp]
        L.ipls_partition_scatter_to.restype = i32
        L.ipls_sort_trace.argtypes = [vp, sz, i32, ctypes.POINTER(_Config), ctypes.POINTER(_Trace), vp]
        L.ipls_sort_trace.restype = i32
        L.ipls_status_string.argtypes = [i32]; L.ipls_status_string.restype = ctypes.c_char_p
        L.ipls_last_cuda_error.restype = ctypes.c_char_p
        L.ipls_kernel_launch_count.restype = u64
        L.ipls_profile_enable.argtypes = [i32]; L.ipls_profile_enable.restype = None
        L.ipls_profile_reset.argtypes = []; L.ipls_profile_reset.restype = None
        L.ipls_profile_read.argtypes = [ctypes.POINTER(_ProfEntry), sz]
        L.ipls_profile_read.restype = sz
        L.ipls_debug_set_epoch.argtypes = [u32]; L.ipls_debug_set_epoch.restype = None
        L.ipls_debug_force_match_rank.argtypes = [i32]; L.ipls_debug_force_match_rank.restype = None
        L.ipls_debug_term_mode.argtypes = [i32]; L.ipls_debug_term_mode.restype = None
        L.ipls_fit_sample.argtypes = [vp, sz, i32, u32, ctypes.POINTER(_Model), vp]
        L.ipls_fit_sample.restype = i32
        L.ipls_sample_size.argtypes = [u64, u32]; L.ipls_sample_size.restype = u32
        L.ipls_sample_strata.argtypes = [vp, sz, u64, u64, u32, u64, vp, vp]
        L.ipls_sample_strata.restype = i32
        L.ipls_assign_ranges.argtypes = [vp, u32, u32, vp]; L.ipls_assign_ranges.restype = i32
        L.ipls_assign_cuts.argtypes = [vp, u32, u32, vp, vp]; L.ipls_assign_cuts.restype = i32
        L.ipls_sort_segments.argtypes = [vp, sz, i32, ctypes.POINTER(_Config), vp, u32, u32,
                                         ctypes.c_uint64, vp]
        L.ipls_sort_segments.restype = i32
        L.ipls_regroup_runs.argtypes = [vp, vp, vp, u32, u32, vp]; L.ipls_regroup_runs.restype = i32
        L.ipls_sort_segments_trace.argtypes = [vp, sz, i32, ctypes.POINTER(_Config), vp, u32, u32,
                                               ctypes.c_uint64, ctypes.POINTER(_Trace), vp]
        L.ipls_sort_segments_trace.restype = i32
        _lib = L
    return _lib


def _check(st: int):
    if st != 0:
        extra = ""
        if st == 5:
            extra = lib().ipls_last_cuda_error().decode()
        raise IPLSError(st, extra)


def _cfg(k: int, base_case: int, seed: int, model: int = MODEL_LINEAR) -> _Config:
    """model: MODEL_LINEAR (FMCD, the paper's IPLS), MODEL_TREE (splitter tree) or MODEL_TREE_EQ
    (the tree with equality buckets)."""
    if model not in (MODEL_LINEAR, MODEL_TREE, MODEL_TREE_EQ):
        raise ValueError("model must be MODEL_LINEAR, MODEL_TREE or MODEL_TREE_EQ")
    flags = {MODEL_TREE: FLAG_TREE_MODEL,
             MODEL_TREE_EQ: FLAG_TREE_MODEL | FLAG_TREE_EQUAL_BUCKETS}.get(model, 0)
    return _Config(k, base_case, seed, flags)


def _stream(stream) -> Optional[int]:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _key_type_of(t, key_type: Optional[int]) -> int:
    import torch
    if key_type is not None:
        return key_type
    if t.dtype == torch.float64:
        return KEY_F64
    if t.dtype in (torch.uint64, torch.int64):
        return KEY_U64
    raise TypeError(f"keys must be float64 or (u)int64, got {t.dtype}")


def _check_tensor(t):
    if not t.is_cuda or not t.is_contiguous() or t.element_size() != 8:
        raise ValueError("keys must be a contiguous CUDA tensor of 8-byte elements")


def profile_enable(on: bool = True) -> None:
    lib().ipls_profile_enable(1 if on else 0)


def profile_reset() -> None:
    lib().ipls_profile_reset()


def profile_read() -> dict:
    """{kernel: (launches, total_ms, algorithmic_bytes)} from the library's event timing."""
    L = lib()
    cnt = L.ipls_profile_read(None, 0)
    arr = (_ProfEntry * max(1, cnt))()
    L.ipls_profile_read(arr, cnt)
    return {arr[i].name.decode(): (int(arr[i].launches), float(arr[i].total_ms),
                                   float(arr[i].bytes)) for i in range(cnt)}


def launch_count() -> int:
    return int(lib().ipls_kernel_launch_count())


def sort(keys, k: int = 256, base_case: int = 4096, seed: int = DEFAULT_SEED,
         key_type: Optional[int] = None, stream=None, workspace=None,
         model: int = MODEL_LINEAR) -> None:
    """Sort a CUDA tensor in place (float64; uint64 or int64 holding uint64 bits)."""
    _check_tensor(keys)
    kt = _key_type_of(keys, key_type)
    c = _cfg(k, base_case, seed, model)
    ws, wsb = (None, 0)
    if workspace is not None:
        ws, wsb = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    _check(lib().ipls_sort_ex(keys.data_ptr(), keys.numel(), kt, ctypes.byref(c), ws, wsb,
                              _stream(stream)))


def sort_segments(keys, sizes, level: int = 1, k: int = 256, base_case: int = 4096,
                  seed: int = DEFAULT_SEED, key_type: Optional[int] = None, stream=None,
                  model: int = MODEL_LINEAR, global_begin: int = 0) -> None:
    """Sort in place a CUDA tensor made of consecutive range-ordered segments of the given
    sizes, resuming the recursion at `level` (ipls_sort_segments); global_begin: the
    position of keys[0] in the array whose recursion is resumed (sampling hash only)."""
    _check_tensor(keys)
    kt = _key_type_of(keys, key_type)
    c = _cfg(k, base_case, seed, model)
    sz = np.ascontiguousarray(np.asarray(sizes, dtype=np.uint64))
    _check(lib().ipls_sort_segments(keys.data_ptr(), keys.numel(), kt, ctypes.byref(c),
                                    sz.ctypes.data if sz.size else None, int(sz.size),
                                    int(level), int(global_begin), _stream(stream)))


def regroup_runs(src, dst, counts, stream=None) -> None:
    """ipls_regroup_runs: G received runs (counts: G x nb per-bucket counts) into bucket-major
    order in dst (CUDA tensors of 8-byte elements)."""
    _check_tensor(src)
    _check_tensor(dst)
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
    G, nb = (c.shape[0], c.shape[1]) if c.ndim == 2 else (0, 0)
    _check(lib().ipls_regroup_runs(src.data_ptr(), dst.data_ptr(),
                                   c.ctypes.data if c.size else None, G, nb, _stream(stream)))


def workspace_bytes(n: int, key_type: int = KEY_F64, k: int = 256, base_case: int = 4096,
                    model: int = MODEL_LINEAR) -> int:
    c = _cfg(k, base_case, DEFAULT_SEED, model)
    return int(lib().ipls_workspace_bytes(n, key_type, ctypes.byref(c)))


def sort_host(keys: np.ndarray, k: int = 256, base_case: int = 4096, seed: int = DEFAULT_SEED,
              stream=None, model: int = MODEL_LINEAR) -> None:
    """Sort a host numpy array (float64/uint64; ideally pinned memory) through the library."""
    if not keys.flags.c_contiguous or keys.dtype.itemsize != 8:
        raise ValueError("keys must be a contiguous 8-byte numpy array")
    kt = KEY_F64 if keys.dtype == np.float64 else KEY_U64
    c = _cfg(k, base_case, seed, model)
    _check(lib().ipls_sort_host(keys.ctypes.data, keys.size, kt, ctypes.byref(c), _stream(stream)))


def sort_host_ptr(ptr: int, n: int, key_type: int, k: int = 256, base_case: int = 4096,
                  seed: int = DEFAULT_SEED, stream=None, model: int = MODEL_LINEAR) -> None:
    c = _cfg(k, base_case, seed, model)
    _check(lib().ipls_sort_host(ptr, n, key_type, ctypes.byref(c), _stream(stream)))


def sort_host_batch(ins, outs, sizes, key_type: int, k: int = 256, base_case: int = 4096,
                    seed: int = DEFAULT_SEED, stream=None, model: int = MODEL_LINEAR) -> None:
    """Sort `len(ins)` host arrays given as raw pointers (ins[j] -> outs[j], sizes[j] keys),
    with the copies pipelined against the sorts (ipls_sort_host_batch)."""
    m = len(ins)
    if len(outs) != m or len(sizes) != m:
        raise ValueError("ins, outs and sizes must have the same length")
    pi = (ctypes.c_void_p * max(m, 1))(*ins)
    po = (ctypes.c_void_p * max(m, 1))(*outs)
    pn = (ctypes.c_size_t * max(m, 1))(*sizes)
    c = _cfg(k, base_case, seed, model)
    _check(lib().ipls_sort_host_batch(pi, po, pn, m, key_type, ctypes.byref(c), _stream(stream)))


@dataclass
class Model:
    a: float
    b: float
    k: int
    D: int
    kind: int
    capped: int
    pivot_ok: int
    degenerate: bool = False


def fit_fmcd(sorted_sample, k: int, key_type: Optional[int] = None, stream=None,
             presorted: bool = True) -> Model:
    """FMCD (Listing 1) of a sample held in a CUDA tensor: sorted (ipls_fit_fmcd), or
    presorted=False to have the fit kernel sort it first (ipls_fit_sample)."""
    _check_tensor(sorted_sample)
    kt = _key_type_of(sorted_sample, key_type)
    m = _Model()
    fn = lib().ipls_fit_sample if not presorted else lib().ipls_fit_fmcd
    st = fn(sorted_sample.data_ptr(), sorted_sample.numel(), kt, k, ctypes.byref(m),
            _stream(stream))
    if st not in (0, 3):
        _check(st)
    return Model(m.a, m.b, m.k, m.D, m.kind, m.capped, m.pivot_ok, st == 3)


def partition_level(keys_in, keys_out, model: Model, key_type: Optional[int] = None,
                    want_ids: bool = False, stream=None):
    """One distribution step with a given model; returns (offsets, ids or None) tensors."""
    import torch
    _check_tensor(keys_in)
    _check_tensor(keys_out)
    kt = _key_type_of(keys_in, key_type)
    ke = 3 if model.kind == MODEL_EQ3 else model.k
    off = torch.empty(ke + 1, dtype=torch.int64, device=keys_in.device)
    ids = torch.empty(max(1, keys_in.numel()), dtype=torch.int16, device=keys_in.device) \
        if want_ids else None
    m = _Model(model.a, model.b, model.k, model.D, model.kind, model.capped, model.pivot_ok)
    _check(lib().ipls_partition_level(keys_in.data_ptr(), keys_out.data_ptr(), keys_in.numel(),
                                      kt, ctypes.byref(m), off.data_ptr(),
                                      ids.data_ptr() if ids is not None else None,
                                      _stream(stream)))
    return off, (ids[:keys_in.numel()] if ids is not None else None)


def partition_count(keys_in, model: Model, key_type: Optional[int] = None, stream=None):
    """The classify half of partition_level: the k_eff + 1 bucket boundaries of keys_in's stable
    partition (int64 CUDA tensor).  include/ipls.h: ipls_partition_count."""
    import torch
    _check_tensor(keys_in)
    kt = _key_type_of(keys_in, key_type)
    ke = 3 if model.kind == MODEL_EQ3 else model.k
    off = torch.empty(ke + 1, dtype=torch.int64, device=keys_in.device)
    m = _Model(model.a, model.b, model.k, model.D, model.kind, model.capped, model.pivot_ok)
    _check(lib().ipls_partition_count(keys_in.data_ptr(), keys_in.numel(), kt, ctypes.byref(m),
                                      off.data_ptr(), _stream(stream)))
    return off


def partition_scatter_to(keys_in, model: Model, bucket_dst, key_type: Optional[int] = None,
                         stream=None) -> None:
    """Stable scatter of keys_in with one destination per bucket: bucket b's keys go to the
    64-bit words from ADDRESS bucket_dst[b] on (int64 CUDA tensor of k_eff device addresses:
    own or peer memory).  include/ipls.h: ipls_partition_scatter_to."""
    _check_tensor(keys_in)
    _check_tensor(bucket_dst)
    kt = _key_type_of(keys_in, key_type)
    ke = 3 if model.kind == MODEL_EQ3 else model.k
    if bucket_dst.numel() < ke:
        raise ValueError("bucket_dst must hold one address per bucket")
    m = _Model(model.a, model.b, model.k, model.D, model.kind, model.capped, model.pivot_ok)
    _check(lib().ipls_partition_scatter_to(keys_in.data_ptr(), keys_in.numel(), kt,
                                           ctypes.byref(m), bucket_dst.data_ptr(),
                                           _stream(stream)))


def sample_size(m: int, k: int) -> int:
    """S(m) of P:473 (R1, R19), from the library (host function, no GPU needed)."""
    return int(lib().ipls_sample_size(m, k))


def sample_strata(keys, global_begin: int, global_m: int, S: int, out,
                  seed: int = DEFAULT_SEED, stream=None) -> None:
    """Write the strata of the global level-0 sample that this shard holds into `out`
    (S int64 slots, CUDA; other slots untouched).  include/ipls.h: ipls_sample_strata."""
    _check_tensor(keys)
    _check_tensor(out)
    if out.numel() < S:
        raise ValueError("out must hold S slots")
    _check(lib().ipls_sample_strata(keys.data_ptr(), keys.numel(), global_begin, global_m, S,
                                    seed & 0xFFFFFFFFFFFFFFFF, out.data_ptr(), _stream(stream)))


def assign_ranges(counts, G: int) -> List[int]:
    """Contiguous bucket ranges per rank balanced by count (host; ipls_assign_ranges)."""
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
    if c.size == 0:
        raise ValueError("counts must not be empty")
    b = np.zeros(G + 1, dtype=np.uint32)
    _check(lib().ipls_assign_ranges(c.ctypes.data, c.size, G, b.ctypes.data))
    return [int(x) for x in b]


def assign_cuts(counts, G: int, splittable=None) -> List[int]:
    """Global cut positions per rank; buckets flagged in `splittable` (one key value each)
    may be split between ranks (host; ipls_assign_cuts)."""
    c = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
    if c.size == 0:
        raise ValueError("counts must not be empty")
    sp = None
    if splittable is not None:
        sp = np.ascontiguousarray(np.asarray(splittable, dtype=np.uint8))
        if sp.size != c.size:
            raise ValueError("splittable must have one flag per bucket")
    out = np.zeros(G + 1, dtype=np.uint64)
    _check(lib().ipls_assign_cuts(c.ctypes.data, c.size, G,
                                  None if sp is None else sp.ctypes.data, out.ctypes.data))
    return [int(x) for x in out]


@dataclass
class Record:
    level: int
    kind: int
    begin: int
    m: int
    S: int
    A: float
    B: float
    D: int
    capped: int
    pivot_ok: int
    k_eff: int
    requeued: int
    sample: np.ndarray
    counts: np.ndarray


@dataclass
class TraceResult:
    records: List[Record]
    levels: int
    snapshots: Optional[object]  # torch tensor [levels, n] or None


def sort_trace(keys, k: int = 256, base_case: int = 4096, seed: int = DEFAULT_SEED,
               key_type: Optional[int] = None, snapshot_levels: int = 0, stream=None,
               max_records: int = 1 << 16, max_counts: int = 1 << 24,
               max_samples: int = 1 << 24, model: int = MODEL_LINEAR, segments=None,
               level: int = 1, global_begin: int = 0) -> TraceResult:
    """Sort in place and return the per-segment trace (records ordered by level, begin).
    segments: sizes of range-ordered segments to resume from at `level`
    (ipls_sort_segments_trace) instead of a whole sort."""
    import torch
    _check_tensor(keys)
    kt = _key_type_of(keys, key_type)
    c = _cfg(k, base_case, seed, model)
    n = keys.numel()
    snaps = None
    if snapshot_levels:
        snaps = torch.zeros((snapshot_levels, n), dtype=torch.int64, device=keys.device)
    for _ in range(3):
        recs = (_Rec * max_records)()
        cnts = np.zeros(max_counts, dtype=np.uint64)
        smps = np.zeros(max_samples, dtype=np.uint64)
        tr = _Trace(ctypes.cast(recs, ctypes.POINTER(_Rec)), max_records, 0,
                    cnts.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), max_counts, 0,
                    smps.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), max_samples, 0,
                    snaps.data_ptr() if snaps is not None else None, snapshot_levels, 0)
        backup = keys.clone()
        if segments is None:
            _check(lib().ipls_sort_trace(keys.data_ptr(), n, kt, ctypes.byref(c),
                                         ctypes.byref(tr), _stream(stream)))
        else:
            sz = np.ascontiguousarray(np.asarray(segments, dtype=np.uint64))
            _check(lib().ipls_sort_segments_trace(keys.data_ptr(), n, kt, ctypes.byref(c),
                                                  sz.ctypes.data if sz.size else None,
                                                  int(sz.size), int(level), int(global_begin),
                                                  ctypes.byref(tr),
                                                  _stream(stream)))
        if tr.records_len <= max_records and tr.counts_len <= max_counts and \
                tr.samples_len <= max_samples:
            break
        keys.copy_(backup)
        max_records = int(tr.records_len) + 16
        max_counts = int(tr.counts_len) + 16
        max_samples = int(tr.samples_len) + 16
    out: List[Record] = []
    ci = si = 0
    for i in range(tr.records_len):
        r = recs[i]
        cn = cnts[ci:ci + r.k_eff].copy(); ci += r.k_eff
        sp = smps[si:si + r.S].copy(); si += r.S
        out.append(Record(r.level, r.kind, r.begin, r.m, r.S, r.a, r.b, r.D, r.capped,
                          r.pivot_ok, r.k_eff, r.requeued, sp, cn))
    return TraceResult(out, int(tr.levels), snaps)
