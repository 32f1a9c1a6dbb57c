"""CPU oracle for the IPLS hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import this package.  The product path
(``paper_2208_06902_b200`` + ``libipls.so``) never imports it and shares no code
with it.

Thin ctypes wrapper over ``liboracle`` (``ipls_oracle.cpp``): plain, slow,
single-threaded C++ written step by step from the paper (PAPER.md, "P:<line>"):

* ``ordering_key``     P:576   (order-preserving double -> integer map)
* ``sample_size``      P:115, P:473 (alpha k - 1 samples, alpha = 0.2 log N; R1, R19)
* ``sample_positions`` P:115   ("random elements"; stratified SplitMix64, R2/R18) — parity
                                unpinned against the paper (the paper shows no sample)
* ``fit_fmcd``         P:410-463 (Listing 1, binary64; R3-R5)
* ``bucket``           P:394-402 (F(x) = clamp(floor(a x + b)); R7)
* ``partition``        P:505-530 (contiguous, stable; R11)
* ``sort``             P:114-121, P:469-475 (recursive partition + base case)

Readings R<n> are listed in DESIGN.md §3.
"""
from __future__ import annotations

import ctypes
import hashlib
import os
import struct
import subprocess
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ipls_oracle.cpp")
_LIB = os.path.join(_HERE, "libipls_oracle.so")

KEY_F64 = 0
KEY_U64 = 1
MODEL_LINEAR = 0
MODEL_EQ3 = 1
MODEL_TREE = 2
MODEL_TREE_EQ = 3   # sort option (R24): records carry kind MODEL_TREE
DEFAULT_SEED = 0x49504C53  # "IPLS"


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: -O2 -ffp-contract=off (no FMA), no fast-math."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "ipls_oracle.h"))
    ):
        subprocess.check_call(
            ["g++", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c++17", "-shared",
             "-fPIC", "-o", _LIB, _SRC]
        )
    return _LIB


class _Rec(ctypes.Structure):
    _fields_ = [
        ("level", ctypes.c_uint32), ("kind", ctypes.c_uint32),
        ("begin", ctypes.c_uint64), ("m", ctypes.c_uint64), ("S", ctypes.c_uint64),
        ("A", ctypes.c_double), ("B", ctypes.c_double),
        ("D", ctypes.c_uint32), ("capped", ctypes.c_uint32),
        ("pivot_ok", ctypes.c_uint64),
        ("k_eff", ctypes.c_uint32), ("requeued", ctypes.c_uint32),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        u64, u32, i32, dbl = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int, ctypes.c_double
        vp, sz = ctypes.c_void_p, ctypes.c_size_t
        L.oracle_ordering_key.argtypes = [u64, i32]; L.oracle_ordering_key.restype = u64
        L.oracle_splitmix64.argtypes = [u64]; L.oracle_splitmix64.restype = u64
        L.oracle_sample_size.argtypes = [u64, u32]; L.oracle_sample_size.restype = u64
        L.oracle_sample_positions.argtypes = [u64, u32, u64, u64, u64, vp]
        L.oracle_sample_positions.restype = None
        L.oracle_fit_fmcd.argtypes = [vp, sz, u32, vp, vp, vp, vp]; L.oracle_fit_fmcd.restype = i32
        L.oracle_bucket.argtypes = [u64, i32, i32, dbl, dbl, u32, u64]; L.oracle_bucket.restype = u32
        L.oracle_partition.argtypes = [vp, vp, sz, i32, i32, dbl, dbl, u32, u64, vp, vp]
        L.oracle_partition.restype = None
        L.oracle_trace_new.argtypes = [i32]; L.oracle_trace_new.restype = vp
        L.oracle_trace_free.argtypes = [vp]; L.oracle_trace_free.restype = None
        L.oracle_trace_num_records.argtypes = [vp]; L.oracle_trace_num_records.restype = sz
        L.oracle_trace_record.argtypes = [vp, sz, ctypes.POINTER(_Rec)]
        L.oracle_trace_record.restype = None
        L.oracle_trace_sample.argtypes = [vp, sz]; L.oracle_trace_sample.restype = vp
        L.oracle_trace_counts.argtypes = [vp, sz]; L.oracle_trace_counts.restype = vp
        L.oracle_trace_num_levels.argtypes = [vp]; L.oracle_trace_num_levels.restype = u32
        L.oracle_trace_snapshot.argtypes = [vp, u32]; L.oracle_trace_snapshot.restype = vp
        L.oracle_sort.argtypes = [vp, sz, i32, u32, u32, u64, vp]; L.oracle_sort.restype = i32
        L.oracle_sort_model.argtypes = [vp, sz, i32, u32, u32, u64, i32, vp]
        L.oracle_sort_model.restype = i32
        L.oracle_tree_splitters.argtypes = [vp, sz, u32, i32, vp]
        L.oracle_tree_splitters.restype = None
        L.oracle_tree_bucket.argtypes = [u64, i32, vp, u32]; L.oracle_tree_bucket.restype = u32
        L.oracle_tree_eq_bucket.argtypes = [u64, i32, vp, u32]; L.oracle_tree_eq_bucket.restype = u32
        _lib = L
    return _lib


def _key_type(a: np.ndarray) -> int:
    if a.dtype == np.float64:
        return KEY_F64
    if a.dtype == np.uint64:
        return KEY_U64
    raise TypeError(f"keys must be float64 or uint64, got {a.dtype}")


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def ordering_key(bits: int, key_type: int) -> int:
    return int(lib().oracle_ordering_key(bits, key_type))


def ordering_keys(a: np.ndarray) -> np.ndarray:
    """Vector form of P:576's map (numpy; the same rule, for test convenience)."""
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint64:
        return a.copy()
    b = a.view(np.uint64)
    neg = (b >> np.uint64(63)).astype(bool)
    return np.where(neg, ~b, b | np.uint64(1 << 63))


def splitmix64(z: int) -> int:
    return int(lib().oracle_splitmix64(z & 0xFFFFFFFFFFFFFFFF))


def sample_size(m: int, k: int) -> int:
    return int(lib().oracle_sample_size(m, k))


def sample_positions(seed: int, level: int, begin: int, m: int, S: int) -> np.ndarray:
    out = np.empty(S, dtype=np.uint64)
    lib().oracle_sample_positions(seed, level, begin, m, S, _ptr(out))
    return out


@dataclass
class Fit:
    A: float
    B: float
    D: int
    capped: bool
    degenerate: bool


def fit_fmcd(sorted_values: np.ndarray, k: int) -> Fit:
    s = np.ascontiguousarray(sorted_values, dtype=np.float64)
    if s.size < 4 or k < 3:
        raise ValueError("Listing 1 needs S >= 4 and k >= 3")
    A = ctypes.c_double(); B = ctypes.c_double()
    D = ctypes.c_uint32(); cap = ctypes.c_uint32()
    deg = lib().oracle_fit_fmcd(_ptr(s), s.size, k, ctypes.byref(A), ctypes.byref(B),
                                ctypes.byref(D), ctypes.byref(cap))
    return Fit(A.value, B.value, int(D.value), bool(cap.value), bool(deg))


def bucket(x, A: float, B: float, k: int, kind: int = MODEL_LINEAR, pivot_ok: int = 0) -> int:
    if isinstance(x, (np.uint64,)) or (isinstance(x, int) and not isinstance(x, bool)):
        bits, kt = int(x), KEY_U64
    else:
        bits, kt = struct.unpack("<Q", struct.pack("<d", float(x)))[0], KEY_F64
    return int(lib().oracle_bucket(bits, kt, kind, A, B, k, pivot_ok))


def partition(keys: np.ndarray, A: float, B: float, k: int, kind: int = MODEL_LINEAR,
              pivot_ok: int = 0):
    """Stable partition; returns (out, offsets[k_eff+1], ids)."""
    a = np.ascontiguousarray(keys)
    kt = _key_type(a)
    ke = 3 if kind == MODEL_EQ3 else k
    out = np.empty_like(a)
    off = np.zeros(ke + 1, dtype=np.uint64)
    ids = np.zeros(a.size, dtype=np.uint16)
    lib().oracle_partition(_ptr(a), _ptr(out), a.size, kt, kind, A, B, k, pivot_ok,
                           _ptr(off), _ptr(ids))
    return out, off, ids


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
    sample: np.ndarray   # sorted sample, raw key bits (uint64)
    counts: np.ndarray   # k_eff child counts (uint64)

    def packed(self) -> bytes:
        """48-byte digest record: pack('<QQQQIIQ', begin, m, bits(A), bits(B), D, kind, pivot_ok)."""
        a_bits = struct.unpack("<Q", struct.pack("<d", self.A))[0]
        b_bits = struct.unpack("<Q", struct.pack("<d", self.B))[0]
        return struct.pack("<QQQQIIQ", self.begin, self.m, a_bits, b_bits, self.D, self.kind,
                           self.pivot_ok)


@dataclass
class SortResult:
    status: int
    records: List[Record]
    levels: int
    snapshots: List[np.ndarray]


def tree_splitters(sorted_keys: np.ndarray, k: int) -> np.ndarray:
    """R22: the k-1 equidistant order statistics of a sorted sample, as ordering keys."""
    a = np.ascontiguousarray(sorted_keys)
    out = np.zeros(k - 1, np.uint64)
    lib().oracle_tree_splitters(_ptr(a), a.size, k, _key_type(a), _ptr(out))
    return out


def tree_bucket(x, spl_ok: np.ndarray, k: int) -> int:
    """R23: leaf of the splitter tree for one key (float64 or uint64 scalar)."""
    a = np.asarray([x])
    if a.dtype not in (np.float64, np.uint64):
        a = a.astype(np.float64)
    s = np.ascontiguousarray(spl_ok, dtype=np.uint64)
    return int(lib().oracle_tree_bucket(int(a.view(np.uint64)[0]), _key_type(a), _ptr(s), k))


def tree_eq_bucket(x, spl_ok: np.ndarray, leaves: int) -> int:
    """R24: bucket (of 2 * leaves) of one key under the tree with equality buckets."""
    a = np.asarray([x])
    if a.dtype not in (np.float64, np.uint64):
        a = a.astype(np.float64)
    s = np.ascontiguousarray(spl_ok, dtype=np.uint64)
    return int(lib().oracle_tree_eq_bucket(int(a.view(np.uint64)[0]), _key_type(a), _ptr(s), leaves))


def sort(keys: np.ndarray, k: int = 256, base_case: int = 4096, seed: int = DEFAULT_SEED,
         trace: bool = False, snapshots: bool = False, model: int = MODEL_LINEAR) -> SortResult:
    """Sort ``keys`` (float64 or uint64 numpy array) IN PLACE with the oracle; ``model``
    MODEL_LINEAR (FMCD, IPLS), MODEL_TREE (splitter tree, IPS4o's classifier) or MODEL_TREE_EQ (the
    tree with equality buckets, R24)."""
    if not keys.flags.c_contiguous:
        raise ValueError("keys must be C-contiguous")
    kt = _key_type(keys)
    L = lib()
    tr = L.oracle_trace_new(1 if snapshots else 0) if (trace or snapshots) else None
    try:
        st = L.oracle_sort_model(_ptr(keys), keys.size, kt, k, base_case, seed, model, tr)
        recs: List[Record] = []
        snaps: List[np.ndarray] = []
        levels = 0
        if tr:
            levels = int(L.oracle_trace_num_levels(tr))
            for i in range(L.oracle_trace_num_records(tr)):
                r = _Rec()
                L.oracle_trace_record(tr, i, ctypes.byref(r))
                sp = L.oracle_trace_sample(tr, i)
                cp = L.oracle_trace_counts(tr, i)
                smp = np.ctypeslib.as_array((ctypes.c_uint64 * r.S).from_address(sp)).copy() \
                    if r.S else np.zeros(0, np.uint64)
                cnt = np.ctypeslib.as_array((ctypes.c_uint64 * r.k_eff).from_address(cp)).copy()
                recs.append(Record(r.level, r.kind, r.begin, r.m, r.S, r.A, r.B, r.D, r.capped,
                                   r.pivot_ok, r.k_eff, r.requeued, smp, cnt))
            if snapshots:
                for lv in range(levels):
                    p = L.oracle_trace_snapshot(tr, lv)
                    snaps.append(np.ctypeslib.as_array(
                        (ctypes.c_uint64 * keys.size).from_address(p)).copy())
        return SortResult(int(st), recs, levels, snaps)
    finally:
        if tr:
            L.oracle_trace_free(tr)


def level_digests(records: List[Record]) -> List[str]:
    """SHA-256 (first 16 hex) per level over the 48-byte records in increasing begin order."""
    by_level = {}
    for r in records:
        by_level.setdefault(r.level, []).append(r)
    out = []
    for lv in sorted(by_level):
        h = hashlib.sha256()
        for r in sorted(by_level[lv], key=lambda r: r.begin):
            h.update(r.packed())
        out.append(h.hexdigest()[:16])
    return out
