"""CPU-side checks of the boundary: libipls.so builds for sm_100a, loads, and exports every
entry point include/ipls.h declares.  No compute call (no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "ipls.h")


@pytest.fixture(scope="module")
def native():
    from paper_2208_06902_b200 import build
    build.build()
    import paper_2208_06902_b200 as ipls
    return ipls.lib()


def declared_symbols():
    text = open(HDR).read()
    return sorted(set(re.findall(r"\b(ipls_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["ipls_sort_f64", "ipls_sort_u64", "ipls_sort_ex", "ipls_fit_fmcd",
              "ipls_partition_level", "ipls_workspace_bytes", "ipls_sort_host"]:
        assert s in syms


def test_library_exports_every_declared_symbol(native):
    for s in declared_symbols():
        assert hasattr(native, s), f"libipls.so does not export {s}"
    import paper_2208_06902_b200 as ipls
    assert sorted(ipls.SYMBOLS) == declared_symbols()


def test_cubin_is_sm100a():
    from paper_2208_06902_b200 import build
    out = subprocess.run(["cuobjdump", "--list-elf", build.LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_host_only_calls(native):
    import paper_2208_06902_b200 as ipls
    c = native.ipls_default_config()
    assert (c.k, c.base_case, c.seed, c.flags) == (256, 4096, ipls.DEFAULT_SEED, 0)
    assert native.ipls_status_string(2) == b"NaN key"
    # workspace: one n-key scratch (8n bytes) plus metadata
    w = ipls.workspace_bytes(10 ** 8, ipls.KEY_F64, k=1024, base_case=4096)
    assert 8 * 10 ** 8 < w < 40 * 10 ** 8
    assert ipls.workspace_bytes(10 ** 6, ipls.KEY_F64, k=2) == 0  # k < 3 is invalid
    # argument validation happens before any CUDA call
    assert native.ipls_sort_f64(None, 10, None) == 1
    assert native.ipls_sort_f64(None, 0, None) == 0
    bad = ipls._Config(2, 4096, 1, 0)
    assert native.ipls_sort_ex(None, 0, 0, ctypes.byref(bad), None, 0, None) == 1
    # flags: equality buckets only with the tree model, k a power of two >= 8 (R24)
    for k, flags, ok in [(1024, 1, True), (1024, 3, True), (8, 3, True), (4, 3, False),
                         (1024, 2, False), (1000, 3, False), (1024, 4, False)]:
        c = ipls._Config(k, 4096, 1, flags)
        assert (native.ipls_sort_ex(None, 0, 0, ctypes.byref(c), None, 0, None) == 0) == ok
        assert (native.ipls_workspace_bytes(10 ** 6, 0, ctypes.byref(c)) > 0) == ok


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle (test infrastructure)."""
    pkg = os.path.join(ROOT, "paper_2208_06902_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dp, f)).read()
                assert "import oracle" not in txt and "ipls_oracle" not in txt, f
