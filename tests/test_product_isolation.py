"""The product path never reaches the oracle and has no CPU fallback (task rule ③).

* No module of the package imports `oracle`, and no CUDA/C++ source includes or links it.
* `oracle/` imports nothing from the package except the seeded input generators' module
  (`datagen`, which holds none of the method's arithmetic).
* With the native library missing, every entry point raises instead of computing.
"""
import ast
import glob
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2208_06902_b200")


def _imports(path):
    tree = ast.parse(open(path).read(), path)
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            for a in node.names:
                yield a.name
        elif isinstance(node, ast.ImportFrom):
            yield (node.module or "")


def test_package_never_imports_the_oracle():
    for py in glob.glob(os.path.join(PKG, "*.py")):
        assert not any(m == "oracle" or m.startswith("oracle.") for m in _imports(py)), py


def test_native_sources_do_not_include_the_oracle():
    for src in glob.glob(os.path.join(PKG, "csrc", "*")) + glob.glob(os.path.join(ROOT, "include", "*")):
        text = open(src).read()
        assert "ipls_oracle" not in text and "oracle/" not in text, src


def test_oracle_imports_only_datagen_from_the_package():
    for py in glob.glob(os.path.join(ROOT, "oracle", "*.py")):
        for m in _imports(py):
            if m.startswith("paper_2208_06902_b200"):
                assert m in ("paper_2208_06902_b200.datagen",), (py, m)


def test_missing_library_raises(monkeypatch):
    import paper_2208_06902_b200 as ipls
    monkeypatch.setattr(ipls, "_lib", None)
    monkeypatch.setattr(ipls, "_LIB_PATH", os.path.join(PKG, "does_not_exist.so"))
    with pytest.raises(ipls.IPLSError):
        ipls.lib()
    with pytest.raises(ipls.IPLSError):
        ipls.sample_size(100, 4)
    with pytest.raises(ipls.IPLSError):
        ipls.assign_ranges([1, 2, 3], 2)
