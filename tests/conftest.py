import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI on cuda:0)")
    config.addinivalue_line("markers", "slow: full-size CPU oracle runs (minutes)")


def read_golden(name):
    """Parse a whitespace golden file: {first_token: [rest tokens]} (ignores # comments)."""
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            tok = line.split()
            out.setdefault(tok[0], []).append(tok[1:])
    return out


@pytest.fixture(scope="session")
def golden():
    return read_golden
