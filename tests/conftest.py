"""Test configuration: `gpu` marker, in-tree builds, shared helpers on sys.path."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a path)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Make sure libvrte.so and the oracle library exist (incremental builds)."""
    from paper_1707_05882_b200 import build as B
    import pyoracle
    lib = B.LIB
    if not os.path.exists(lib):
        B.build()
    if not os.path.exists(pyoracle.LIB_PATH):
        pyoracle.build()
    yield
