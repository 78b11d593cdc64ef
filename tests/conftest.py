import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")


@pytest.fixture(scope="session")
def lib():
    """The in-tree C-ABI library (built on demand; nvcc cross-compiles)."""
    from paper_1812_10624_b200.build import build_library
    from paper_1812_10624_b200 import _lib
    build_library()
    return _lib.load()


@pytest.fixture(params=[1, 0], ids=["tma", "cp.async"])
def producer(request, lib):
    """Run a GPU op test under both GEMM producers (TMA tensor maps and the
    cp.async gather); restore TMA afterwards."""
    lib.stz_set_tma(request.param)
    yield request.param
    lib.stz_set_tma(1)


@pytest.fixture(params=[1, 0], ids=["cluster2", "cta1"])
def clusters(request, lib):
    """Run with CTA-pair (cta_group::2) GEMMs and with single CTAs; restore after."""
    lib.stz_set_cluster(request.param)
    yield request.param
    lib.stz_set_cluster(1)
