import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def gemm_tol(k: int) -> float:
    """Tolerance (rel_err against the float64 oracle) of one BF16x6 GEMM with
    contraction length k.  The product sums are exact; the error is the
    tcgen05 accumulator's truncation when it adds each 16-deep MMA into the
    big b0*b0 accumulator, up to 1 ulp per MMA.  The library
    caps one work item at K = 4096 (split-K beyond), so the worst-case bias is
    ceil(min(k, 4096) / 16) * 2^-23 of the output max; the tolerance is half
    of that (measured errors sit at about a fifth), floored at 3e-6."""
    import math
    return max(3e-6, 0.5 * math.ceil(min(k, 4096) / 16) * 2.0 ** -23)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")


@pytest.fixture(scope="session")
def lib():
    """The in-tree C-ABI library (built on demand; nvcc cross-compiles)."""
    from paper_1812_10624_b200.build import build_library
    from paper_1812_10624_b200 import _lib
    build_library()
    return _lib.load()


@pytest.fixture(params=[1, 2, 0], ids=["tma", "tma2d", "cp.async"])
def producer(request, lib):
    """Run a GPU op test under every GEMM producer (TMA tensor maps with 3D
    MN-major boxes, TMA with 2D boxes only, and the cp.async gather);
    restore the default afterwards."""
    lib.stz_set_tma(request.param)
    yield request.param
    lib.stz_set_tma(1)


@pytest.fixture(params=[1, 0], ids=["cluster2", "cta1"])
def clusters(request, lib):
    """Run with CTA-pair (cta_group::2) GEMMs and with single CTAs; restore after."""
    lib.stz_set_cluster(request.param)
    yield request.param
    lib.stz_set_cluster(1)
