"""The C-ABI library builds (nvcc cross-compiles here), loads, and exports
every symbol include/stanza_b200.h declares; no compute without a GPU."""

import os
import subprocess

from paper_1812_10624_b200 import _lib
from paper_1812_10624_b200.build import LIB_PATH


def test_header_symbols_exported(lib):
    declared = _lib.header_symbols()
    assert len(declared) >= 18
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing
    assert set(declared) == set(_lib.SIGNATURES), "ctypes table must match the header"
    out = subprocess.run(["nm", "-D", LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(declared) <= exported


def test_version_and_control_calls(lib):
    assert lib.stz_abi_version() == 2
    assert lib.stz_set_max_k_per_split(-1) == 1         # invalid -> ShapeMismatch code
    assert b"max_k_per_split" in lib.stz_last_error()
    assert lib.stz_set_max_k_per_split(0) == 0


def test_sm100a_code_in_library(lib):
    sass = subprocess.run(["cuobjdump", "-sass", LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "UTCHMMA" in sass or "UTCQMMA" in sass     # tcgen05.mma
    assert "LDTM" in sass                              # tcgen05.ld
    assert os.path.getsize(LIB_PATH) > 100_000
