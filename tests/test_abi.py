"""The C-ABI library: builds for sm_100a, loads, exports every declared symbol."""
import os
import re

from conftest import ROOT


def test_library_exports_header_symbols(native_lib):
    hdr = open(os.path.join(ROOT, "include", "hybridwave_b200.h")).read()
    names = set(re.findall(r"\b(hw_[a-z0-9_]+)\s*\(", hdr))
    names -= {n for n in names if n.startswith("hw_nbr")}
    assert {"hw_rhs", "hw_lsrk_stage", "hw_ab_step"} <= names
    for n in names:
        assert hasattr(native_lib, n), n
    assert native_lib.hw_version() >= 1
    orders = native_lib.hw_supported_orders()
    assert all((orders >> n) & 1 for n in range(1, 8))


def test_sass_is_sm100a(native_lib):
    import subprocess
    from paper_1507_02557_b200 import _native
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
