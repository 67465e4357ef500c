"""CPU checks of the C-ABI boundary: the library loads and exports exactly
what include/minions.h declares (no kernel is launched here)."""
import ctypes
import os
import re

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "minions.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ms_\w+)\s*\(", src)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("ms_vote", "ms_accept_greedy", "ms_argmax_rows", "ms_linear", "ms_attention",
              "ms_linear_splits", "ms_draft_commit", "ms_pack_verify"):
        assert s in syms, s


def test_library_exports_every_declared_symbol():
    from paper_2402_15678_b200 import _native
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # the Python binding declares a signature for every header symbol
    assert set(declared_symbols()) == set(_native.exported_symbols())


def test_status_codes_map_to_reference_errors():
    from paper_2402_15678_b200 import _native
    from paper_2402_15678_b200.core import DistMismatch, LengthMismatch
    import pytest
    assert _native.lib.ms_version() >= 100
    for code, exc in ((-1, ValueError), (-2, LengthMismatch), (-3, DistMismatch),
                      (-4, NotImplementedError), (-5, RuntimeError)):
        with pytest.raises(exc):
            _native.check(code, "probe")


def test_kernels_are_sm100a_cubins():
    """The fatbin carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    from paper_2402_15678_b200 import _native
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
