"""The C-ABI library loads and exports every symbol include/fluxattn_b200.h
declares (no compute: this runs on the CPU-only container too)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fluxattn_b200.h")).read()
    return sorted(set(re.findall(r"^FX_API [^(]*?\b(fx_\w+)\(", src, flags=re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "fx_decode_step" in syms and "fx_build_metadata_levels" in syms
    assert len(syms) >= 25


def test_library_exports_every_declared_symbol():
    from paper_2605_07719_b200 import _native
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding covers exactly the header
    assert sorted(_native.EXPORTED) == declared_symbols()


def test_abi_version_and_errors_without_gpu():
    from paper_2605_07719_b200 import _native
    assert _native.LIB.fx_abi_version() == _native.ABI_VERSION == 5
    assert _native.LIB.fx_block_count(33, 16) == 3
    assert _native.LIB.fx_block_count(10, 0) == 0


def test_sm100a_cubin_present():
    """The library carries sm_100a SASS (checked with cuobjdump when available)."""
    import shutil
    import subprocess
    from paper_2605_07719_b200 import _native
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        return
    out = subprocess.run([exe, "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
