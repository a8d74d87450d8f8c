"""CPU-side checks of the drop-in boundary: the C ABI library loads and exports
every symbol include/ctb200.h declares (no compute without a GPU)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def header_functions():
    text = (ROOT / "include" / "ctb200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ctb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = header_functions()
    for must in ("ctb_ctx_create", "ctb_ntt_forward", "ctb_ntt_inverse", "ctb_cpmul", "ctb_pp_mul", "ctb_ring_mul"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2409_16675_b200 import _lib
    if not _lib.LIB_PATH.exists():
        from paper_2409_16675_b200 import build
        build.build()
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in header_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes binding covers exactly the header
    assert sorted(_lib.SIGNATURES) == header_functions()


def test_version_and_error_without_gpu():
    from paper_2409_16675_b200 import _lib
    lib = _lib.load()
    assert lib.ctb_version() >= 1
    h = ctypes.c_void_p()
    # invalid degree is rejected before touching the device
    rc = lib.ctb_ctx_create(ctypes.byref(h), 3, _lib.u64_array([17]), 1, _lib.u64_array([]), 0, 16)
    assert rc == _lib.CTB_ERR_ARG
    assert b"power of two" in lib.ctb_last_error()
