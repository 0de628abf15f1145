"""CPU: the C-ABI library loads, exports every symbol include/vr_capi.h declares,
and its struct layouts match the ctypes mirrors (no compute calls)."""
import ctypes
import re
from pathlib import Path

import pytest

from paper_2404_16221_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "vr_capi.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vr_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    assert "vr_sample_count" in syms and "vr_global_train" in syms
    assert len(syms) >= 20


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    assert set(declared_symbols()) == set(_lib.SIGNATURES), \
        set(declared_symbols()) ^ set(_lib.SIGNATURES)


def test_struct_layouts_and_version():
    lib = _lib.load()
    assert lib.vr_abi_version() == 1
    sizes = (ctypes.c_int64 * 5)()
    assert lib.vr_struct_sizes(sizes) == 0
    assert list(sizes) == [ctypes.sizeof(_lib.VrTree), ctypes.sizeof(_lib.VrAnalyticField),
                           ctypes.sizeof(_lib.VrVoxelDesc), ctypes.sizeof(_lib.VrHashGridDesc),
                           ctypes.sizeof(_lib.VrBlob)]


def test_bad_arguments_are_rejected_without_a_gpu():
    lib = _lib.load()
    t = _lib.VrTree()
    t.n_leaves = 0  # invalid
    rc = lib.vr_sample_count(ctypes.addressof(t), None, 0, 1, 0.1, 0, 1, None, None, None, None,
                             None, None, None, None)
    assert rc == 1
    assert b"bad argument" in lib.vr_last_error()
    with pytest.raises(ValueError):
        _lib.call("vr_segment_fwd", None, None, None, None, None, None, 4, 0, None, None, None,
                  0, None)


def test_header_constants_match_ctypes_mirror():
    """Every #define VR_* integer of the header has the same value in _lib."""
    defs = dict(re.findall(r"#define\s+(VR_[A-Z0-9_]+)\s+(-?\d+)\b", HEADER.read_text()))
    assert "VR_SUM_PARTIALS" in defs and "VR_MAX_REGIONS" in defs
    mirrored = {k: v for k, v in defs.items() if hasattr(_lib, k)}
    assert len(mirrored) >= 8
    for k, v in mirrored.items():
        assert getattr(_lib, k) == int(v), k
