"""CPU-side checks of the C-ABI library: it builds, loads and exports the header (no compute)."""

import ctypes as C

import numpy as np
import pytest

from paper_2512_02281_b200 import _lib


def test_library_exports_every_header_symbol():
    lib = _lib.load_library()
    syms = _lib.header_symbols()
    assert len(syms) >= 25
    for name in syms:
        assert hasattr(lib, name), f"{name} declared in include/trinity_b200.h but not exported"
    assert set(syms) == set(_lib._SIGS), "ctypes signature table out of sync with the header"


def test_version_and_error_plumbing():
    lib = _lib.load_library()
    assert lib.tri_version() == 1
    with pytest.raises(ValueError, match="unknown option"):
        _lib.set_option("no_such_option", 1)
    assert b"unknown option" in lib.tri_last_error()


def test_option_ranges_validated():
    """Tuning knobs reject out-of-range values (host-side, no device work)."""
    for name, bad in (("scan_abufs", 3), ("scan_qbufs", 0), ("fx_slice_rows", 8), ("coarse_split", 0),
                      ("tc_box_rows", 48)):
        with pytest.raises(ValueError):
            _lib.set_option(name, bad)
    for name, good, default in (("scan_abufs", 2, 1), ("pack_mixed", 0, 1), ("scan_l2hint", 2, 1),
                                ("scan_reserve", 16, -1), ("rerank_skip", 0, 1), ("fx_slice_rows", 512, 256)):
        _lib.set_option(name, good)
        _lib.set_option(name, default)


def test_invalid_arguments_rejected_before_device_work():
    lib = _lib.load_library()
    h = C.c_void_p()
    x = np.zeros((0, 4), np.float32)
    rc = lib.tri_store_create(x.ctypes.data, 0, 4, 0, C.byref(h))
    assert rc == _lib.TRI_EINVAL and b"nonempty" in lib.tri_last_error()
    x = np.array([[np.nan, 1.0]], np.float32)
    rc = lib.tri_store_create(x.ctypes.data, 1, 2, 0, C.byref(h))
    assert rc == _lib.TRI_EINVAL and b"finite" in lib.tri_last_error()


def test_no_cpu_fallback_without_gpu():
    """On a CPU-only host every compute entry point fails loudly."""
    n = C.c_int32(-1)
    _lib.load_library().tri_device_count(C.byref(n))
    if n.value > 0:
        pytest.skip("a GPU is visible")
    from paper_2512_02281_b200 import VectorStore, brute_force_knn

    store = VectorStore(data=np.eye(3, dtype=np.float32))
    with pytest.raises(RuntimeError, match="no CUDA device"):
        brute_force_knn(store, np.zeros(3), 1)
