"""ctypes binding of libtrinity_b200.so (the C-ABI in include/trinity_b200.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is visible, every compute entry point raises RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libtrinity_b200.so")
HEADER = os.path.join(os.path.dirname(PKG), "include", "trinity_b200.h")

TRI_OK, TRI_EINVAL, TRI_EINTERNAL, TRI_ECUDA = 0, 1, 2, 3
TRI_MAX_K = 1638

_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_f64p = C.POINTER(C.c_double)
_f32p = C.POINTER(C.c_float)
_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)

# name -> argtypes (restype is int unless listed in _RESTYPE)
_SIGS = {
    "tri_last_error": [],
    "tri_version": [],
    "tri_graph_counters": [_i64p, _i64p, _i64p],
    "tri_device_count": [_i32p],
    "tri_set_option": [C.c_char_p, _i64],
    "tri_store_create": [_vp, _i64, _i32, _i32, C.POINTER(_vp)],
    "tri_store_destroy": [_vp],
    "tri_store_info": [_vp, _i64p, _i32p, _f64p],
    "tri_store_set_id_offset": [_vp, _i64],
    "tri_knn_bruteforce": [_vp, _vp, _i32, _vp, _i32, _vp, _vp, _vp],
    "tri_knn_bruteforce_dev": [_vp, _vp, _i32, _vp, _i32, _vp, _vp, _vp],
    "tri_rowwise_sq_dists": [_vp, _vp, _vp, _i64, _vp, _vp],
    "tri_rowwise_sq_dists_f64": [_vp, _i32, _vp, _i64, _i32, _i32, _vp],
    "tri_distance_tasks": [_vp, _vp, _vp, _i32, _vp, _i32, _vp, _vp],
    "tri_ivf_train": [_vp, _i32, _i32, _vp, C.POINTER(_vp)],
    "tri_kmeans_assign": [_vp, _vp, _i32, _vp],
    "tri_ivf_create": [_vp, _vp, _i32, _vp, _i64, C.POINTER(_vp)],
    "tri_ivf_destroy": [_vp],
    "tri_ivf_info": [_vp, _i32p, _i64p, _i32p],
    "tri_ivf_export": [_vp, _vp, _vp],
    "tri_ivf_list_sizes": [_vp, _vp],
    "tri_ivf_search": [_vp, _vp, _i32, _vp, _vp, _i32, _vp, _vp, _vp],
    "tri_ivf_search_dev": [_vp, _vp, _i32, _vp, _vp, _i32, _vp, _vp, _vp],
    "tri_ivf_last_probes": [_vp, _vp, _i32],
    "tri_ivf_last_fixups": [_vp, _i32p],
    "tri_store_last_fixups": [_vp, _i32p],
    "tri_ivf_set_profiling": [_vp, _i32],
    "tri_ivf_scan_time": [_vp, _f64p, _i32p],
    "tri_ivf_stage_times": [_vp, _vp, _i32p],
    "tri_ivf_last_scan_bytes": [_vp, _i64p, _i64p],
    "tri_ivf_last_scan_kind": [_vp, _i32p],
    "tri_engine_create": [_vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _i32, C.POINTER(_vp)],
    "tri_engine_destroy": [_vp],
    "tri_engine_submit": [_vp, _vp, _i32, _i64p],
    "tri_engine_counts": [_vp, _i32p, _i32p],
    "tri_engine_request_state": [_vp, _i64, _i32p, _i32p, _vp, _vp, _vp, _vp, _i32p, _i32p],
    "tri_engine_submit_batch": [_vp, _vp, _i32, _vp, _vp],
    "tri_engine_device_time": [_vp, _f64p, _i64p],
    "tri_engine_run": [_vp, _i32, _i32, _i32p, _vp, _vp, _vp],
    "tri_engine_retired": [_vp, _i32, _i32, _i32p, _vp, _vp, _vp, _vp, _vp, _vp],
    "tri_engine_retired_by_id": [_vp, _i64, _i32, _i32p, _vp, _vp, _vp, _vp, _vp],
    "tri_engine_pending_retired": [_vp, _i32p],
    "tri_debug_bound": [_i32, _i32, _f64p, _f64p],
    "tri_ivf_debug_keys": [_vp, _i32, _vp, _i64, _i64p, _vp],
    "tri_debug_scan_ts": [_vp, _i32],
    "tri_merge_topk": [_vp, _vp, _i32, _i32, _i32, _i32, _vp, _vp, _vp],
    "tri_merge_topk_ld": [_vp, _vp, _i32, _i32, _i32, _i32, _i64, _i32, _vp, _vp, _i32, _vp],
    "tri_comm_unique_id": [_vp],
    "tri_comm_init": [_vp, _i32, _i32, _i32, C.POINTER(_vp)],
    "tri_comm_destroy": [_vp],
    "tri_ivf_search_sharded": [_vp, _vp, _vp, _i32, _i32, _vp, _i32, _vp, _vp, _vp],
}
_RESTYPE = {"tri_last_error": C.c_char_p}

_lib = None


def header_symbols() -> list[str]:
    """Every function the public header declares."""
    with open(HEADER) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+(tri_\w+)\s*\(", text, flags=re.M)))


def load_library() -> C.CDLL:
    """Load the shared library (no device needed); raise loudly if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the B200 path has no CPU fallback)"
        )
    lib = C.CDLL(LIB_PATH)
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, C.c_int)
    _lib = lib
    return lib


def check(rc: int) -> None:
    if rc == TRI_OK:
        return
    msg = (load_library().tri_last_error() or b"").decode(errors="replace")
    if rc == TRI_EINVAL:
        raise ValueError(msg)
    if rc == TRI_EINTERNAL:
        raise RuntimeError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


_gpu_ok = None


def gpu() -> C.CDLL:
    """The library, after asserting a CUDA device exists (no CPU fallback)."""
    global _gpu_ok
    lib = load_library()
    if _gpu_ok is None:
        n = C.c_int32(0)
        lib.tri_device_count(C.byref(n))
        _gpu_ok = n.value > 0
    if not _gpu_ok:
        raise RuntimeError("no CUDA device visible: the Trinity B200 search path has no CPU fallback")
    return lib


def ptr(a) -> int:
    """Address of a numpy array's data or a torch tensor's storage."""
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


def graph_counters() -> dict:
    """Process-wide whole-search executions: eager, graph captures, graph replays."""
    e, c, r = C.c_int64(0), C.c_int64(0), C.c_int64(0)
    check(load_library().tri_graph_counters(C.byref(e), C.byref(c), C.byref(r)))
    return {"eager": e.value, "captured": c.value, "replayed": r.value}


def set_option(name: str, value: int) -> None:
    check(load_library().tri_set_option(name.encode(), int(value)))
