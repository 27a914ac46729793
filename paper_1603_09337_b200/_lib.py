"""ctypes binding of libtoposmooth_b200.so (the C ABI in include/toposmooth_b200.h).

The product path has no CPU fallback: if the shared library is missing (and
cannot be built) or no CUDA device is present, every device call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TS_LIB_PATH") or os.path.join(HERE, "libtoposmooth_b200.so")

TS_OK, TS_ERR_VALUE, TS_ERR_CUDA, TS_ERR_INTERNAL, TS_ERR_UNSUPPORTED = 0, 1, 2, 3, 4

_lib = None
_lock = threading.Lock()

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64

# name -> (argtypes, restype); every symbol include/toposmooth_b200.h declares
SIGNATURES = {
    "ts_version": ([], ctypes.c_int),
    "ts_last_error": ([], ctypes.c_char_p),
    "ts_max_radius": ([], ctypes.c_int),
    "ts_hasf_batch": ([_vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp], ctypes.c_int),
    "ts_hasf_batch_host": ([_vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp], ctypes.c_int),
    "ts_hasf_batch_async": ([_vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp, _vp], ctypes.c_int),
    "ts_check_device_error": ([_i32], ctypes.c_int),
    "ts_cutting_batch": ([_vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp], ctypes.c_int),
    "ts_filling_batch": ([_vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp], ctypes.c_int),
    "ts_thin_batch": ([_vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _i64, _vp], ctypes.c_int),
    "ts_thicken_batch": ([_vp, _vp, _vp, _vp, _i64, _i32, _i32, _i32, _i64, _vp], ctypes.c_int),
    "ts_edt_sq_batch": ([_vp, _vp, _i64, _i32, _i32, _i32, _vp], ctypes.c_int),
    "ts_edt_phase1_batch": ([_vp, _vp, _i64, _i32, _i32, _vp], ctypes.c_int),
    "ts_edt_phase2_batch": ([_vp, _vp, _i64, _i32, _i32, _vp], ctypes.c_int),
    "ts_dilate_batch": ([_vp, _vp, _i64, _i32, _i32, _i32, _vp], ctypes.c_int),
    "ts_erode_batch": ([_vp, _vp, _i64, _i32, _i32, _i32, _vp], ctypes.c_int),
    "ts_neighborhood_codes_batch": ([_vp, _vp, _i64, _i32, _i32, _vp], ctypes.c_int),
    "ts_simple_point_mask_batch": ([_vp, _vp, _i64, _i32, _i32, _i32, _vp], ctypes.c_int),
    "ts_connectivity_tables": ([_vp, _vp, _vp, _vp], ctypes.c_int),
    "ts_component_counts_batch": ([_vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _vp], ctypes.c_int),
    "ts_selftest_circuit": ([_vp, _vp], ctypes.c_int),
    "ts_p4_to_rows": ([_vp, _vp, _i64, _i32, _i32, _vp], ctypes.c_int),
    "ts_rows_to_p4": ([_vp, _vp, _i64, _i32, _i32, _vp], ctypes.c_int),
    "ts_hasf_batch_p4": ([_vp, _vp, _i64, _i32, _i32, _i32, _i32, _vp, _vp, _vp], ctypes.c_int),
    "ts_set_smem_budget": ([_i64], _i64),
    "ts_set_dense_divisor": ([_i32], _i32),
    "ts_set_team_size": ([_i32], _i32),
    "ts_set_cluster_teams": ([_i32], _i32),
    "ts_set_cta_threads": ([_i32], _i32),
    "ts_set_host_streaming": ([_i32], _i32),
    "ts_set_fused_prep": ([_i32], _i32),
    "ts_set_segment_stages": ([_i32], _i32),
    "ts_set_segment_fine": ([_i32], _i32),
    "ts_set_segment_force": ([_i32], _i32),
    "ts_set_host_segments": ([_i32, _i32], _i32),
    "ts_set_trace": ([_vp, _i64], None),
    "ts_hasf_plan": ([_i32, _i32, _i32, _i32, _i32, _vp], ctypes.c_int),
}


def load(build_if_missing: bool = True):
    """Load (building in-tree with nvcc if needed) the shared library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if build_if_missing and not os.environ.get("TS_LIB_PATH"):
            from . import build as _build
            if _build.needs_build():
                _build.build()
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA library missing: {LIB_PATH} (run python -m paper_1603_09337_b200.build)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (argt, rest) in SIGNATURES.items():
            if os.environ.get("TS_LIB_PATH") and not hasattr(lib, name):
                continue   # A/B against an older experimental build
            fn = getattr(lib, name)
            fn.argtypes = argt
            fn.restype = rest
        _lib = lib
        return lib


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's exception classes."""
    if rc == TS_OK:
        return
    msg = load().ts_last_error().decode(errors="replace")
    if rc == TS_ERR_VALUE:
        raise ValueError(msg)
    raise RuntimeError(f"toposmooth_b200 error {rc}: {msg}")
