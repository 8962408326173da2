"""ctypes binding of libdbtsdf.so (include/dbtsdf.h).

The engine is the only compute path: if the shared library is missing or no
CUDA device is usable, every entry point raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import CODE_TO_ERROR, BitsdfError

# $DBT_LIB: another build of the engine (same-box A/B measurements only)
LIB_PATH = Path(os.environ.get("DBT_LIB") or Path(__file__).resolve().parent / "libdbtsdf.so")

DBT_F32 = 0
DBT_F64 = 1
FLAG_MAP_FRAME = 1
FLAG_SKIP_NORM_CHECK = 2
FLAG_NO_DEDUP = 4
FLAG_NO_SKIP = 8
FLAG_FUSE_SHADOW = 16
FLAG_GENERIC_SWEEP = 32
FLAG_STAGE_COPY = 64
FLAG_EXACT_WRITTEN = 128

_c_i64p = ctypes.POINTER(ctypes.c_int64)
_c_dp = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p


class Params(ctypes.Structure):
    _fields_ = [
        ("h_max", ctypes.c_int32),
        ("t_occ", ctypes.c_int32),
        ("downsample", ctypes.c_int32),
        ("first_return", ctypes.c_int32),
        ("flags", ctypes.c_uint32),
        ("reserved", ctypes.c_int32),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("points_in", ctypes.c_int64),
        ("points_discarded", ctypes.c_int64),
        ("voxels_written", ctypes.c_int64),
        ("points_applied", ctypes.c_int64),
        ("unique_centers", ctypes.c_int64),
        ("centers_skipped", ctypes.c_int64),
        ("bin_fallbacks", ctypes.c_int64),
        ("elapsed_ms", ctypes.c_double),
        ("device_ms", ctypes.c_double),
        ("rows_swept", ctypes.c_int64),
    ]


class Deskew(ctypes.Structure):
    """dbt_deskew: per-scan constants of the device motion compensation."""
    _fields_ = [
        ("mode", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("q", ctypes.c_double * 4),
        ("rv", ctypes.c_double * 3),
        ("y0", ctypes.c_double),
        ("dy", ctypes.c_double),
        ("t0", ctypes.c_double * 3),
        ("t1", ctypes.c_double * 3),
        ("r1", ctypes.c_double * 9),
    ]


DESKEW_YAW, DESKEW_SE3 = 1, 2

# name -> (restype, argtypes); mirrors include/dbtsdf.h one to one
SIGNATURES = {
    "dbt_last_error": (ctypes.c_char_p, []),
    "dbt_version": (ctypes.c_char_p, []),
    "dbt_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "dbt_grid_create": (ctypes.c_int, [_c_i64p, ctypes.c_double, _c_dp, ctypes.c_int, ctypes.c_int64,
                                       ctypes.c_int64, ctypes.POINTER(_vp)]),
    "dbt_grid_create_interleaved": (ctypes.c_int, [_c_i64p, ctypes.c_double, _c_dp, ctypes.c_int, ctypes.c_int64,
                                                   ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(_vp)]),
    "dbt_grid_layout": (ctypes.c_int, [_vp, _c_i64p, _c_i64p]),
    "dbt_grid_destroy": (ctypes.c_int, [_vp]),
    "dbt_grid_reset": (ctypes.c_int, [_vp]),
    "dbt_grid_info": (ctypes.c_int, [_vp, _c_i64p, _c_i64p, _c_i64p]),
    "dbt_grid_upload": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "dbt_grid_download": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "dbt_grid_download_range": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, _vp, _vp, _vp]),
    "dbt_grid_to_records": (ctypes.c_int, [_vp, _vp]),
    "dbt_grid_from_records": (ctypes.c_int, [_vp, _vp]),
    "dbt_probe_l2": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.POINTER(ctypes.c_double)]),
    "dbt_grid_to_records_range": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, _vp]),
    "dbt_grid_from_records_range": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int64, _vp]),
    "dbt_grid_gather": (ctypes.c_int, [_vp, _vp, ctypes.c_int64, _vp, _vp, _vp]),
    "dbt_popcount": (ctypes.c_int, [_vp, _vp]),
    "dbt_observed": (ctypes.c_int, [_vp, _vp]),
    "dbt_signed_distance_field": (ctypes.c_int, [_vp, _vp, _vp]),
    "dbt_grid_counts": (ctypes.c_int, [_vp, _c_i64p, _c_i64p]),
    "dbt_bank_create": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _vp, _vp, _vp, ctypes.c_int,
                                       ctypes.POINTER(_vp)]),
    "dbt_bank_destroy": (ctypes.c_int, [_vp]),
    "dbt_integrate_frame": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int64, _vp,
                                           ctypes.POINTER(Params), ctypes.POINTER(Stats)]),
    "dbt_integrate_batch": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, _c_i64p, ctypes.c_int32, _vp,
                                           ctypes.POINTER(Params), ctypes.POINTER(Stats)]),
    "dbt_integrate_scans": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, _c_i64p, ctypes.c_int32, _vp,
                                           ctypes.POINTER(Params), ctypes.POINTER(Stats)]),
    "dbt_integrate_points_map": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_int64, ctypes.POINTER(Params),
                                                ctypes.POINTER(Stats), _vp]),
    "dbt_integrate_device": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, _c_i64p, ctypes.c_int32, _vp,
                                            ctypes.POINTER(Params), _vp]),
    "dbt_stats_read": (ctypes.c_int, [_vp, ctypes.POINTER(Stats), ctypes.c_int32]),
    "dbt_synchronize": (ctypes.c_int, [_vp]),
    "dbt_grid_stream": (ctypes.c_int, [_vp, ctypes.POINTER(_vp)]),
    "dbt_bin_index_array": (ctypes.c_int, [_vp, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _vp, _vp,
                                           ctypes.c_int]),
    "dbt_profile_enable": (ctypes.c_int, [_vp, ctypes.c_int]),
    "dbt_profile_read": (ctypes.c_int, [_vp, ctypes.c_char_p, _c_dp, _c_i64p, ctypes.c_int32,
                                        ctypes.POINTER(ctypes.c_int32)]),
    "dbt_profile_reset": (ctypes.c_int, [_vp]),
    "dbt_launch_count": (ctypes.c_int64, []),
    "dbt_mesh_extract": (ctypes.c_int, [_vp, ctypes.c_double, _vp, ctypes.POINTER(_vp), _c_i64p, _c_i64p]),
    "dbt_mesh_info": (ctypes.c_int, [_vp, _c_i64p, _c_i64p]),
    "dbt_mesh_download": (ctypes.c_int, [_vp, _vp, _vp]),
    "dbt_mesh_device_buffers": (ctypes.c_int, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    "dbt_mesh_destroy": (ctypes.c_int, [_vp]),
    "dbt_mesh_from_host": (ctypes.c_int, [ctypes.c_int, _vp, ctypes.c_int64, _vp, ctypes.c_int64, ctypes.POINTER(_vp)]),
    "dbt_mesh_normals": (ctypes.c_int, [_vp]),
    "dbt_mesh_download_normals": (ctypes.c_int, [_vp, _vp]),
    "dbt_replica_mark": (ctypes.c_int, [_vp]),
    "dbt_replica_pack": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp]),
    "dbt_replica_apply": (ctypes.c_int, [_vp, _vp, _vp, _vp, ctypes.c_int32, ctypes.c_int32, _vp]),
    "dbt_integrate_frame_async": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int64, _vp, _vp, _c_i64p]),
    "dbt_frame_wait": (ctypes.c_int, [_vp, ctypes.c_int64, _vp]),
    "dbt_deskew_available": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int32)]),
    "dbt_integrate_frame_deskew": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int64, _vp, _vp, _vp, _vp,
                                                  _vp]),
    "dbt_deskew_points": (ctypes.c_int, [ctypes.c_int, _vp, ctypes.c_int, ctypes.c_int64, _vp, ctypes.c_int32, _vp,
                                         _vp]),
    "dbt_replica_bricks": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int32)]),
    "dbt_replica_dirty": (ctypes.c_int, [_vp, _vp, _vp]),
    "dbt_replica_select": (ctypes.c_int, [_vp, _vp, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64), _vp]),
    "dbt_replica_pack_bricks": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "dbt_replica_apply_bricks": (ctypes.c_int, [_vp, _vp, _vp, ctypes.c_int32, ctypes.c_int32, _vp]),
    "dbt_host_alloc": (ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(_vp)]),
    "dbt_host_free": (ctypes.c_int, [_vp]),
}

_LIB = None


def lib():
    """Load libdbtsdf.so once. Raises ImportError when it was not built."""
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA engine with "
                "`python -m paper_2509_20081_b200.build` (there is no CPU fallback)"
            )
        L = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def check(rc: int) -> None:
    if rc:
        msg = lib().dbt_last_error().decode(errors="replace")
        raise CODE_TO_ERROR.get(int(rc), BitsdfError)(msg)


def ptr(a: np.ndarray):
    """Address of an array's data as c_void_p (the buffer-protocol path costs
    ~1 us less per call than ndarray.ctypes; read-only or empty arrays take
    the ctypes path)."""
    try:
        return ctypes.c_void_p(ctypes.addressof(ctypes.c_char.from_buffer(a)))
    except (TypeError, ValueError, BufferError):
        return ctypes.c_void_p(a.ctypes.data)


def device_count() -> int:
    n = ctypes.c_int(0)
    rc = lib().dbt_device_count(ctypes.byref(n))
    return int(n.value) if rc == 0 else 0


def default_device() -> int:
    """LOCAL_RANK under torchrun, else 0 (one process per GPU)."""
    return int(os.environ.get("DBT_DEVICE", os.environ.get("LOCAL_RANK", "0")))


_params_cache: dict = {}


# measurement-only engine flags OR-ed into every launch (A/B runs, e.g. DBT_EXTRA_FLAGS=16)
_EXTRA_FLAGS = int(os.environ.get("DBT_EXTRA_FLAGS", "0"), 0)


def make_params(h_max=255, t_occ=2, downsample=1, first_return=False, flags=0) -> Params:
    """dbt_params for these values (cached: the struct is read-only for the engine)."""
    key = (int(h_max), int(t_occ), int(downsample), int(bool(first_return)), int(flags) | _EXTRA_FLAGS)
    p = _params_cache.get(key)
    if p is None:
        p = _params_cache[key] = Params(*key, 0)
    return p
