"""bitsdf/_b200.py — the GPU backend a reference maintainer would add.

Drop this file into the reference package as ``bitsdf/_b200.py``: it keeps
the reference's own objects (``VoxelGrid`` with its in-place numpy
``mask``/``sign``/``hits`` arrays, ``KernelBank``, ``ScanFrame``,
``IntegrationParams``) and moves only the hot path onto the B200 engine
through the C ABI of ``libdbtsdf.so`` (``include/dbtsdf.h``) with ctypes —
no torch, no package from this repository. Entry points, each with the
contract of the reference function it replaces:

* ``integrate_frame(grid, bank, scan, params, threads=1)`` — integrator.py:207-287
* ``integrate_point(grid, bank, p_map, sensor_pos, params)`` — integrator.py:163-189
* ``extract_mesh(grid, iso=0.0)`` — mesher.py:43-110

Wiring it in is one line at the top of ``integrator.integrate_frame``
(``if os.environ.get("BITSDF_B200"): return _b200.integrate_frame(...)``)
or in ``cli.run_fuse`` (cli.py:158). The grid arrays are uploaded before and
downloaded after every call (the reference's in-place semantics); a fuse
loop that does not read them between scans can call ``keep_on_device(grid)``
to upload once and ``sync_to_host(grid)`` at the end.

Inside the reference the imports below resolve relatively; run standalone
(tests/test_integration_shim.py) it falls back to ``bitsdf`` on the path, or
to minimal stand-ins, so the ABI bindings can be checked without it.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass

import numpy as np

try:  # inside the reference package (bitsdf/_b200.py)
    from . import errors as _errors  # type: ignore
    from .integrator import FrameStats, motion_compensate  # type: ignore
except ImportError:  # standalone: the installed reference, else stand-ins
    try:
        from bitsdf import errors as _errors  # type: ignore
        from bitsdf.integrator import FrameStats, motion_compensate  # type: ignore
    except ImportError:
        _errors = None
        motion_compensate = None

        @dataclass
        class FrameStats:  # integrator.py:76-81
            points_in: int = 0
            points_discarded: int = 0
            voxels_written: int = 0
            elapsed_ms: float = 0.0

# --------------------------------------------------------------- the ABI
_LIB_PATH = os.environ.get("BITSDF_B200_LIB", "libdbtsdf.so")
_L = None


def lib(path: str | None = None):
    """Load libdbtsdf.so once ($BITSDF_B200_LIB, else the loader's search
    path) and declare every signature used here."""
    global _L
    if _L is None or path is not None:
        L = ctypes.CDLL(path or _LIB_PATH)
        vp, i64p, dp = ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double)
        sig = {
            "dbt_last_error": (ctypes.c_char_p, []),
            "dbt_grid_create": (ctypes.c_int, [i64p, ctypes.c_double, dp, ctypes.c_int, ctypes.c_int64,
                                               ctypes.c_int64, ctypes.POINTER(vp)]),
            "dbt_grid_destroy": (ctypes.c_int, [vp]),
            "dbt_grid_upload": (ctypes.c_int, [vp, vp, vp, vp]),
            "dbt_grid_download": (ctypes.c_int, [vp, vp, vp, vp]),
            "dbt_bank_create": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, vp, vp, vp,
                                               ctypes.c_int, ctypes.POINTER(vp)]),
            "dbt_bank_destroy": (ctypes.c_int, [vp]),
            "dbt_integrate_frame": (ctypes.c_int, [vp, vp, vp, ctypes.c_int, ctypes.c_int64, dp,
                                                   ctypes.POINTER(Params), ctypes.POINTER(Stats)]),
            "dbt_integrate_points_map": (ctypes.c_int, [vp, vp, vp, vp, ctypes.c_int64, ctypes.POINTER(Params),
                                                        ctypes.POINTER(Stats), vp]),
            "dbt_deskew_available": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int32)]),
            "dbt_integrate_frame_deskew": (ctypes.c_int, [vp, vp, vp, ctypes.c_int, ctypes.c_int64, vp, dp,
                                                          ctypes.POINTER(Deskew), ctypes.POINTER(Params),
                                                          ctypes.POINTER(Stats)]),
            "dbt_mesh_extract": (ctypes.c_int, [vp, ctypes.c_double, ctypes.POINTER(McTables), ctypes.POINTER(vp),
                                                i64p, i64p]),
            "dbt_mesh_download": (ctypes.c_int, [vp, vp, vp]),
            "dbt_mesh_destroy": (ctypes.c_int, [vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _L = L
    return _L


class Params(ctypes.Structure):  # dbt_params, 24 bytes
    _fields_ = [("h_max", ctypes.c_int32), ("t_occ", ctypes.c_int32), ("downsample", ctypes.c_int32),
                ("first_return", ctypes.c_int32), ("flags", ctypes.c_uint32), ("reserved", ctypes.c_int32)]


class Stats(ctypes.Structure):  # dbt_stats, 80 bytes
    _fields_ = [(n, ctypes.c_int64) for n in ("points_in", "points_discarded", "voxels_written", "points_applied",
                                              "unique_centers", "centers_skipped", "bin_fallbacks")] + \
               [("elapsed_ms", ctypes.c_double), ("device_ms", ctypes.c_double), ("rows_swept", ctypes.c_int64)]


class Deskew(ctypes.Structure):  # dbt_deskew, 240 bytes
    _fields_ = [("mode", ctypes.c_int32), ("reserved", ctypes.c_int32), ("q", ctypes.c_double * 4),
                ("rv", ctypes.c_double * 3), ("y0", ctypes.c_double), ("dy", ctypes.c_double),
                ("t0", ctypes.c_double * 3), ("t1", ctypes.c_double * 3), ("r1", ctypes.c_double * 9)]


class McTables(ctypes.Structure):  # dbt_mc_tables
    _fields_ = [("edge_table", ctypes.c_int32 * 256), ("tri_table", ctypes.c_int32 * 4096),
                ("corner_offsets", ctypes.c_int32 * 24), ("edge_base", ctypes.c_int32 * 36),
                ("edge_axis", ctypes.c_int32 * 12)]


DBT_F32, DBT_F64 = 0, 1
FLAG_MAP_FRAME, FLAG_SKIP_NORM_CHECK, FLAG_EXACT_WRITTEN = 1, 2, 128
_CODES = {2: "ConfigurationError", 3: "FormatError", 4: "CorruptionError", 5: "EvaluationError",
          6: "ResourceError"}  # cli.py:34-40


def _check(rc: int):
    if rc:
        msg = (lib().dbt_last_error() or b"").decode()
        cls = getattr(_errors, _CODES.get(rc, "BitsdfError"), None) if _errors is not None else None
        raise (cls or RuntimeError)(msg)


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


class _Handle:
    def __init__(self, ptr, destroy):
        self.ptr, self._destroy = ptr, destroy

    def __del__(self):
        try:
            self._destroy(self.ptr)
        except Exception:  # interpreter shutdown
            pass


# ----------------------------------------------------- reference objects
def device_grid(grid, device: int = 0):
    """dbt_grid mirroring a reference VoxelGrid (created on first use and
    cached on the object, like integrator._shadow_flat_offsets caches its
    table on the bank, integrator.py:129-135)."""
    h = getattr(grid, "_dbt_grid", None)
    if h is None:
        out = ctypes.c_void_p()
        dims = np.array(grid.dims, np.int64)
        org = np.ascontiguousarray(grid.origin, np.float64)
        _check(lib().dbt_grid_create(dims.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), float(grid.voxel_size),
                                     org.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), device, 0,
                                     int(grid.dims[0]), ctypes.byref(out)))
        h = _Handle(out, lib().dbt_grid_destroy)
        grid._dbt_grid = h
        grid._dbt_resident = False
    return h.ptr


def bank_tables(bank):
    """The KernelBank's tables as the C ABI takes them (kernels.py:122-141):
    size^3 uint32 run masks, concatenated int32 (dx,dy,dz) shadow offsets per
    flat bin, int32 counts per bin."""
    dk = np.ascontiguousarray(bank.distance_kernel, np.uint32)
    offs = [np.asarray(o, np.int64).reshape(-1, 3) for o in bank.shadow_offsets]
    xyz = np.ascontiguousarray(np.concatenate(offs) if offs else np.zeros((0, 3)), np.int32)
    cnt = np.array([len(o) for o in offs], np.int32)
    return dk, xyz, cnt


def device_bank(bank, device: int = 0):
    """dbt_bank built from a reference KernelBank (cached on the object)."""
    h = getattr(bank, "_dbt_bank", None)
    if h is None:
        dk, xyz, cnt = bank_tables(bank)
        out = ctypes.c_void_p()
        _check(lib().dbt_bank_create(int(bank.size), int(bank.b_az), int(bank.b_el), _ptr(dk), _ptr(xyz), _ptr(cnt),
                                     device, ctypes.byref(out)))
        h = _Handle(out, lib().dbt_bank_destroy)
        object.__setattr__(bank, "_dbt_bank", h)
    return h.ptr


def _fields(grid):
    arrs = (grid.mask, grid.sign, grid.hits)
    for a, dt in zip(arrs, (np.uint32, np.uint8, np.uint8)):
        if a.dtype != dt or not a.flags.c_contiguous or a.shape != tuple(grid.dims):
            raise ValueError("grid field arrays must be C-contiguous (nx,ny,nz) uint32/uint8/uint8")
    return arrs


def _upload(grid):
    g = device_grid(grid)
    if not getattr(grid, "_dbt_resident", False):
        _check(lib().dbt_grid_upload(g, *(_ptr(a) for a in _fields(grid))))
    return g


def _download(grid):
    if not getattr(grid, "_dbt_resident", False):
        _check(lib().dbt_grid_download(device_grid(grid), *(_ptr(a) for a in _fields(grid))))


def keep_on_device(grid):
    """Upload once; later calls skip the per-call upload/download until
    sync_to_host (nothing may read or write the arrays in between)."""
    _upload(grid)
    grid._dbt_resident = True


def sync_to_host(grid):
    """Download the device grid into the reference arrays (in place) and
    return to per-call transfers."""
    grid._dbt_resident = False
    _download(grid)


def _exact_flag() -> int:
    """DBT_FLAG_EXACT_WRITTEN when $DBT_EXACT_VOXELS_WRITTEN=1: FrameStats.
    voxels_written is then the reference's serial count (integrator.py:
    268-285) instead of the engine's concurrent change count."""
    return FLAG_EXACT_WRITTEN if os.environ.get("DBT_EXACT_VOXELS_WRITTEN") == "1" else 0


def _params(params, flags=0, downsample=None):
    return Params(int(params.h_max), int(params.t_occ), int(params.downsample if downsample is None else downsample),
                  int(bool(params.first_return_per_voxel)), flags, 0)


_DESKEW_OK = None


def _deskew(scan, mode):
    """The point-independent part of motion_compensate (integrator.py:
    91-123), computed with scipy as the reference does; the per-point part
    (pose at each point's time, the move to the end-of-sweep frame, the C
    library's sin/cos restated) runs in the engine's preprocessing."""
    from scipy.spatial.transform import Rotation, Slerp

    global _DESKEW_OK
    if _DESKEW_OK is None:
        ok = ctypes.c_int32()
        _check(lib().dbt_deskew_available(ctypes.byref(ok)))
        _DESKEW_OK = bool(ok.value)
    if not _DESKEW_OK or scan.prev_pose is None:
        return None
    T0, T1 = np.asarray(scan.prev_pose, np.float64), np.asarray(scan.pose, np.float64)
    d = Deskew()
    if mode == "se3":
        s = Slerp([0.0, 1.0], Rotation.from_matrix(np.stack([T0[:3, :3], T1[:3, :3]])))
        d.mode = 2
        d.q[:] = [float(v) for v in s.rotations[0].as_quat(canonical=False)]
        d.rv[:] = [float(v) for v in s.rotvecs[0]]
    else:
        y0 = Rotation.from_matrix(T0[:3, :3]).as_euler("zyx")[0]
        y1 = Rotation.from_matrix(T1[:3, :3]).as_euler("zyx")[0]
        tilt = Rotation.from_euler("z", -y1) * Rotation.from_matrix(T1[:3, :3])
        d.mode = 1
        d.q[:] = [float(v) for v in np.asarray(tilt.as_quat(canonical=False)).reshape(4)]
        d.y0, d.dy = float(y0), float((y1 - y0 + np.pi) % (2 * np.pi) - np.pi)
    d.t0[:] = [float(v) for v in T0[:3, 3]]
    d.t1[:] = [float(v) for v in T1[:3, 3]]
    d.r1[:] = [float(v) for v in T1[:3, :3].reshape(9)]
    return d


# ----------------------------------------------------------- entry points
def integrate_frame(grid, bank, scan, params, threads: int = 1):
    """integrator.integrate_frame on the GPU: same FrameStats fields
    (voxels_written is the engine's concurrent change count unless
    $DBT_EXACT_VOXELS_WRITTEN=1), same in-place grid mutation."""
    t0 = time.perf_counter()
    if scan.points.shape[0] == 0:
        return FrameStats()
    downsample = params.downsample
    dk = _deskew(scan, params.compensation) if params.compensation != "none" else None
    if dk is not None:
        # deskewed on the device (bit-identical to motion_compensate)
        pts = np.ascontiguousarray(scan.points, np.float64)
        ts = None if scan.timestamps is None else np.ascontiguousarray(scan.timestamps, np.float64)
        pose = np.ascontiguousarray(scan.pose, np.float64)
        g = _upload(grid)
        prm = _params(params, flags=_exact_flag())
        st = Stats()
        _check(lib().dbt_integrate_frame_deskew(
            g, device_bank(bank), _ptr(pts), DBT_F64, pts.shape[0], None if ts is None else _ptr(ts),
            pose.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(dk), ctypes.byref(prm),
            ctypes.byref(st)))
        _download(grid)
        grid.h_max, grid.t_occ = params.h_max, params.t_occ
        return FrameStats(int(st.points_in), int(st.points_discarded), int(st.voxels_written),
                          (time.perf_counter() - t0) * 1e3)
    if params.compensation != "none":
        if motion_compensate is None:
            raise RuntimeError("compensation needs the reference's motion_compensate")
        if downsample > 1:
            k = slice(None, None, downsample)
            scan = type(scan)(points=scan.points[k], pose=scan.pose,
                              timestamps=None if scan.timestamps is None else scan.timestamps[k],
                              prev_pose=scan.prev_pose)
            downsample = 1
        scan = motion_compensate(scan, params.compensation)
    pts = np.ascontiguousarray(scan.points, np.float64)  # ScanFrame holds float64 (integrator.py:43)
    # float32 scans widened by ScanFrame go over the link at half the bytes
    p32 = pts.astype(np.float32)
    exact32 = bool(np.array_equal(p32.astype(np.float64), pts, equal_nan=True))
    payload, dtype = (p32, DBT_F32) if exact32 else (pts, DBT_F64)
    pose = np.ascontiguousarray(scan.pose, np.float64)
    g = _upload(grid)
    prm = _params(params, flags=_exact_flag(), downsample=downsample)
    st = Stats()
    _check(lib().dbt_integrate_frame(g, device_bank(bank), _ptr(payload), dtype, payload.shape[0],
                                     pose.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(prm),
                                     ctypes.byref(st)))
    _download(grid)
    grid.h_max, grid.t_occ = params.h_max, params.t_occ
    return FrameStats(int(st.points_in), int(st.points_discarded), int(st.voxels_written),
                      (time.perf_counter() - t0) * 1e3)


def integrate_point(grid, bank, p_map, sensor_pos, params) -> str:
    """integrator.integrate_point on the GPU: "applied" or "discarded"."""
    p = np.asarray(p_map, np.float64).reshape(1, 3)
    s = np.asarray(sensor_pos, np.float64).reshape(1, 3)
    if np.linalg.norm(p[0] - s[0]) < grid.voxel_size:  # the reference's 1-D norm (integrator.py:173-175)
        return "discarded"
    g = _upload(grid)
    prm = _params(params, flags=FLAG_MAP_FRAME | FLAG_SKIP_NORM_CHECK, downsample=1)
    prm.first_return = 0
    st = Stats()
    out = np.zeros(1, np.int8)
    _check(lib().dbt_integrate_points_map(g, device_bank(bank), _ptr(p), _ptr(s), 1, ctypes.byref(prm),
                                          ctypes.byref(st), _ptr(out)))
    _download(grid)
    grid.h_max, grid.t_occ = params.h_max, params.t_occ
    return "applied" if out[0] else "discarded"


def mc_tables(tables_module=None) -> McTables:
    """dbt_mc_tables from the reference's bitsdf._mc_tables (or any module /
    mapping with EDGE_TABLE, TRI_TABLE, CORNER_OFFSETS, EDGE_BASE, EDGE_AXIS)."""
    if tables_module is None:
        try:
            from . import _mc_tables as tables_module  # type: ignore
        except ImportError:
            from bitsdf import _mc_tables as tables_module  # type: ignore
    get = (lambda k: tables_module[k]) if isinstance(tables_module, dict) or hasattr(tables_module, "files") \
        else (lambda k: getattr(tables_module, k))
    t = McTables()
    for f, k in (("edge_table", "EDGE_TABLE"), ("tri_table", "TRI_TABLE"), ("corner_offsets", "CORNER_OFFSETS"),
                 ("edge_base", "EDGE_BASE"), ("edge_axis", "EDGE_AXIS")):
        a = np.ascontiguousarray(np.asarray(get(k)), np.int32).ravel()
        dst = getattr(t, f)
        if a.size != len(dst):
            raise ValueError(f"{k}: {a.size} entries, the ABI takes {len(dst)}")
        ctypes.memmove(dst, a.ctypes.data, a.nbytes)
    return t


def extract_mesh(grid, iso: float = 0.0, tables=None):
    """mesher.extract_mesh on the GPU: (vertices (n,3) float64, triangles
    (m,3) int64), identical to the reference's arrays."""
    g = _upload(grid)
    tab = tables if isinstance(tables, McTables) else mc_tables(tables)
    m, nv, nf = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib().dbt_mesh_extract(g, ctypes.c_double(iso), ctypes.byref(tab), ctypes.byref(m), ctypes.byref(nv),
                                  ctypes.byref(nf)))
    try:
        v = np.empty((nv.value, 3), np.float64)
        f = np.empty((nf.value, 3), np.int64)
        _check(lib().dbt_mesh_download(m, _ptr(v), _ptr(f)))
    finally:
        lib().dbt_mesh_destroy(m)
    return v, f
